"""B200-native LAPLEX hot path (arXiv 2605.24584): device plan, forward,
transpose, backward, phased and Gram products behind the reference's API."""
from .laplex import (  # noqa: F401
    AsymmetricCotangent, CudaError, NumericalBreakdown, DeviceOperator, Dispatch, DimensionMismatch, EmptyInput, Error,
    GramResult, InvalidArgument, InvalidSize, LaplexOperator, MatvecCotangents, NonFinite, PhaseAbsent,
    PhasePresent, SortedAnchors, gram_vjp_weights, kernel_launches, matvec_vjp, phased_matvec_vjp,
    prefix_decay_scan, sort_anchors, suffix_decay_scan, symmetric_matvec, sort_anchors_dev, decay_scan_dev, pool_trim,
)
