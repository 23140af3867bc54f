"""Density callers of the drop-in: the reference's
FactorGaussian (proj/include/laplex/density.hpp:24-226) on the B200 operator.

Gaussian N(mean, D + F F^T) with D = diag(d^2) and F = sum_c diag(w_c) A L_c^T
for the implicit kernel operator A (n x k_lap).  F is never formed: every
product with F / F^T is ONE batched device call over all components (and all
right-hand sides) instead of the reference's per-component, per-vector
matvecs:

  apply_F(Z)   density.hpp:75-84   rows (s, c) = L_c^T z_s -> batch matvec -> sum_c w_c (.) y
  apply_Ft(R)  density.hpp:87-97   rows (s, c) = w_c (.) r_s -> batch matvec_transpose -> sum_c L_c y
  capacitance  density.hpp:99-124  M = I + sum_{c<=d} L_c G_cd L_d^T (+ mirror), G_cd one weighted
                                   Gram on the role-swapped operator (laplex_gram_dev)
  log_likelihood / map_reconstruct / sample   density.hpp:127-184 (Woodbury, Cholesky of M)
  FitDriver.build_blocks                      density.hpp:246-260: B_c = A L_c^T as ONE batch

The small k_lap x k_lap algebra (L_c products, Cholesky, solves) is cuBLAS /
cuSOLVER through torch (library calls, fp64); every product with A runs on the
library's kernels.  Validation order and error types follow the reference
(validate(), density.hpp:198-217).  `sample` draws its normals from torch's
generator, so draws match the reference in distribution, not bit for bit
(the reference uses std::mt19937_64 + std::normal_distribution).
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence

from .laplex import DeviceOperator, DimensionMismatch, EmptyInput, NonFinite, NumericalBreakdown


class FactorGaussian:
    """density.hpp:24-226 over a DeviceOperator (fp64 recommended, as the reference)."""

    def __init__(self, mean, diag_noise, weights: Sequence, op: DeviceOperator, factors: Sequence):
        import torch
        self.torch = torch
        self.op = op
        dev = torch.device("cuda", torch.cuda.current_device())
        t = lambda v: torch.as_tensor(v, dtype=op.dtype, device=dev)  # noqa: E731
        self.mean_ = t(mean).reshape(-1)
        self.diag_ = t(diag_noise).reshape(-1)
        self.weights_ = [t(w).reshape(-1) for w in weights]
        self.factors_ = [t(L) for L in factors]
        self._cap: Optional[object] = None
        self._chol: Optional[object] = None
        self._validate()

    # ---- shape (density.hpp:42-44) ----
    def n(self) -> int:
        return self.mean_.numel()

    def k_lap(self) -> int:
        return self.op.k

    def components(self) -> int:
        return len(self.weights_)

    def _validate(self):  # density.hpp:198-217, same order
        torch = self.torch
        nn = self.mean_.numel()
        if nn == 0:
            raise EmptyInput("FactorGaussian: empty mean")
        if self.op.n != nn:
            raise DimensionMismatch("FactorGaussian: operator rows")
        if self.diag_.numel() != nn:
            raise DimensionMismatch("FactorGaussian: diag length")
        if not self.weights_ or len(self.factors_) != len(self.weights_):
            raise DimensionMismatch("FactorGaussian: component counts")
        if not bool(torch.isfinite(self.mean_).all()):
            raise NonFinite("FactorGaussian mean: non-finite entry")
        if not bool(torch.isfinite(self.diag_).all()):
            raise NonFinite("FactorGaussian diag: non-finite entry")
        if not bool((self.diag_ > 0).all()):
            raise NonFinite("FactorGaussian: diag_noise must be positive")
        for w in self.weights_:
            if w.numel() != nn:
                raise DimensionMismatch("FactorGaussian: weight length")
            if not bool(torch.isfinite(w).all()):
                raise NonFinite("FactorGaussian weights: non-finite entry")
        kl = self.op.k
        for L in self.factors_:
            if L.dim() != 2 or L.shape[0] != kl or L.shape[1] != kl:
                raise DimensionMismatch("FactorGaussian: factor shape")
            if not bool(torch.isfinite(L).all()):
                raise NonFinite("FactorGaussian: non-finite factor")

    def _invalidate(self):
        self._cap = self._chol = None

    def set_mean(self, m):
        self.mean_ = self.torch.as_tensor(m, dtype=self.op.dtype, device=self.mean_.device).reshape(-1)
        self._invalidate()
        self._validate()

    def set_diag_noise(self, d):
        self.diag_ = self.torch.as_tensor(d, dtype=self.op.dtype, device=self.mean_.device).reshape(-1)
        self._invalidate()
        self._validate()

    # ---- operator products (op_matvec / op_matvec_transpose, density.hpp:189-195) ----
    def _matvec(self, X):
        return self.op.apply(X)  # phased operators: phased_matvec (the plan knows)

    def _matvec_transpose(self, G):
        if not self.op.phased:
            return self.op.apply(G, transpose=True)
        return self.op.transposed().apply(G)  # density.hpp:193: transposed().phased_matvec

    def apply_F(self, Z):
        """F z for one z (k_lap) or each row of Z (S x k_lap): density.hpp:75-84."""
        torch = self.torch
        single = Z.dim() == 1 if hasattr(Z, "dim") else True
        Z = torch.as_tensor(Z, dtype=self.op.dtype, device=self.mean_.device)
        Z = Z.reshape(1, -1) if Z.dim() == 1 else Z
        if Z.shape[1] != self.k_lap():
            raise DimensionMismatch("apply_F: z length")
        S, C = Z.shape[0], self.components()
        # rows ordered (s, c): L_c^T z_s == z_s L_c
        X = torch.stack([Z @ L for L in self.factors_], dim=1).reshape(S * C, -1).contiguous()
        Y = self._matvec(X).reshape(S, C, -1)
        out = torch.zeros((S, self.n()), dtype=self.op.dtype, device=Z.device)
        for c in range(C):  # component order as the reference's accumulation
            out += self.weights_[c] * Y[:, c]
        return out[0] if single else out

    def apply_Ft(self, Rm):
        """F^T r for one r (n) or each row of R (S x n): density.hpp:87-97."""
        torch = self.torch
        Rm = torch.as_tensor(Rm, dtype=self.op.dtype, device=self.mean_.device)
        single = Rm.dim() == 1
        Rm = Rm.reshape(1, -1) if single else Rm
        if Rm.shape[1] != self.n():
            raise DimensionMismatch("apply_Ft: r length")
        S, C = Rm.shape[0], self.components()
        W = torch.stack([self.weights_[c] * Rm for c in range(C)], dim=1).reshape(S * C, -1).contiguous()
        Y = self._matvec_transpose(W).reshape(S, C, -1)
        out = torch.zeros((S, self.k_lap()), dtype=self.op.dtype, device=Rm.device)
        for c in range(C):
            out += Y[:, c] @ self.factors_[c].T  # L_c y
        return out[0] if single else out

    # ---- capacitance M = I + F^T D^{-1} F (density.hpp:99-124) ----
    def capacitance(self):
        torch = self.torch
        if self._cap is None:
            kl, C = self.k_lap(), self.components()
            M = torch.eye(kl, dtype=self.op.dtype, device=self.mean_.device)
            swapped = self.op.transposed()
            d2 = self.diag_ * self.diag_
            for c in range(C):
                for d in range(c, C):
                    wts = self.weights_[c] * self.weights_[d] / d2
                    G = swapped.weighted_gram(wts.contiguous())
                    term = self.factors_[c] @ G @ self.factors_[d].T
                    M = M + (term if c == d else term + term.T)
            self._cap = M
            L, info = torch.linalg.cholesky_ex(M)
            if int(info.item()) != 0:
                raise NumericalBreakdown("capacitance: Cholesky factorization failed")
            self._chol = L
        return self._cap

    def _solve(self, rhs):
        self.capacitance()
        return self.torch.cholesky_solve(rhs.reshape(-1, 1), self._chol).reshape(-1)

    def log_likelihood(self, x) -> float:
        """log N(x; mean, Sigma) via Woodbury + the capacitance Cholesky (density.hpp:127-147)."""
        torch = self.torch
        x = torch.as_tensor(x, dtype=self.op.dtype, device=self.mean_.device).reshape(-1)
        if x.numel() != self.n():
            raise DimensionMismatch("log_likelihood: x length")
        self.capacitance()
        r = x - self.mean_
        d2 = self.diag_ * self.diag_
        rdi = r / d2
        quad = float((r * rdi).sum())
        logdet_d = float((2.0 * torch.log(self.diag_)).sum())
        u = self.apply_Ft(rdi)
        quad -= float(u @ self._solve(u))
        logdet_m = float((2.0 * torch.log(torch.diagonal(self._chol))).sum())
        return -0.5 * (quad + logdet_d + logdet_m + self.n() * math.log(2.0 * math.pi))

    def map_reconstruct(self, x):
        """(z*, x_hat): M z* = F^T D^{-1} (x - mean), x_hat = mean + F z* (density.hpp:151-162)."""
        torch = self.torch
        x = torch.as_tensor(x, dtype=self.op.dtype, device=self.mean_.device).reshape(-1)
        if x.numel() != self.n():
            raise DimensionMismatch("map_reconstruct: x length")
        rdi = (x - self.mean_) / (self.diag_ * self.diag_)
        z = self._solve(self.apply_Ft(rdi))
        if not bool(torch.isfinite(z).all()):
            raise NumericalBreakdown("map_reconstruct: solve failed")
        return z, self.apply_F(z) + self.mean_

    def sample(self, count: int, seed: int):
        """count draws x = mean + F z + d (.) eps as rows (density.hpp:165-179); all
        count draws' F z in one batched product."""
        torch = self.torch
        if count == 0:
            raise EmptyInput("sample: count must be >= 1")
        g = torch.Generator(device=self.mean_.device)
        g.manual_seed(int(seed))
        Z = torch.randn((count, self.k_lap()), generator=g, dtype=self.op.dtype, device=self.mean_.device)
        eps = torch.randn((count, self.n()), generator=g, dtype=self.op.dtype, device=self.mean_.device)
        return self.mean_ + self.apply_F(Z) + self.diag_ * eps

    # ---- FitDriver.build_blocks (density.hpp:246-260) ----
    def build_blocks(self):
        """B_c = A L_c^T (n x k_lap) for every component, and F = sum_c diag(w_c) B_c:
        the reference's k_lap matvecs per component as one batched call."""
        torch = self.torch
        C, kl = self.components(), self.k_lap()
        X = torch.cat(self.factors_, dim=0).contiguous()  # row p of L_c -> column p of B_c
        Y = self._matvec(X).reshape(C, kl, -1)
        B = [Y[c].T.contiguous() for c in range(C)]
        F = torch.zeros((self.n(), kl), dtype=self.op.dtype, device=X.device)
        for c in range(C):
            F += self.weights_[c][:, None] * B[c]
        return B, F
