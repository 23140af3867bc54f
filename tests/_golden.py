"""Loader for tests/golden/*.npz (produced from the unmodified reference by
tests/golden/make_golden.py)."""
import os
from collections import defaultdict

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name))
    cases = defaultdict(dict)
    for key in z.files:
        case, field = key.split("::", 1)
        cases[case][field] = z[key]
    return dict(cases)
