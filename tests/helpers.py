"""Shared test helpers (checkers only; the product is never imported from oracle)."""
import hashlib

import numpy as np

CONFIGS = [(32, 14, 128), (32, 7, 128), (4, 4, 16)]
# build_xcache(FORCE_HUBS): a hub table whatever the matrix size (the
# automatic mode skips matrices too small for it to pay, i.e. every small
# test matrix; the hub code paths are tested with it forced)
FORCE_HUBS = 1 << 30


def h(*arrays):
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:32]


def tolerance_bound(a, x, dtype):
    """ToleranceBound (tests/support/checks.hpp:20-42): 4 eps len max|A| max|x|."""
    vals = np.asarray(a.values, np.float64)
    max_a = float(np.abs(vals).max(initial=0.0))
    max_x = float(np.abs(np.asarray(x, np.float64)).max(initial=0.0))
    eps = float(np.finfo(dtype).eps)
    lens = np.diff(a.row_offsets).astype(np.float64)
    return 4.0 * eps * lens * max_a * max_x


def first_violation(bound, want, got):
    diff = np.abs(np.asarray(got, np.float64) - np.asarray(want, np.float64))
    bad = np.nonzero(~(diff <= bound))[0]
    return int(bad[0]) if bad.size else -1
