"""One randomized-tree ANN pass on the GPU: the per-leaf body of the
reference's ann_iteration (proj/include/gfmm/neighbors.hpp:88-106) for every leaf of a host-built
random tree (C-ABI gofmm_ann_leaf_merge)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

GEOMETRIC = 0  # DistanceKind::GeometricL2 (metric.hpp:8)
KERNEL = 1     # DistanceKind::KernelL2 over a Gaussian oracle


def ann_leaf_merge(coords: np.ndarray, kind: int, h: float, kappa: int, leaf_off: np.ndarray,
                   leaf_idx: np.ndarray, table_j: np.ndarray, table_d: np.ndarray, table_len: np.ndarray,
                   device: int = 0) -> float:
    """Merge every leaf's pairwise candidates into the neighbor table (n x kappa, updated in
    place); returns the kernel milliseconds."""
    d, n = coords.shape
    cf = np.asfortranarray(coords, dtype=np.float64)
    lo = np.ascontiguousarray(leaf_off, dtype=np.int32)
    li = np.ascontiguousarray(leaf_idx, dtype=np.int32)
    for a, dt in ((table_j, np.int32), (table_d, np.float64), (table_len, np.int32)):
        if a.dtype != dt or not a.flags.c_contiguous:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "table arrays must be C-contiguous int32/float64/int32")
    ms = C.c_double(0.0)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = L.lib().gofmm_ann_leaf_merge(n, d, p(cf), int(kind), float(h), int(kappa), len(lo) - 1, p(lo), p(li),
                                      int(device), p(table_j), p(table_d), p(table_len), C.byref(ms))
    if rc != L.GOFMM_OK:
        msg = L.lib().gofmm_ann_last_error().decode()
        raise (L.InvalidArgument if rc == L.GOFMM_ERR_INVALID else L.GofmmError)(rc, msg)
    return ms.value
