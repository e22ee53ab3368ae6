"""Batched node skeletonisation on the GPU: the compress phase's
skeletonize_node (reference proj/include/gfmm/compress.hpp:149-187) for many nodes at once,
bit-identical to the reference on the same sampled blocks (C-ABI gofmm_skeletonize_batch)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L


@dataclass
class Skeleton:
    """Skeleton (compress.hpp:39-47) of one node, in pivot terms: ``skel`` are column indices of
    the node's block (candidates[skel] are the reference's skeleton ids)."""

    rank: int
    skel: np.ndarray        # rank pivot columns
    proj: np.ndarray        # rank x cols interpolation matrix (column-major)
    achieved_tol: float
    perm: np.ndarray        # full column pivot order


def skeletonize_batch(blocks: list[np.ndarray], s: int, tau: float, device: int = 0,
                      stats: dict | None = None) -> list[Skeleton]:
    """ID of every block K(sample_cols, candidates) (rows x cols, float64) as skeletonize_node
    computes it: column-pivoted QR, rank = #{l: |R_ll| > tau |R_11|} clamped to [1, s]."""
    n = len(blocks)
    rows = np.array([b.shape[0] for b in blocks], dtype=np.int32)
    cols = np.array([b.shape[1] for b in blocks], dtype=np.int32)
    off = np.zeros(n, dtype=np.int64)
    if n:
        off[1:] = np.cumsum(rows.astype(np.int64) * cols)[:-1]
    blob = np.concatenate([np.asfortranarray(b, dtype=np.float64).ravel(order="F") for b in blocks]) if n \
        else np.zeros(1)
    maxr = np.minimum(np.minimum(rows, cols), s).astype(np.int64)
    perm = np.zeros(max(int(cols.sum()), 1), dtype=np.int32)
    proj = np.zeros(max(int((maxr * cols).sum()), 1), dtype=np.float64)
    rank = np.zeros(max(n, 1), dtype=np.int32)
    ach = np.zeros(max(n, 1), dtype=np.float64)
    st = L.SkelStats()
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = L.lib().gofmm_skeletonize_batch(n, p(rows), p(cols), p(off), p(blob), int(s), float(tau), int(device),
                                         p(rank), p(ach), p(perm), p(proj), C.byref(st))
    if rc != L.GOFMM_OK:
        msg = L.lib().gofmm_skeletonize_last_error().decode()
        raise (L.InvalidArgument if rc == L.GOFMM_ERR_INVALID else L.GofmmError)(rc, msg)
    if stats is not None:
        stats.update(seconds=st.seconds, kernel_ms=st.kernel_ms, bytes=st.bytes, flops=st.flops)
    out, po, pp = [], 0, 0
    for t in range(n):
        k, c = int(rank[t]), int(cols[t])
        pr = proj[pp:pp + k * c].reshape((k, c), order="F").copy()
        pm = perm[po:po + c].copy()
        out.append(Skeleton(k, pm[:k].copy(), pr, float(ach[t]), pm))
        po += c
        pp += int(maxr[t]) * c
    return out
