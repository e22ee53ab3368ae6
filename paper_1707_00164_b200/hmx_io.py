"""GHMX — on-disk format for a compressed tree (the flattened HMatrix, compress.hpp:65-79).

The reference has no HMatrix persistence (io.hpp:11-14 lists GFMM matrices, GPTS points and GNNT
neighbour dumps only). This file format decouples the (CPU, hours-long at
N = 2^20) compress from GPU evaluation: the oracle harness or any producer writes the tree once,
gofmm_create reads it on any box. Layout follows the reference's binary conventions (io.hpp:
magic | u32 version | little-endian fixed-width fields):

    "GHMX" | u32 version=1
    u64 n, num_nodes, num_near, num_far, skel_total, proj_total, dim   (dim = 0: no coordinates)
    i32 kernel, i32 has_blocks, f64 kparam0, f64 kparam1
    i32 parent, left, right, level, start, end [num_nodes]; i32 iperm [n]; i32 rank [num_nodes]
    i64 skel_off [num_nodes+1]; i32 skel_idx [skel_total]
    i64 proj_off [num_nodes+1]; f64 proj [proj_total]     (per node rank x ncand, column-major)
    i32 near_a, near_b [num_near]; i32 far_a, far_b [num_far]
    f64 coords [dim * n]                                    (d x n column-major, original order)
    if has_blocks: i64 diag_off [num_nodes+1], f64 diag, i64 near_off [num_near+1], f64 near_blk,
                   i64 far_off [num_far+1], f64 far_blk
"""
from __future__ import annotations

import numpy as np

from .gofmm import CompressedTree

MAGIC = b"GHMX"
VERSION = 1


def save(path: str, t: CompressedTree) -> None:
    nn = t.num_nodes
    dim = 0 if t.coords is None else int(np.asarray(t.coords).shape[0])
    has_blocks = int(t.diag is not None)
    with open(path, "wb") as f:
        f.write(MAGIC)
        np.array([VERSION], dtype="<u4").tofile(f)
        np.array([t.n, nn, len(t.near_a), len(t.far_a), len(t.skel_idx), len(t.proj), dim], dtype="<u8").tofile(f)
        np.array([int(t.kernel), has_blocks], dtype="<i4").tofile(f)
        kp = list(t.kparams) + [0.0, 0.0]
        np.array(kp[:2], dtype="<f8").tofile(f)
        for a in (t.parent, t.left, t.right, t.level, t.start, t.end, t.iperm, t.rank):
            np.asarray(a, dtype="<i4").tofile(f)
        np.asarray(t.skel_off, dtype="<i8").tofile(f)
        np.asarray(t.skel_idx, dtype="<i4").tofile(f)
        np.asarray(t.proj_off, dtype="<i8").tofile(f)
        np.asarray(t.proj, dtype="<f8").tofile(f)
        for a in (t.near_a, t.near_b, t.far_a, t.far_b):
            np.asarray(a, dtype="<i4").tofile(f)
        if dim:
            np.asfortranarray(t.coords, dtype="<f8").ravel(order="F").tofile(f)
        if has_blocks:
            for off, blk in ((t.diag_off, t.diag), (t.near_off, t.near_blk), (t.far_off, t.far_blk)):
                np.asarray(off, dtype="<i8").tofile(f)
                np.asarray(blk, dtype="<f8").tofile(f)


def load(path: str) -> CompressedTree:
    with open(path, "rb") as f:
        if f.read(4) != MAGIC:
            raise ValueError(f"bad magic in {path} (expected GHMX)")
        (ver,) = np.fromfile(f, dtype="<u4", count=1)
        if ver != VERSION:
            raise ValueError(f"unsupported GHMX version {ver}")
        n, nn, nnear, nfar, nskel, nproj, dim = (int(x) for x in np.fromfile(f, dtype="<u8", count=7))
        kernel, has_blocks = (int(x) for x in np.fromfile(f, dtype="<i4", count=2))
        kparams = tuple(float(x) for x in np.fromfile(f, dtype="<f8", count=2))

        def rd(dt, k):
            a = np.fromfile(f, dtype=dt, count=k)
            if a.shape[0] != k:
                raise ValueError(f"truncated GHMX file {path}")
            return a

        parent, left, right, level, start, end = (rd("<i4", nn) for _ in range(6))
        iperm = rd("<i4", n)
        rank = rd("<i4", nn)
        skel_off = rd("<i8", nn + 1)
        skel_idx = rd("<i4", nskel)
        proj_off = rd("<i8", nn + 1)
        proj = rd("<f8", nproj)
        near_a, near_b = rd("<i4", nnear), rd("<i4", nnear)
        far_a, far_b = rd("<i4", nfar), rd("<i4", nfar)
        coords = rd("<f8", dim * n).reshape((dim, n), order="F") if dim else None
        blocks = {}
        if has_blocks:
            for name, cnt in (("diag", nn + 1), ("near", nnear + 1), ("far", nfar + 1)):
                off = rd("<i8", cnt)
                blocks[name] = (off, rd("<f8", int(off[-1])))
    t = CompressedTree(n=n, parent=parent, left=left, right=right, level=level, start=start, end=end, iperm=iperm,
                       rank=rank, skel_off=skel_off, skel_idx=skel_idx, proj_off=proj_off, proj=proj, near_a=near_a,
                       near_b=near_b, far_a=far_a, far_b=far_b, coords=coords, kernel=kernel, kparams=kparams,
                       depth=int(level.max()) if nn else 0)
    if has_blocks:
        t.diag_off, t.diag = blocks["diag"]
        t.near_off, t.near_blk = blocks["near"]
        t.far_off, t.far_blk = blocks["far"]
    return t
