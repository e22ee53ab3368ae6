"""compress(): the evaluator's input from a point cloud, over the C-ABI
gofmm_compress (csrc/gofmm_compress.cu).

Reference interface replaced (same configuration fields and statistics):
    gfmm::HMatrix compress(const EntryOracle&, const PointCloud*, const RunConfig&)
                                                             compress.hpp:331-434
    struct RunConfig { m, s, tau, kappa, budget, kind, seed, ann_iterations, threads }
                                                             compress.hpp:12-34
    struct CompressStats { entries_evaluated, compress_flops, near_field_entries, ... }
                                                             compress.hpp:49-59
The kernel oracle is given by id + parameters + coordinates (oracle.hpp:141-219; the Matérn-1/2
kernel of BASELINE config 4). ``entries="host"`` reproduces the reference compress bit for bit
(entries on the host in the reference's formulas and reduction order, CPQR on the GPU);
``entries="device"`` generates ANN distances and sampled blocks on the GPU as well."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .gofmm import CompressedTree

DIST = {"geom": 0, "geometric": 0, "kernel": 1, "angle": 2}
ENTRIES = {"host": 0, "device": 1}


class CompressConfig(C.Structure):
    _fields_ = [("m", C.c_int32), ("s", C.c_int32), ("tau", C.c_double), ("kappa", C.c_int32),
                ("budget", C.c_double), ("distance", C.c_int32), ("seed", C.c_uint64),
                ("ann_iterations", C.c_int32), ("threads", C.c_int32), ("entries", C.c_int32),
                ("device", C.c_int32)]


class CompressStatsC(C.Structure):
    _fields_ = [("entries_evaluated", C.c_int64), ("compress_flops", C.c_int64),
                ("near_field_entries", C.c_int64), ("max_skeleton", C.c_int32),
                ("ann_iterations_done", C.c_int32), ("mean_skeleton", C.c_double),
                ("compress_seconds", C.c_double), ("tree_seconds", C.c_double),
                ("ann_recall", C.c_double * 64), ("ann_seconds", C.c_double), ("ann_kernel_ms", C.c_double),
                ("skeleton_seconds", C.c_double), ("skel_kernel_ms", C.c_double), ("depth", C.c_int32),
                ("num_nodes", C.c_int32), ("num_leaves", C.c_int32), ("reserved", C.c_int32),
                ("num_near", C.c_int64), ("num_far", C.c_int64)]


_bound = False


def _lib():
    global _bound
    lib = L.lib()
    if not _bound:
        P = C.c_void_p
        lib.gofmm_compress_default_config.argtypes = [C.POINTER(CompressConfig)]
        lib.gofmm_compress.argtypes = [C.c_int32, P, C.c_int32, C.c_int32, P, C.POINTER(CompressConfig),
                                       C.POINTER(P)]
        lib.gofmm_compressed_desc.argtypes = [P, C.POINTER(L.TreeDesc)]
        lib.gofmm_compressed_stats.argtypes = [P, C.POINTER(CompressStatsC)]
        lib.gofmm_compressed_free.argtypes = [P]
        lib.gofmm_compress_last_error.restype = C.c_char_p
        _bound = True
    return lib


@dataclass
class CompressResult:
    tree: CompressedTree
    stats: dict


def _arr(ptr, n, ct, dt):
    if n == 0:
        return np.zeros(0, dtype=dt)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).astype(dt, copy=True)


def compress(coords: np.ndarray, kernel: int = L.KERNEL_GAUSSIAN, kparams=(1.0, 0.0), *, m: int = 256,
             s: int = 256, tau: float = 1e-5, kappa: int = 32, budget: float = 0.03, distance: str = "kernel",
             seed: int = 0, ann_iterations: int = 10, threads: int | None = None, entries: str = "device",
             device: int = 0) -> CompressResult:
    """gfmm::compress over a kernel oracle of d x n coordinates (original order). Raises
    InvalidArgument on RunConfig::validate failures (compress.hpp:24-33)."""
    lib = _lib()
    x = np.asfortranarray(coords, dtype=np.float64)
    if x.ndim != 2:
        raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "coords must be d x n")
    cfg = CompressConfig()
    lib.gofmm_compress_default_config(C.byref(cfg))
    cfg.m, cfg.s, cfg.tau, cfg.kappa, cfg.budget = m, s, tau, kappa, budget
    if distance not in DIST or entries not in ENTRIES:
        raise L.InvalidArgument(L.GOFMM_ERR_INVALID, f"distance in {sorted(DIST)}, entries in {sorted(ENTRIES)}")
    cfg.distance, cfg.seed, cfg.ann_iterations = DIST[distance], seed, ann_iterations
    if threads is not None:
        cfg.threads = threads
    cfg.entries, cfg.device = ENTRIES[entries], device
    kp = np.zeros(4, dtype=np.float64)
    kp[:len(kparams)] = kparams
    h = C.c_void_p()
    rc = lib.gofmm_compress(int(kernel), kp.ctypes.data_as(C.c_void_p), x.shape[0], x.shape[1],
                            x.ctypes.data_as(C.c_void_p), C.byref(cfg), C.byref(h))
    if rc != L.GOFMM_OK:
        msg = lib.gofmm_compress_last_error().decode()
        if rc == L.GOFMM_ERR_INVALID:
            raise L.InvalidArgument(rc, msg)
        raise L.GofmmError(rc, msg)
    try:
        d = L.TreeDesc()
        L.check(lib.gofmm_compressed_desc(h, C.byref(d)))
        st = CompressStatsC()
        L.check(lib.gofmm_compressed_stats(h, C.byref(st)))
        nn, n = d.num_nodes, d.n
        i32, i64, f64 = (C.c_int32, np.int32), (C.c_int64, np.int64), (C.c_double, np.float64)
        skel_off = _arr(d.skel_offset, nn + 1, *i64)
        proj_off = _arr(d.proj_offset, nn + 1, *i64)
        tree = CompressedTree(
            n=n, parent=_arr(d.parent, nn, *i32), left=_arr(d.left, nn, *i32), right=_arr(d.right, nn, *i32),
            level=_arr(d.level, nn, *i32), start=_arr(d.start, nn, *i32), end=_arr(d.end, nn, *i32),
            iperm=_arr(d.iperm, n, *i32), rank=_arr(d.rank, nn, *i32), skel_off=skel_off,
            skel_idx=_arr(d.skel_idx, int(skel_off[-1]), *i32), proj_off=proj_off,
            proj=_arr(d.proj, int(proj_off[-1]), *f64), near_a=_arr(d.near_a, d.num_near, *i32),
            near_b=_arr(d.near_b, d.num_near, *i32), far_a=_arr(d.far_a, d.num_far, *i32),
            far_b=_arr(d.far_b, d.num_far, *i32), coords=x.copy(order="F"), kernel=int(kernel),
            kparams=tuple(float(v) for v in kp[:2]), depth=int(st.depth))
        stats = {name: getattr(st, name) for name, _ in CompressStatsC._fields_ if name != "ann_recall"}
        stats["ann_recall"] = [st.ann_recall[i] for i in range(st.ann_iterations_done)]
        stats.pop("reserved", None)
    finally:
        lib.gofmm_compressed_free(h)
    return CompressResult(tree=tree, stats=stats)
