"""ctypes bindings to the ORACLE (oracle/_ref/libgfmm_ref.so) — TEST INFRASTRUCTURE ONLY.

The library is the reference GOFMM (``/root/reference/proj/include/gfmm``) compiled unmodified
against ``oracle/eigen_shim`` by ``oracle/Makefile``. Only ``tests/``, ``__graft_entry__.smoke()``
and bench.py's reference / cpu_baseline legs may import this module; the product package
(``paper_1707_00164_b200``) never does.

Entry points mirror the reference API they drive:
  compress_*      -> gfmm::compress             (compress.hpp:331-434)
  RefHMatrix.evaluate -> gfmm::evaluate         (evaluate.hpp:287-317)
  RefHMatrix.error_eps2 -> gfmm::error_eps2     (evaluate.hpp:330-373)
  RefHMatrix.unpermute -> gfmm::unpermute       (evaluate.hpp:21-25)
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libgfmm_ref.so")

# kernel ids (shared with include/gofmm_b200.h)
GAUSSIAN, LAPLACE, POLYNOMIAL, COSINE, EXPONENTIAL = 0, 1, 2, 3, 4
# DistanceKind (metric.hpp:8)
GEOM, KERNEL, ANGLE = 0, 1, 2
LEVEL_BY_LEVEL, TASK_DAG = 0, 1


def _find_openblas() -> str:
    """scipy's bundled OpenBLAS (LP64, ``scipy_cblas_dgemm``) backs the shim's products."""
    try:
        import scipy  # noqa: F401

        base = os.path.dirname(os.path.dirname(scipy.__file__))
    except Exception:  # pragma: no cover
        return ""
    hits = sorted(glob.glob(os.path.join(base, "scipy.libs", "libscipy_openblas-*.so")))
    return hits[0] if hits else ""


def build(force: bool = False) -> str:
    """Compile the oracle (needs /root/reference; on the GPU box the prebuilt .so travels)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


class RefConfig(C.Structure):
    """gfmm::RunConfig (compress.hpp:12-34) defaults."""

    _fields_ = [
        ("m", C.c_int32), ("s", C.c_int32), ("tau", C.c_double), ("kappa", C.c_int32),
        ("budget", C.c_double), ("kind", C.c_int32), ("seed", C.c_uint64), ("r", C.c_int32),
        ("ann_iterations", C.c_int32), ("threads", C.c_int32),
    ]

    @classmethod
    def make(cls, m=256, s=256, tau=1e-5, kappa=32, budget=0.03, kind=KERNEL, seed=0, r=1,
             ann_iterations=10, threads=1):
        return cls(m, s, tau, kappa, budget, kind, seed, r, ann_iterations, threads)


class _Sizes(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("num_nodes", C.c_int32), ("depth", C.c_int32), ("num_leaves", C.c_int32),
        ("dim", C.c_int32), ("has_points", C.c_int32),
        ("skel_total", C.c_int64), ("proj_total", C.c_int64), ("num_near", C.c_int64),
        ("num_far", C.c_int64), ("diag_total", C.c_int64), ("near_total", C.c_int64),
        ("far_total", C.c_int64),
    ]


_P = C.c_void_p


class _ExportArgs(C.Structure):
    _fields_ = [(n, _P) for n in (
        "parent", "left", "right", "level", "start", "end", "iperm", "rank", "ncand", "skel_off",
        "skel_idx", "proj_off", "proj", "near_a", "near_b", "far_a", "far_b", "diag_off", "diag",
        "near_off", "near_blk", "far_off", "far_blk", "coords")]


class _ImportArgs(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("num_nodes", C.c_int32), ("kernel", C.c_int32), ("dim", C.c_int32),
        ("p0", C.c_double), ("p1", C.c_double), ("coords", _P),
        ("parent", _P), ("left", _P), ("right", _P), ("level", _P), ("start", _P), ("end", _P),
        ("iperm", _P), ("rank", _P), ("skel_off", _P), ("skel_idx", _P), ("proj_off", _P),
        ("proj", _P), ("num_near", C.c_int64), ("near_a", _P), ("near_b", _P),
        ("num_far", C.c_int64), ("far_a", _P), ("far_b", _P), ("threads", C.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            if os.path.isdir("/root/reference"):
                build()
            else:
                raise RuntimeError(f"oracle library missing: {LIB_PATH} (build it where /root/reference exists)")
        os.environ.setdefault("GFMM_SHIM_BLAS", _find_openblas())
        L = C.CDLL(LIB_PATH)
        L.gfmm_ref_last_error.restype = C.c_char_p
        L.gfmm_ref_compress_kernel.argtypes = [C.c_int32, _P, C.c_int32, C.c_int32, C.c_double,
                                               C.c_double, C.POINTER(RefConfig), C.POINTER(_P)]
        L.gfmm_ref_compress_dense.argtypes = [_P, C.c_int32, C.POINTER(RefConfig), C.POINTER(_P)]
        L.gfmm_ref_compress_randspd.argtypes = [C.c_int32, C.c_uint64, C.POINTER(RefConfig), C.POINTER(_P)]
        L.gfmm_ref_free.argtypes = [_P]
        L.gfmm_ref_points_gaussian.argtypes = [C.c_int32, C.c_int32, C.c_uint64, _P]
        L.gfmm_ref_rng_gauss.argtypes = [C.c_int64, C.c_int32, C.c_uint64, C.c_uint64, _P]
        L.gfmm_ref_splitmix64.argtypes = [C.c_uint64]
        L.gfmm_ref_splitmix64.restype = C.c_uint64
        L.gfmm_ref_default_laplace_floor.argtypes = [_P, C.c_int32, C.c_int32, C.c_uint64]
        L.gfmm_ref_default_laplace_floor.restype = C.c_double
        L.gfmm_ref_dense.argtypes = [_P, _P]
        L.gfmm_ref_exact_rows.argtypes = [_P, _P, C.c_int32, _P, C.c_int32, _P]
        L.gfmm_ref_get_sizes.argtypes = [_P, C.POINTER(_Sizes)]
        L.gfmm_ref_export.argtypes = [_P, C.POINTER(_ExportArgs)]
        L.gfmm_ref_import.argtypes = [C.POINTER(_ImportArgs), C.POINTER(_P)]
        L.gfmm_ref_evaluate.argtypes = [_P, _P, C.c_int32, C.c_int32, _P, C.c_int32, C.c_int32,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        L.gfmm_ref_unpermute.argtypes = [_P, _P, C.c_int32, _P]
        L.gfmm_ref_error_eps2.argtypes = [_P, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                          C.POINTER(C.c_double), _P, C.POINTER(C.c_int32),
                                          C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_double), _P]
        L.gfmm_ref_eps2_draw.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_uint64, _P, _P]
        L.gfmm_ref_compress_stats.argtypes = [_P] + [_P] * 6
        L.gfmm_ref_ann_leaves.argtypes = [_P, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_uint64,
                                          _P, _P, _P]
        L.gfmm_ref_ann_iteration.argtypes = [_P, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                             C.c_int32, C.c_uint64, C.c_int32, _P, _P, _P, C.POINTER(C.c_double)]
        L.gfmm_ref_skeletonize_batch.argtypes = [C.c_int32, _P, _P, _P, _P, C.c_int32, C.c_double, C.c_int32,
                                                 _P, _P, _P, _P, C.POINTER(C.c_double)]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().gfmm_ref_last_error().decode())


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------------ generators (reference RNG)

def points_gaussian(n: int, d: int, seed: int) -> np.ndarray:
    """PointCloud::random_gaussian (oracle.hpp:18-25): returns d x n (Fortran order)."""
    out = np.empty((d, n), dtype=np.float64, order="F")
    lib().gfmm_ref_points_gaussian(n, d, seed, _ptr(out))
    return out


def rng_gauss(n: int, r: int, seed: int, stream: int = 0) -> np.ndarray:
    """random_rhs (test_evaluate.cpp:15-21): n x r column-major standard normals."""
    out = np.empty((n, r), dtype=np.float64, order="F")
    lib().gfmm_ref_rng_gauss(n, r, seed, stream, _ptr(out))
    return out


def splitmix64(x: int) -> int:
    return int(lib().gfmm_ref_splitmix64(x))


def default_laplace_floor(coords: np.ndarray, seed: int = 0) -> float:
    c = np.asfortranarray(coords, dtype=np.float64)
    return float(lib().gfmm_ref_default_laplace_floor(_ptr(c), c.shape[0], c.shape[1], seed))


def eps2_draw(n: int, r: int, sample_rows: int, seed: int):
    """error_eps2's first RNG draws (evaluate.hpp:336-346): (rows, W)."""
    k = min(sample_rows, n)
    rows = np.empty(k, dtype=np.int32)
    w = np.empty((n, r), dtype=np.float64, order="F")
    _check(lib().gfmm_ref_eps2_draw(n, r, sample_rows, seed, _ptr(rows), _ptr(w)))
    return rows, w


# ------------------------------------------------------------------ compressed structure

@dataclass
class Flat:
    """Flattened HMatrix (compress.hpp:65-79) in the layout include/gofmm_b200.h consumes."""

    n: int
    depth: int
    parent: np.ndarray
    left: np.ndarray
    right: np.ndarray
    level: np.ndarray
    start: np.ndarray
    end: np.ndarray
    iperm: np.ndarray
    rank: np.ndarray
    ncand: np.ndarray
    skel_off: np.ndarray
    skel_idx: np.ndarray
    proj_off: np.ndarray
    proj: np.ndarray
    near_a: np.ndarray
    near_b: np.ndarray
    far_a: np.ndarray
    far_b: np.ndarray
    diag_off: np.ndarray | None = None
    diag: np.ndarray | None = None
    near_off: np.ndarray | None = None
    near_blk: np.ndarray | None = None
    far_off: np.ndarray | None = None
    far_blk: np.ndarray | None = None
    coords: np.ndarray | None = None  # d x n, original order
    kernel: int = -1
    kparams: tuple = (0.0, 0.0)

    @property
    def num_nodes(self) -> int:
        return int(self.parent.shape[0])


class RefHMatrix:
    """A reference HMatrix living inside the oracle library."""

    def __init__(self, handle, kernel: int = -1, kparams=(0.0, 0.0)):
        self._h = handle
        self.kernel = kernel
        self.kparams = kparams

    def __del__(self):
        if getattr(self, "_h", None):
            lib().gfmm_ref_free(self._h)
            self._h = None

    def sizes(self) -> _Sizes:
        s = _Sizes()
        _check(lib().gfmm_ref_get_sizes(self._h, C.byref(s)))
        return s

    @property
    def n(self) -> int:
        return self.sizes().n

    def export(self, blocks: bool = True) -> Flat:
        s = self.sizes()
        nn, n = s.num_nodes, s.n
        i32 = lambda k: np.empty(k, dtype=np.int32)  # noqa: E731
        i64 = lambda k: np.empty(k, dtype=np.int64)  # noqa: E731
        f = Flat(
            n=n, depth=s.depth, parent=i32(nn), left=i32(nn), right=i32(nn), level=i32(nn),
            start=i32(nn), end=i32(nn), iperm=i32(n), rank=i32(nn), ncand=i32(nn),
            skel_off=i64(nn + 1), skel_idx=i32(max(s.skel_total, 1)), proj_off=i64(nn + 1),
            proj=np.empty(max(s.proj_total, 1)), near_a=i32(s.num_near), near_b=i32(s.num_near),
            far_a=i32(s.num_far), far_b=i32(s.num_far), kernel=self.kernel, kparams=self.kparams,
        )
        if blocks:
            f.diag_off, f.diag = i64(nn + 1), np.empty(max(s.diag_total, 1))
            f.near_off, f.near_blk = i64(s.num_near + 1), np.empty(max(s.near_total, 1))
            f.far_off, f.far_blk = i64(s.num_far + 1), np.empty(max(s.far_total, 1))
        if s.has_points:
            f.coords = np.empty((s.dim, n), dtype=np.float64, order="F")
        a = _ExportArgs()
        for name, _ in _ExportArgs._fields_:
            setattr(a, name, _ptr(getattr(f, name)))
        _check(lib().gfmm_ref_export(self._h, C.byref(a)))
        f.skel_idx = f.skel_idx[: s.skel_total]
        f.proj = f.proj[: s.proj_total]
        return f

    def evaluate(self, w: np.ndarray, mode: int = TASK_DAG, threads: int = 1):
        """gfmm::evaluate -> (u_perm, flops, seconds)."""
        w = np.asfortranarray(w, dtype=np.float64)
        if w.ndim == 1:
            w = w.reshape(-1, 1, order="F")
        u = np.empty_like(w, order="F")
        fl, sec = C.c_int64(), C.c_double()
        _check(lib().gfmm_ref_evaluate(self._h, _ptr(w), w.shape[0], w.shape[1], _ptr(u), mode, threads,
                                       C.byref(fl), C.byref(sec)))
        return u, fl.value, sec.value

    def unpermute(self, u_perm: np.ndarray) -> np.ndarray:
        u_perm = np.asfortranarray(u_perm, dtype=np.float64)
        out = np.empty_like(u_perm, order="F")
        _check(lib().gfmm_ref_unpermute(self._h, _ptr(u_perm), u_perm.shape[1], _ptr(out)))
        return out

    def error_eps2(self, r: int, sample_rows: int, seed: int, mode: int = TASK_DAG, threads: int = 1):
        n = self.n
        k = min(sample_rows, n) if sample_rows > 0 else 0
        rows = np.empty(max(k, 1), dtype=np.int32)
        first = np.empty(10)
        eps2, mean, sec = C.c_double(), C.c_double(), C.c_double()
        nfirst, fl = C.c_int32(), C.c_int64()
        _check(lib().gfmm_ref_error_eps2(self._h, r, sample_rows, seed, mode, threads, C.byref(eps2),
                                         _ptr(first), C.byref(nfirst), C.byref(mean), C.byref(fl),
                                         C.byref(sec), _ptr(rows)))
        return dict(eps2=eps2.value, per_entry=first[: nfirst.value].tolist(), mean_sample=mean.value,
                    eval_flops=fl.value, eval_seconds=sec.value, sample_rows=rows[:k].tolist())

    def dense(self) -> np.ndarray:
        n = self.n
        k = np.empty((n, n), dtype=np.float64, order="F")
        _check(lib().gfmm_ref_dense(self._h, _ptr(k)))
        return k

    def exact_rows(self, rows, w: np.ndarray) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        w = np.asfortranarray(w, dtype=np.float64)
        out = np.empty((rows.shape[0], w.shape[1]), dtype=np.float64, order="F")
        _check(lib().gfmm_ref_exact_rows(self._h, _ptr(rows), rows.shape[0], _ptr(w), w.shape[1], _ptr(out)))
        return out

    def compress_stats(self) -> dict:
        e, cf, ne = C.c_int64(), C.c_int64(), C.c_int64()
        ms, mean, sec = C.c_int32(), C.c_double(), C.c_double()
        _check(lib().gfmm_ref_compress_stats(self._h, C.byref(e), C.byref(cf), C.byref(ne), C.byref(ms),
                                             C.byref(mean), C.byref(sec)))
        return dict(entries_evaluated=e.value, compress_flops=cf.value, near_field_entries=ne.value,
                    max_skeleton=ms.value, mean_skeleton=mean.value, compress_seconds=sec.value)


def compress_kernel(kernel: int, coords: np.ndarray, p0: float, p1: float = 0.0, **cfg) -> RefHMatrix:
    """gfmm::compress over a kernel oracle built from d x n coordinates."""
    c = np.asfortranarray(coords, dtype=np.float64)
    h = C.c_void_p()
    conf = RefConfig.make(**cfg)
    _check(lib().gfmm_ref_compress_kernel(kernel, _ptr(c), c.shape[0], c.shape[1], p0, p1, C.byref(conf),
                                          C.byref(h)))
    if kernel == LAPLACE and p0 < 0:
        p0 = default_laplace_floor(c)
    return RefHMatrix(h, kernel, (p0, p1))


def compress_dense(K: np.ndarray, **cfg) -> RefHMatrix:
    k = np.asfortranarray(K, dtype=np.float64)
    h = C.c_void_p()
    conf = RefConfig.make(**cfg)
    _check(lib().gfmm_ref_compress_dense(_ptr(k), k.shape[0], C.byref(conf), C.byref(h)))
    return RefHMatrix(h)


def compress_randspd(n: int, seed: int, **cfg) -> RefHMatrix:
    """random_spd_oracle(n, seed) (oracle.hpp:321-333) then compress."""
    h = C.c_void_p()
    conf = RefConfig.make(**cfg)
    _check(lib().gfmm_ref_compress_randspd(n, seed, C.byref(conf), C.byref(h)))
    return RefHMatrix(h)


def import_flat(f: Flat, threads: int = 1) -> RefHMatrix:
    """Build a reference HMatrix (blocks via the reference oracle) from a flattened structure."""
    if f.coords is None or f.kernel < 0:
        raise ValueError("import_flat needs coordinates and a kernel id")
    a = _ImportArgs()
    a.n, a.num_nodes, a.kernel, a.dim = f.n, f.num_nodes, f.kernel, f.coords.shape[0]
    a.p0, a.p1 = float(f.kparams[0]), float(f.kparams[1])
    keep = {}
    for name in ("coords", "parent", "left", "right", "level", "start", "end", "iperm", "rank",
                 "skel_off", "skel_idx", "proj_off", "proj", "near_a", "near_b", "far_a", "far_b"):
        arr = getattr(f, name)
        dt = {"coords": np.float64, "proj": np.float64, "skel_off": np.int64, "proj_off": np.int64}.get(name, np.int32)
        arr = np.asfortranarray(arr, dtype=dt) if name == "coords" else np.ascontiguousarray(arr, dtype=dt)
        if arr.size == 0:
            arr = np.zeros(1, dtype=dt)
        keep[name] = arr
        setattr(a, name, _ptr(arr))
    a.num_near, a.num_far, a.threads = len(f.near_a), len(f.far_a), threads
    h = C.c_void_p()
    _check(lib().gfmm_ref_import(C.byref(a), C.byref(h)))
    return RefHMatrix(h, f.kernel, f.kparams)


def skeletonize_batch(blocks, s: int, tau: float, threads: int = 1):
    """The reference skeletonize_node (compress.hpp:149-187) on given blocks (rows x cols):
    list of (rank, skel pivot columns, proj rank x cols, achieved_tol), and the wall seconds."""
    n = len(blocks)
    rows = np.array([b.shape[0] for b in blocks], dtype=np.int32)
    cols = np.array([b.shape[1] for b in blocks], dtype=np.int32)
    off = np.zeros(n, dtype=np.int64)
    if n:
        off[1:] = np.cumsum(rows.astype(np.int64) * cols)[:-1]
    blob = np.concatenate([np.asfortranarray(b, dtype=np.float64).ravel(order="F") for b in blocks])
    maxr = np.minimum(np.minimum(rows, cols), s).astype(np.int64)
    skel = np.zeros(int(cols.sum()), dtype=np.int32)
    proj = np.zeros(max(int((maxr * cols).sum()), 1), dtype=np.float64)
    rank = np.zeros(n, dtype=np.int32)
    ach = np.zeros(n, dtype=np.float64)
    sec = C.c_double(0.0)
    _check(lib().gfmm_ref_skeletonize_batch(n, _ptr(rows), _ptr(cols), _ptr(off), _ptr(blob), int(s), float(tau),
                                            int(threads), _ptr(rank), _ptr(ach), _ptr(skel), _ptr(proj),
                                            C.byref(sec)))
    out, so, pp = [], 0, 0
    for t in range(n):
        k, c = int(rank[t]), int(cols[t])
        out.append((k, skel[so:so + k].copy(), proj[pp:pp + k * c].reshape((k, c), order="F").copy(),
                    float(ach[t])))
        so += c
        pp += int(maxr[t]) * c
    return out, sec.value


def ann_leaves(coords: np.ndarray, kind: int, h: float, m: int, seed: int):
    """Leaves of build_random_tree(metric, m, seed) (tree.hpp:244-247) as (leaf_off, leaf_idx)."""
    d, n = coords.shape
    cf = np.asfortranarray(coords, dtype=np.float64)
    off = np.zeros(n + 1, dtype=np.int32)
    idx = np.zeros(n, dtype=np.int32)
    nl = C.c_int32(0)
    _check(lib().gfmm_ref_ann_leaves(_ptr(cf), d, n, int(kind), float(h), int(m), C.c_uint64(seed),
                                     _ptr(off), _ptr(idx), C.byref(nl)))
    return off[:nl.value + 1].copy(), idx


def ann_iteration(coords: np.ndarray, kind: int, h: float, kappa: int, m: int, seed: int, tj, td, tlen,
                  threads: int = 1) -> float:
    """One reference ann_iteration (neighbors.hpp:88-106) on the table (tj, td: n x kappa, tlen: n),
    updated in place; returns the wall seconds."""
    d, n = coords.shape
    cf = np.asfortranarray(coords, dtype=np.float64)
    sec = C.c_double(0.0)
    _check(lib().gfmm_ref_ann_iteration(_ptr(cf), d, n, int(kind), float(h), int(kappa), int(m), C.c_uint64(seed),
                                        int(threads), _ptr(tj), _ptr(td), _ptr(tlen), C.byref(sec)))
    return sec.value
