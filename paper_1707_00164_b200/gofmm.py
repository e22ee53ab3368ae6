"""Host-side mirror of the reference evaluate API over the C-ABI (include/gofmm_b200.h).

Reference interface replaced (same names, argument meaning and error behaviour):
    gfmm::Potentials evaluate(const HMatrix&, const Matrix& w, const EvalOptions&)
        -> Evaluator.evaluate(w)                       evaluate.hpp:287-317
    gfmm::unpermute(const MetricTree&, const Matrix&) -> Evaluator.unpermute(u_perm)
                                                       evaluate.hpp:21-25
    struct Potentials { Matrix u; long long flops; double seconds; }
                                                       evaluate.hpp:15-19
The compressed input is the reference HMatrix (compress.hpp:65-79) flattened into
``CompressedTree``. All compute runs in the sm_100a extension; this module only marshals arrays.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib as L


@dataclass
class CompressedTree:
    """Flattened HMatrix: node table (tree.hpp:13-46), skeletons (compress.hpp:39-47), near/far lists."""

    n: int
    parent: np.ndarray
    left: np.ndarray
    right: np.ndarray
    level: np.ndarray
    start: np.ndarray
    end: np.ndarray
    iperm: np.ndarray
    rank: np.ndarray          # -1 = invalid skeleton (root)
    skel_off: np.ndarray      # [num_nodes+1]
    skel_idx: np.ndarray
    proj_off: np.ndarray      # [num_nodes+1]
    proj: np.ndarray          # per node rank x ncand column-major
    near_a: np.ndarray
    near_b: np.ndarray
    far_a: np.ndarray
    far_b: np.ndarray
    coords: np.ndarray | None = None   # d x n original order (kernel sources)
    kernel: int = -1
    kparams: tuple = (0.0, 0.0)
    diag_off: np.ndarray | None = None  # stored sources (DenseOracle-backed trees)
    diag: np.ndarray | None = None
    near_off: np.ndarray | None = None
    near_blk: np.ndarray | None = None
    far_off: np.ndarray | None = None
    far_blk: np.ndarray | None = None
    depth: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def num_nodes(self) -> int:
        return int(self.parent.shape[0])

    @classmethod
    def from_any(cls, obj) -> "CompressedTree":
        """Adopt any object with the same field names (e.g. a test oracle's export)."""
        names = {f.name for f in fields(cls)}
        return cls(**{k: getattr(obj, k) for k in names if hasattr(obj, k)})


@dataclass
class Potentials:
    """evaluate.hpp:15-19 — u is N x r in PERMUTED (tree) order."""

    u: np.ndarray
    flops: int
    seconds: float
    stats: dict = field(default_factory=dict)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def make_desc(tree: CompressedTree, stored: bool | None = None):
    """Flatten a CompressedTree into the C descriptor; returns (desc, keepalive list, stored flag)."""
    keep = []

    def k(a):
        keep.append(a)
        return _p(a)

    d = L.TreeDesc()
    d.n, d.num_nodes = int(tree.n), tree.num_nodes
    d.parent, d.left, d.right = k(_i32(tree.parent)), k(_i32(tree.left)), k(_i32(tree.right))
    d.level, d.start, d.end = k(_i32(tree.level)), k(_i32(tree.start)), k(_i32(tree.end))
    d.iperm, d.rank = k(_i32(tree.iperm)), k(_i32(tree.rank))
    d.skel_offset, d.skel_idx = k(_i64(tree.skel_off)), k(_i32(np.append(tree.skel_idx, 0)))
    d.proj_offset, d.proj = k(_i64(tree.proj_off)), k(_f64(np.append(tree.proj, 0.0)))
    d.num_near, d.near_a, d.near_b = len(tree.near_a), k(_i32(np.append(tree.near_a, 0))), k(
        _i32(np.append(tree.near_b, 0)))
    d.num_far, d.far_a, d.far_b = len(tree.far_a), k(_i32(np.append(tree.far_a, 0))), k(
        _i32(np.append(tree.far_b, 0)))
    use_stored = stored if stored is not None else (tree.coords is None or tree.kernel < 0)
    if use_stored:
        if tree.diag is None:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "stored source needs diag/near/far blocks")
        d.source = L.SOURCE_STORED
        d.diag_offset, d.diag_blocks = k(_i64(tree.diag_off)), k(_f64(tree.diag))
        d.near_offset, d.near_blocks = k(_i64(tree.near_off)), k(_f64(tree.near_blk))
        d.far_offset, d.far_blocks = k(_i64(tree.far_off)), k(_f64(tree.far_blk))
    else:
        d.source = L.SOURCE_KERNEL
        d.kernel = int(tree.kernel)
        coords = np.asfortranarray(tree.coords, dtype=np.float64)
        d.dim = int(coords.shape[0])
        d.coords = k(coords)
        for i, v in enumerate(tree.kparams[:4]):
            d.kparam[i] = float(v)
    return d, keep, use_stored


def rng_eps2_draw(seed: int, n: int, r: int, sample_rows: int, attempt: int = 0):
    """error_eps2's draws from the reference Rng (evaluate.hpp:336-346): (rows, W of `attempt`)."""
    k = min(sample_rows, n)
    rows = np.empty(k, dtype=np.int32)
    w = np.empty((n, r), dtype=np.float64, order="F")
    L.check(L.lib().gofmm_rng_eps2_draw_attempt(seed, n, r, sample_rows, attempt, _p(rows), _p(w), n))
    return rows, w


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library's NCCL (rank 0 calls it; the caller broadcasts it)."""
    buf = C.create_string_buffer(128)
    L.check(L.lib().gofmm_nccl_unique_id(buf))
    return buf.raw


def dist_plan_host(tree: CompressedTree, rank: int, nranks: int) -> tuple[dict, list[int]]:
    """Host-only subtree-split plan (no device): info and the exported ids in send order
    (what: node id; W rows: -(leaf id + 1))."""
    d, keep, _ = make_desc(tree)
    info = L.DistInfo()
    L.check(L.lib().gofmm_dist_plan_host(C.byref(d), rank, nranks, C.byref(info), 0, None))
    ids = np.zeros(max(info.n_exports, 1), dtype=np.int32)
    L.check(L.lib().gofmm_dist_plan_host(C.byref(d), rank, nranks, C.byref(info), info.n_exports, _p(ids)))
    return info.as_dict(), ids[:info.n_exports].tolist()


class Evaluator:
    """A compressed tree resident on one B200, ready for repeated u = K~ W (gofmm_create)."""

    def __init__(self, tree: CompressedTree, device: int = 0, near_mode: int = L.BLOCKS_MATRIX_FREE,
                 far_mode: int = L.BLOCKS_MATRIX_FREE, stored: bool | None = None, max_rhs_chunk: int = 0,
                 rank: int | None = None, nranks: int = 1, precision: str = "fp64"):
        """precision "fp64" (the reference's arithmetic, common.hpp:18) or "fp32" (north_star's
        1e-5 class: 3xTF32 on the tcgen05 tensor cores; W / u are float32)."""
        if precision not in ("fp64", "fp32"):
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, f"precision must be 'fp64' or 'fp32', not {precision!r}")
        self.tree = tree
        self.n = int(tree.n)
        self.precision = precision
        self.dtype = np.float64 if precision == "fp64" else np.float32
        lib = L.lib()
        d, keep, use_stored = make_desc(tree, stored)
        o = L.Options(device, near_mode, far_mode, max_rhs_chunk,
                      L.PRECISION_F64 if precision == "fp64" else L.PRECISION_F32)
        h = C.c_void_p()
        if rank is None:
            L.check(lib.gofmm_create(C.byref(d), C.byref(o), C.byref(h)))
        else:
            L.check(lib.gofmm_create_dist(C.byref(d), C.byref(o), rank, nranks, C.byref(h)))
        self._h = h
        self.stored = use_stored
        self.rank, self.nranks = rank, nranks

    def close(self):
        if getattr(self, "_h", None):
            L.lib().gofmm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ API
    def flops(self, r: int) -> int:
        """Reference flop counter (evaluate.hpp:154-214) for r right-hand sides."""
        return int(L.lib().gofmm_flops(self._h, r))

    def phase_flops(self, r: int) -> dict:
        """Reference flops split by phase: upward (N2S), downward (S2S+S2N), output (L2L+leaf S2N)."""
        out = np.zeros(3, dtype=np.int64)
        L.check(L.lib().gofmm_phase_flops(self._h, r, _p(out)))
        return dict(upward=int(out[0]), downward=int(out[1]), output=int(out[2]))

    def launch_profile(self, r: int) -> list[dict]:
        """Per-launch phase/level/flops and the CUDA-event ms of the last timed evaluation."""
        n = C.c_int32()
        L.check(L.lib().gofmm_launch_profile(self._h, r, 0, None, C.byref(n)))
        arr = (L.LaunchInfo * max(n.value, 1))()
        L.check(L.lib().gofmm_launch_profile(self._h, r, n.value, arr, C.byref(n)))
        names = ("upward", "downward", "output")
        return [dict(phase=names[x.phase], level=x.level, ctas=x.ctas, flops=x.flops, ms=x.ms,
                     generated=bool(x.generated)) for x in arr[:n.value]]

    @property
    def launches_per_eval(self) -> int:
        return int(L.lib().gofmm_launches_per_eval(self._h))

    @property
    def device_bytes(self) -> int:
        return int(L.lib().gofmm_device_bytes(self._h))

    def evaluate(self, w: np.ndarray, out: np.ndarray | None = None) -> Potentials:
        """u_perm = K~ w from HOST memory (the drop-in for gfmm::evaluate; evaluate.hpp:287-317).
        `out` (optional, N x r Fortran-ordered, e.g. a pinned buffer) receives u_perm."""
        w = np.asarray(w, dtype=self.dtype)
        if w.ndim == 1:
            w = w.reshape(-1, 1)
        if w.shape[0] != self.n:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "evaluate: w has wrong row count")
        if w.shape[1] < 1:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "evaluate: w needs at least one column")
        w = np.asfortranarray(w)
        r = int(w.shape[1])
        if out is None:
            u = np.empty((self.n, r), dtype=self.dtype, order="F")
        else:
            u = out
            if u.shape != (self.n, r) or u.dtype != self.dtype or not u.flags.f_contiguous:
                raise L.InvalidArgument(L.GOFMM_ERR_INVALID,
                                        f"evaluate: out must be N x r {np.dtype(self.dtype).name} Fortran order")
        st = L.EvalStats()
        t0 = time.perf_counter()
        fn = L.lib().gofmm_evaluate if self.precision == "fp64" else L.lib().gofmm_evaluate_f32
        L.check(fn(self._h, _p(w), self.n, r, _p(u), self.n, C.byref(st)))
        secs = time.perf_counter() - t0
        return Potentials(u=u, flops=int(st.flops), seconds=secs, stats=_stats(st))

    def evaluate_device(self, w_ptr: int, ldw: int, r: int, u_ptr: int, ldu: int, stream: int = 0,
                        sync_stats: bool = False) -> dict:
        """Device-pointer variant (W and u_perm already resident in HBM); enqueues on `stream`."""
        st = L.EvalStats()
        fn = L.lib().gofmm_evaluate_device if self.precision == "fp64" else L.lib().gofmm_evaluate_device_f32
        # torch's default stream is the legacy NULL stream: pass cudaStreamLegacy (0x1) explicitly,
        # because NULL selects the handle's own stream in the C-ABI
        L.check(fn(self._h, C.c_void_p(w_ptr), ldw, r, C.c_void_p(u_ptr), ldu,
                                              C.c_void_p(stream if stream else 1), 1 if sync_stats else 0,
                                              C.byref(st)))
        return _stats(st)

    def evaluate_torch(self, w, out=None, sync_stats: bool = False):
        """u_perm = K~ w for CUDA torch tensors (column-major = transposed contiguous views)."""
        import torch

        tdt = torch.float64 if self.precision == "fp64" else torch.float32
        if not (w.is_cuda and w.dtype == tdt):
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, f"evaluate_torch: w must be a CUDA {tdt} tensor")
        if w.dim() != 2 or w.shape[0] != self.n:  # evaluate.hpp:288
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "evaluate: w has wrong row count")
        if w.shape[1] < 1:  # evaluate.hpp:289
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "evaluate: w needs at least one column")
        wt = _colmajor(w)
        r = int(w.shape[1])
        if out is None:
            out = torch.empty((r, self.n), dtype=tdt, device=w.device).t()
        else:
            _check_out(out, self.n, r, tdt, w.device)
        stream = torch.cuda.current_stream(w.device).cuda_stream
        stats = self.evaluate_device(wt.data_ptr(), wt.stride(1), r, out.data_ptr(), out.stride(1), stream,
                                     sync_stats)
        return out, stats

    # ------------------------------------------------------------------ subtree-split (multi-GPU)
    def dist_info(self) -> dict:
        info = L.DistInfo()
        L.check(L.lib().gofmm_dist_get_info(self._h, C.byref(info)))
        return info.as_dict()

    def send_elems(self, r: int) -> int:
        """Elements of this rank's all-gather slot: max_send_rows x r (FP64), twice that (FP32 hi/lo)."""
        return self.dist_info()["max_send_rows"] * r * (1 if self.precision == "fp64" else 2)

    def dist_stage1_torch(self, w, send):
        """Own-subtree upward pass + pack of this rank's exports into `send` (CUDA float64)."""
        import torch

        wt = _colmajor(w)
        stream = torch.cuda.current_stream(w.device).cuda_stream
        fn = L.lib().gofmm_dist_stage1 if self.precision == "fp64" else L.lib().gofmm_dist_stage1_f32
        L.check(fn(self._h, C.c_void_p(wt.data_ptr()), wt.stride(1), int(w.shape[1]),
                                          C.c_void_p(send.data_ptr()) if send.numel() else None,
                                          C.c_void_p(stream if stream else 1)))

    def dist_stage2_torch(self, recv, r: int, out):
        """Ghost unpack + top tree + downward + output of this rank's rows of u_perm (into `out`)."""
        import torch

        stream = torch.cuda.current_stream(out.device).cuda_stream
        fn = L.lib().gofmm_dist_stage2 if self.precision == "fp64" else L.lib().gofmm_dist_stage2_f32
        L.check(fn(self._h, C.c_void_p(recv.data_ptr()) if recv.numel() else None, r,
                                          C.c_void_p(out.data_ptr()), out.stride(1),
                                          C.c_void_p(stream if stream else 1)))

    def init_comm(self, unique_id: bytes):
        """Create the library-owned NCCL communicator of this rank (collective over all ranks)."""
        if len(unique_id) != 128:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "unique id must be 128 bytes")
        buf = C.create_string_buffer(bytes(unique_id), 128)
        L.check(L.lib().gofmm_dist_init_comm(self._h, buf))

    def attach_comm(self, comm_ptr: int):
        """Borrow an existing ncclComm_t (e.g. ProcessGroupNCCL._comm_ptr()) of the same NCCL."""
        L.check(L.lib().gofmm_dist_attach_comm(self._h, C.c_void_p(comm_ptr)))

    def dist_evaluate_torch(self, w, out, timed: bool = False) -> dict | None:
        """One distributed evaluation on the library's own data plane (stage 1 -> ncclAllGather ->
        stage 2, the own D + near output terms overlapping the all-gather); writes this rank's rows
        of u_perm into `out`. timed: {stage1_ms, allgather_ms, total_ms} (synchronises)."""
        import torch

        if w.dim() != 2 or w.shape[0] != self.n or w.shape[1] < 1:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "evaluate: w has wrong shape")
        wt = _colmajor(w)
        r = int(w.shape[1])
        _check_out(out, self.n, r, wt.dtype, w.device)
        stream = torch.cuda.current_stream(w.device).cuda_stream
        ms = (C.c_double * 3)()
        fn = L.lib().gofmm_dist_evaluate if self.precision == "fp64" else L.lib().gofmm_dist_evaluate_f32
        L.check(fn(self._h, C.c_void_p(wt.data_ptr()), wt.stride(1), r, C.c_void_p(out.data_ptr()), out.stride(1),
                   C.c_void_p(stream if stream else 1), 1 if timed else 0, ms))
        return dict(stage1_ms=ms[0], allgather_ms=ms[1], total_ms=ms[2]) if timed else None

    def evaluate_dist_torch(self, w, out, all_gather):
        """One distributed evaluation: stage1, all_gather(send) -> recv, stage2. `all_gather` maps
        this rank's flat send tensor to the rank-ordered concatenation of every rank's."""
        import torch

        info = self.dist_info()
        r = int(w.shape[1])
        send = torch.empty(self.send_elems(r), dtype=w.dtype, device=w.device)
        self.dist_stage1_torch(w, send)
        recv = all_gather(send)
        self.dist_stage2_torch(recv, r, out)
        return out

    # ------------------------------------------------------------------ error_eps2 (evaluate.hpp:330-373)
    def exact_rows(self, rows, w: np.ndarray) -> np.ndarray:
        """K(rows, all) @ w computed matrix-free on the device (evaluate.hpp:353)."""
        import torch

        rows = np.ascontiguousarray(rows, dtype=np.int32)
        w = np.asarray(w, dtype=np.float64)
        if w.ndim == 1:
            w = w.reshape(-1, 1)
        wd = torch.from_numpy(np.ascontiguousarray(w.T)).cuda().t()
        out = torch.empty((w.shape[1], rows.shape[0]), dtype=torch.float64, device="cuda").t()
        L.check(L.lib().gofmm_exact_rows(self._h, _p(rows), rows.shape[0], C.c_void_p(wd.data_ptr()), wd.stride(1),
                                         int(w.shape[1]), C.c_void_p(out.data_ptr()), out.stride(1), None))
        return out.cpu().numpy()

    def error_eps2(self, r: int, sample_rows: int, seed: int) -> dict:
        """error_eps2 (evaluate.hpp:330-373) through gofmm_error_eps2: the reference's draws (rows,
        then up to 3 W draws from Rng(seed, 0xe952)), this handle's evaluation and the exact rows of
        K W generated on the device. Same report fields as ErrorReport (evaluate.hpp:319-326)."""
        if sample_rows < 1:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "sample_rows must be >= 1")
        if r < 1:
            raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "r must be >= 1")
        rep = L.Eps2Report()
        rows = np.empty(min(sample_rows, self.n), dtype=np.int32)
        L.check(L.lib().gofmm_error_eps2(self._h, int(r), int(sample_rows), int(seed), C.byref(rep), _p(rows)))
        return dict(eps2=rep.eps2, per_entry=[rep.per_entry[i] for i in range(rep.num_per_entry)],
                    mean_sample=rep.mean_sample, sample_rows=rows.tolist(), eval_flops=rep.eval_flops,
                    eval_seconds=rep.eval_seconds)

    def unpermute(self, u_perm: np.ndarray) -> np.ndarray:
        """out.row(iperm[t]) = u_perm.row(t) (evaluate.hpp:21-25)."""
        u_perm = np.asarray(u_perm)
        out = np.empty_like(u_perm)
        out[np.asarray(self.tree.iperm, dtype=np.int64)] = u_perm
        return out


def _check_out(out, n: int, r: int, dtype, device) -> None:
    """A caller-supplied device output must be exactly what the kernels write: N x r, the handle's
    dtype, on w's device, column-major (stride(0) == 1, stride(1) >= N) — else the C side, which
    only sees a pointer and ldu, would write past the tensor."""
    if out.dim() != 2 or tuple(out.shape) != (n, r):
        raise L.InvalidArgument(L.GOFMM_ERR_INVALID, f"out must be {n} x {r}, got {tuple(out.shape)}")
    if out.dtype != dtype:
        raise L.InvalidArgument(L.GOFMM_ERR_INVALID, f"out must be {dtype}, got {out.dtype}")
    if out.device != device:
        raise L.InvalidArgument(L.GOFMM_ERR_INVALID, f"out must be on {device}, got {out.device}")
    if out.stride(0) != 1 or (r > 1 and out.stride(1) < n):
        raise L.InvalidArgument(L.GOFMM_ERR_INVALID, "out must be column-major (stride(0) == 1, stride(1) >= N)")


def _colmajor(t):
    """Return t if it is column-major (stride(0)==1), else a column-major copy."""
    if t.dim() == 2 and t.stride(0) == 1 and t.stride(1) >= t.shape[0]:
        return t
    return t.t().contiguous().t()


def _stats(st: L.EvalStats) -> dict:
    return {name: getattr(st, name) for name, _ in L.EvalStats._fields_}
