"""Loader for the in-tree sm_100a extension ``_lib/libgofmm_b200.so`` (C-ABI of include/gofmm_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is present, every entry
point fails loudly (GofmmError with GOFMM_ERR_CUDA), mirroring north_star's "no CPU fallback".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "_lib", "libgofmm_b200.so")
CLI_PATH = os.path.join(PKG_DIR, "_lib", "gofmm_b200_cli")
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO_DIR, "include")

GOFMM_OK = 0
GOFMM_ERR_INVALID = 2
GOFMM_ERR_IO = 3
GOFMM_ERR_NUMERIC = 4
GOFMM_ERR_CUDA = 5

SOURCE_STORED = 0
SOURCE_KERNEL = 1
KERNEL_GAUSSIAN = 0
KERNEL_LAPLACE = 1
KERNEL_POLYNOMIAL = 2
KERNEL_EXPONENTIAL = 4
PRECISION_F64 = 0
PRECISION_F32 = 1
BLOCKS_MATRIX_FREE = 0
BLOCKS_MATERIALIZE = 1

# host code: no FP contraction (the compress pipeline reproduces the reference's SSE2 rounding)
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off"]
# translation units of the library, compiled in parallel then linked: the C-ABI + FP64 DMMA
# kernels, the FP32 3xTF32 tcgen05 kernels, and the compress-side batched skeletonisation and ANN pass
UNITS = ("gofmm_capi.cu", "gofmm_f32.cu", "gofmm_skel.cu", "gofmm_ann.cu", "gofmm_compress.cu")


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the CUDA extension in-tree with nvcc for sm_100a (cross-compiles without a GPU)."""
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cuh", ".h", ".cpp"))]
    srcs.append(os.path.join(INCLUDE, "gofmm_b200.h"))
    if not force and os.path.exists(LIB_PATH) and os.path.exists(CLI_PATH):
        newest = max(os.path.getmtime(s) for s in srcs)
        if min(os.path.getmtime(LIB_PATH), os.path.getmtime(CLI_PATH)) >= newest:
            return LIB_PATH
    out_dir = os.path.dirname(LIB_PATH)
    os.makedirs(out_dir, exist_ok=True)
    objs, procs = [], []
    for unit in UNITS:
        obj = os.path.join(out_dir, unit.replace(".cu", ".o"))
        cmd = ["nvcc", *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, unit)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(obj)
    for cmd, p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_PATH, *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    for obj in objs:
        os.remove(obj)
    # the command-line driver (gfmm_cli compress / bench over the C-ABI), next to the library
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-o", CLI_PATH, os.path.join(CSRC, "gofmm_cli.cpp"), "-L", out_dir,
           "-lgofmm_b200", "-Xlinker", "-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return LIB_PATH


class TreeDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("num_nodes", C.c_int32),
        ("parent", C.c_void_p), ("left", C.c_void_p), ("right", C.c_void_p), ("level", C.c_void_p),
        ("start", C.c_void_p), ("end", C.c_void_p), ("iperm", C.c_void_p),
        ("rank", C.c_void_p), ("skel_offset", C.c_void_p), ("skel_idx", C.c_void_p),
        ("proj_offset", C.c_void_p), ("proj", C.c_void_p),
        ("num_near", C.c_int64), ("near_a", C.c_void_p), ("near_b", C.c_void_p),
        ("num_far", C.c_int64), ("far_a", C.c_void_p), ("far_b", C.c_void_p),
        ("source", C.c_int32), ("kernel", C.c_int32), ("dim", C.c_int32), ("coords", C.c_void_p),
        ("kparam", C.c_double * 4),
        ("diag_offset", C.c_void_p), ("diag_blocks", C.c_void_p),
        ("near_offset", C.c_void_p), ("near_blocks", C.c_void_p),
        ("far_offset", C.c_void_p), ("far_blocks", C.c_void_p),
    ]


class Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("near_mode", C.c_int32), ("far_mode", C.c_int32),
                ("max_rhs_chunk", C.c_int32), ("precision", C.c_int32)]


class EvalStats(C.Structure):
    _fields_ = [("flops", C.c_int64), ("seconds", C.c_double), ("ms_permute", C.c_double),
                ("ms_upward", C.c_double), ("ms_downward", C.c_double), ("ms_output", C.c_double),
                ("ms_h2d", C.c_double), ("ms_d2h", C.c_double)]


class LaunchInfo(C.Structure):
    _fields_ = [("phase", C.c_int32), ("level", C.c_int32), ("ctas", C.c_int64), ("flops", C.c_int64),
                ("ms", C.c_double), ("generated", C.c_int32), ("reserved", C.c_int32)]


class DistInfo(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("split_level", C.c_int32), ("n_exports", C.c_int32),
                ("send_rows", C.c_int64), ("max_send_rows", C.c_int64), ("own_row_begin", C.c_int64),
                ("own_row_end", C.c_int64), ("flops_per_rhs", C.c_int64), ("full_flops_per_rhs", C.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class GofmmError(RuntimeError):
    """Raised for non-zero C-ABI return codes; ``code`` follows gfmm_cli.cpp:289-305."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(GofmmError, ValueError):
    """std::invalid_argument in the reference (evaluate.hpp:288-289)."""


_lib = None

# every symbol include/gofmm_b200.h declares
EXPORTS = ("gofmm_create", "gofmm_evaluate", "gofmm_evaluate_device", "gofmm_unpermute_device",
           "gofmm_flops", "gofmm_phase_flops", "gofmm_launch_profile", "gofmm_device_bytes", "gofmm_launches_per_eval", "gofmm_destroy",
           "gofmm_last_error", "gofmm_abi_version", "gofmm_create_dist", "gofmm_dist_get_info",
           "gofmm_dist_plan_host", "gofmm_dist_stage1", "gofmm_dist_stage2", "gofmm_exact_rows",
           "gofmm_rng_eps2_draw", "gofmm_evaluate_f32", "gofmm_evaluate_device_f32",
           "gofmm_unpermute_device_f32", "gofmm_precision", "gofmm_dist_stage1_f32", "gofmm_dist_stage2_f32",
           "gofmm_skeletonize_batch", "gofmm_skeletonize_last_error", "gofmm_ann_leaf_merge",
           "gofmm_ann_last_error", "gofmm_rng_eps2_draw_attempt", "gofmm_nccl_unique_id", "gofmm_dist_init_comm",
           "gofmm_dist_attach_comm", "gofmm_dist_evaluate", "gofmm_dist_evaluate_f32", "gofmm_compress_default_config",
           "gofmm_compress", "gofmm_compressed_desc", "gofmm_compressed_stats", "gofmm_compressed_free",
           "gofmm_compress_last_error", "gofmm_error_eps2", "gofmm_points_gaussian",
           "gofmm_default_laplace_floor", "gofmm_rng_gauss_stream", "gofmm_dist_evaluate_host")


class Eps2Report(C.Structure):
    _fields_ = [("eps2", C.c_double), ("per_entry", C.c_double * 10), ("num_per_entry", C.c_int32),
                ("mean_sample", C.c_double), ("eval_flops", C.c_int64), ("eval_seconds", C.c_double)]


class SkelStats(C.Structure):
    _fields_ = [("seconds", C.c_double), ("kernel_ms", C.c_double), ("bytes", C.c_double), ("flops", C.c_double)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GofmmError(GOFMM_ERR_CUDA, f"CUDA extension not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.gofmm_create.argtypes = [C.POINTER(TreeDesc), C.POINTER(Options), C.POINTER(P)]
        L.gofmm_evaluate.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, C.POINTER(EvalStats)]
        L.gofmm_evaluate_device.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P, C.c_int32,
                                            C.POINTER(EvalStats)]
        L.gofmm_unpermute_device.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P]
        L.gofmm_evaluate_f32.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, C.POINTER(EvalStats)]
        L.gofmm_evaluate_device_f32.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P, C.c_int32,
                                                C.POINTER(EvalStats)]
        L.gofmm_unpermute_device_f32.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P]
        L.gofmm_precision.argtypes = [P]
        L.gofmm_flops.argtypes = [P, C.c_int32]
        L.gofmm_flops.restype = C.c_int64
        L.gofmm_phase_flops.argtypes = [P, C.c_int32, P]
        L.gofmm_launch_profile.argtypes = [P, C.c_int32, C.c_int32, P, C.POINTER(C.c_int32)]
        L.gofmm_create_dist.argtypes = [C.POINTER(TreeDesc), C.POINTER(Options), C.c_int32, C.c_int32, C.POINTER(P)]
        L.gofmm_dist_get_info.argtypes = [P, C.POINTER(DistInfo)]
        L.gofmm_dist_plan_host.argtypes = [C.POINTER(TreeDesc), C.c_int32, C.c_int32, C.POINTER(DistInfo), C.c_int32, P]
        L.gofmm_dist_stage1.argtypes = [P, P, C.c_int64, C.c_int32, P, P]
        L.gofmm_dist_stage2.argtypes = [P, P, C.c_int32, P, C.c_int64, P]
        L.gofmm_dist_stage1_f32.argtypes = [P, P, C.c_int64, C.c_int32, P, P]
        L.gofmm_dist_stage2_f32.argtypes = [P, P, C.c_int32, P, C.c_int64, P]
        L.gofmm_exact_rows.argtypes = [P, P, C.c_int32, P, C.c_int64, C.c_int32, P, C.c_int64, P]
        L.gofmm_rng_eps2_draw.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, P, P, C.c_int64]
        L.gofmm_rng_eps2_draw_attempt.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P, P,
                                                  C.c_int64]
        L.gofmm_nccl_unique_id.argtypes = [P]
        L.gofmm_dist_init_comm.argtypes = [P, P]
        L.gofmm_dist_attach_comm.argtypes = [P, P]
        L.gofmm_dist_evaluate.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P, C.c_int32, P]
        L.gofmm_dist_evaluate_host.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P]
        L.gofmm_dist_evaluate_f32.argtypes = [P, P, C.c_int64, C.c_int32, P, C.c_int64, P, C.c_int32, P]
        L.gofmm_error_eps2.argtypes = [P, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(Eps2Report), P]
        L.gofmm_points_gaussian.argtypes = [C.c_int32, C.c_int32, C.c_uint64, P]
        L.gofmm_default_laplace_floor.argtypes = [C.c_int32, C.c_int32, P, C.c_uint64, P]
        L.gofmm_rng_gauss_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_int32, C.c_int32, P, C.c_int64]
        L.gofmm_device_bytes.argtypes = [P]
        L.gofmm_device_bytes.restype = C.c_int64
        L.gofmm_launches_per_eval.argtypes = [P]
        L.gofmm_destroy.argtypes = [P]
        L.gofmm_last_error.restype = C.c_char_p
        L.gofmm_skeletonize_batch.argtypes = [C.c_int32, P, P, P, P, C.c_int32, C.c_double, C.c_int32, P, P, P, P,
                                              C.POINTER(SkelStats)]
        L.gofmm_skeletonize_last_error.restype = C.c_char_p
        L.gofmm_ann_leaf_merge.argtypes = [C.c_int32, C.c_int32, P, C.c_int32, C.c_double, C.c_int32, C.c_int32,
                                           P, P, C.c_int32, P, P, P, C.POINTER(C.c_double)]
        L.gofmm_ann_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def check(rc: int):
    if rc != GOFMM_OK:
        msg = lib().gofmm_last_error().decode()
        if rc == GOFMM_ERR_INVALID:
            raise InvalidArgument(rc, msg)
        raise GofmmError(rc, msg)
