#!/usr/bin/env python
"""bench.py — GOFMM evaluation phase u = K~ W on B200 (BASELINE.json metric, config 3 by default).

One "step" = one evaluation of the c3 workload (N = 2^20 COVTYPE-shaped d=8 points, Gaussian h=1,
m = s = 512, budget 0.03, r = 512 RHS, FP64) over the compressed tree the product compress
(gofmm_compress: the reference compress algorithm, GPU entries) builds from that cloud before the
timed region (~45 s at 1M; --tree synth: synth.py's saturated-rank tree). Inputs (W, 4.3 GB) exceed
L2 (126 MB), so no extra flush is needed between steps. The CPU legs (reference arm, cpu_baseline,
same-config GPU leg) share one bounded sample: the reference compress() of the config's cloud at
N = 2^16.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

Under torchrun (N > 1, N a power of two) the SAME config-3 evaluation is split across the ranks
(strong scaling): the tree is cut at level log2(N) (+ up to 3 for balance), each rank owns a
contiguous run of subtrees, nodes above the cut are evaluated redundantly, and one NCCL all-gather
per evaluation — issued by the library itself (gofmm_dist_evaluate) on an NCCL communicator it
creates from a broadcast unique id — exchanges the skeleton weights other ranks need (W is
replicated), overlapped with the own leaves' D + near output terms (north_star (4)).
The timed region is bracketed by a barrier + synchronize and the max over ranks is used.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

FP64_PEAK_FILE = os.path.join(HERE, "profiles", "r01_fp64_peak.json")
NCU_SUMMARY_FILE = os.path.join(HERE, "profiles", "r02_ncu_summary.json")


def tf32x3_peak_tflops() -> tuple[float, str]:
    """Peak for the FP32 path: 3xTF32 issues three TF32 tensor-core MMAs per algorithmic product,
    so the algorithmic ceiling is the dense TF32 peak / 3. Dense TF32 = half the dense bf16 rate:
    from MEASURED_PEAKS.json (driver-written cuBLAS bf16) when present, else the 1.1 PF/s nominal of
    /opt/skills/guides/B200_PROFILING.md."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        for k, v in d.items():
            if "bf16" in k.lower() and isinstance(v, (int, float)) and v > 100:
                tf = float(v) / 2.0  # TF/s
                return tf / 3.0, f"MEASURED_PEAKS.json {k}={v} -> tf32 dense {tf:.0f} TF/s, / 3 (3xTF32)"
    except Exception:
        pass
    return 1100.0 / 3.0, "nominal tf32 dense 1.1 PF/s (B200_PROFILING.md) / 3 (3xTF32)"


FP32_SIMT_PEAK = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4 TF/s: FFMA peak, for context


def fp64_peak_tflops() -> tuple[float, str]:
    """Measured FP64 DMMA peak of this pool's B200 (MEASURED_PEAKS.json has no FP64 entry)."""
    try:
        with open(FP64_PEAK_FILE) as f:
            d = json.load(f)
        return float(d["mma16816_sustained_tflops"]), "measured: profiles/r01_fp64_peak.json (DMMA sustained)"
    except Exception:
        return 37.2, "nominal 148 SM x 64 FMA x 2 x 1.965 GHz (no measurement found)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL's init lines (rank count, NVLink / NVLS transport) on stderr for the run log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allmax(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ CPU reference (oracle) legs
def host_info() -> dict:
    """The host the CPU legs run on: lscpu model, usable cores, memory (free -g)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                info["cpu_model"] = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            mem = {ln.split(":")[0]: int(ln.split()[1]) for ln in f if ln.split()}
        info["mem_total_gb"] = round(mem["MemTotal"] / 2 ** 20, 1)
        info["mem_available_gb"] = round(mem["MemAvailable"] / 2 ** 20, 1)
    except Exception:
        pass
    return info


def config_cloud(cfg: dict, n: int, seed: int) -> np.ndarray:
    """The config's synthetic point cloud (d x n): uniform [0,1]^d (c1), standard normal (c2, c4,
    c5), COVTYPE-shaped Gaussian mixture (c3) — synth.py."""
    from paper_1707_00164_b200 import synth

    fn = {"uniform": synth.uniform_cloud, "gaussian": synth.gaussian_cloud, "covtype": synth.covtype_like}[cfg["cloud"]]
    return fn(n, cfg["d"], seed)


def workload_tree(cfg: dict, n: int, seed: int, source: str):
    """The timed tree. "compress": the product compress (gofmm_compress: the reference's compress
    algorithm with ANN passes, sampled blocks and CPQR on the GPU) of the config's cloud with the
    config's kernel / m / s / budget and the reference RunConfig defaults otherwise (tau 1e-5,
    kappa 32, kernel distance, 10 ANN iterations); "synth": synth.py's saturated-rank tree."""
    from paper_1707_00164_b200 import compress, synth

    if source == "synth":
        tree, _ = synth.make_config_tree(cfg["name"], seed=seed, n=n, budget=cfg["budget"])
        return tree, {"tree": "synthetic saturated-rank tree (synth.py)"}
    pc = config_cloud(cfg, n, seed)
    res = compress(pc, cfg["kernel"], (cfg["h"], 0.0), m=cfg["m"], s=cfg["s"], budget=cfg["budget"], tau=1e-5,
                   kappa=32, distance="kernel", seed=seed, threads=os.cpu_count() or 1, entries="device")
    st = res.stats
    info = {"tree": "product compress (gofmm_compress, GPU entries) of the config's cloud",
            "compress": {"seconds": round(st["compress_seconds"], 2), "mean_rank": round(st["mean_skeleton"], 1),
                         "max_rank": st["max_skeleton"], "entries_evaluated": st["entries_evaluated"],
                         "ann_recall_last": round(st["ann_recall"][-1], 4) if st["ann_recall"] else None}}
    return res.tree, info


def cpu_sample_tree(cfg: dict, n_sample: int, seed: int):
    """A bounded sample of the workload for the CPU legs: the REFERENCE compress() (oracle/_ref) of
    the config's cloud at n_sample points (same d, kernel, m, s, budget, RunConfig defaults) — the
    SAME HMatrix for the reference arm, the cpu_baseline leg and the GPU's same-config leg.
    Returns (reference HMatrix, its flattened tree)."""
    from oracle import refpy as R
    from paper_1707_00164_b200 import CompressedTree

    pc = config_cloud(cfg, n_sample, seed)
    h = R.compress_kernel(cfg["kernel"], pc, cfg["h"], 0.0, m=cfg["m"], s=cfg["s"], tau=1e-5, kappa=32,
                          budget=cfg["budget"], seed=seed, threads=os.cpu_count() or 1)
    return h, CompressedTree.from_any(h.export(blocks=False))


def sample_rhs(n: int, r: int) -> np.ndarray:
    return np.asfortranarray(np.random.default_rng(1).standard_normal((n, r)))


def cpu_protocol(ref, w: np.ndarray, threads: int, reps: int, warmup: int) -> dict:
    """THE CPU timing protocol of both CPU legs (reference arm and cpu_baseline): the reference
    gfmm::evaluate (oracle/_ref, unmodified headers) in both executors — TaskDag (EvalOptions'
    default, evaluate.hpp:122-126) and LevelByLevel (evaluate.hpp:222-235) — `warmup` untimed
    runs each, then the median of `reps` Potentials.seconds per mode. value = TaskDag."""
    from oracle import refpy as R

    out, flops, u = {}, 0, None
    for name, mode in (("task_dag", R.TASK_DAG), ("level_by_level", R.LEVEL_BY_LEVEL)):
        for _ in range(warmup):
            ref.evaluate(w, mode=mode, threads=threads)
        secs = []
        for _ in range(reps):
            u, flops, sec = ref.evaluate(w, mode=mode, threads=threads)
            secs.append(sec)
        out[name] = {"median_s": float(np.median(secs)), "runs_s": [round(x, 4) for x in secs]}
    out["flops"] = int(flops)
    out["u"] = u
    return out


def reference_arm(args, world, rank):
    """--impl reference: the reference CPU evaluate on this box's host cores (cpu_protocol with
    reps = --steps, warmup = --warmup, on the bounded c3-shaped sample)."""
    if rank != 0:
        return 0
    from paper_1707_00164_b200 import synth

    cfg = dict(synth.CONFIGS[args.config])
    cfg["name"] = args.config
    r = args.r or cfg["r"]
    threads = os.cpu_count() or 1
    ref, tree = cpu_sample_tree(cfg, min(args.cpu_n, cfg["n"]), seed=args.seed)
    w = sample_rhs(tree.n, r)
    res = cpu_protocol(ref, w, threads, reps=max(args.steps, 3), warmup=max(args.warmup, 1))
    sec = res["task_dag"]["median_s"]
    val = res["flops"] / sec / 1e9
    sample = (f"{args.config} cloud at N={tree.n} compressed by the reference compress() (same d/kernel/m/s/"
              f"budget, seed {args.seed}), r={r}; reference gfmm::evaluate, TaskDag x{threads} threads, median of "
              f"{max(args.steps, 3)} Potentials.seconds after {max(args.warmup, 1)} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sec, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} sample N={tree.n} r={r}", "n": tree.n, "r": r, "cpu_threads": threads},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": sample,
                         "level_by_level_gflops": round(res["flops"] / res["level_by_level"]["median_s"] / 1e9, 3),
                         "runs_s": res["task_dag"]["runs_s"], "host": host_info()},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def same_config_leg(ev_cls, tree, w: np.ndarray, precision: str, local: int, reps: int = 5) -> dict:
    """The GPU on exactly the reference arm's tree and W: device-resident (CUDA events, median of
    `reps` after a warm-up, L2 flushed before each) and end to end through the host API
    (gofmm_evaluate with pinned host buffers, median of >= `reps` wall times)."""
    import torch

    tdt = torch.float32 if precision == "fp32" else torch.float64
    ndt = np.float32 if precision == "fp32" else np.float64
    with ev_cls(tree, device=local, precision=precision) as es:
        flops = es.flops(w.shape[1])
        wd = torch.from_numpy(np.ascontiguousarray(w.T.astype(ndt))).cuda().t()
        ud = torch.empty_like(wd.t()).t()
        flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")
        es.evaluate_torch(wd, out=ud)
        st = torch.cuda.current_stream()
        ms = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            es.evaluate_torch(wd, out=ud)
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        wh = torch.empty((w.shape[1], w.shape[0]), dtype=tdt, pin_memory=True)
        wh.copy_(torch.from_numpy(np.ascontiguousarray(w.T.astype(ndt))))
        uh = torch.empty_like(wh).pin_memory()
        wn, un = wh.numpy().T, uh.numpy().T
        es.evaluate(wn, out=un)
        ts = []
        t0 = time.perf_counter()
        # at least `reps`, and up to 50 within ~2 s: a sub-ms evaluation's wall-time median must not
        # hang on a few host hiccups (the CPU leg's worker threads winding down just before)
        while len(ts) < reps or (len(ts) < 50 and time.perf_counter() - t0 < 2.0):
            t1 = time.perf_counter()
            p = es.evaluate(wn, out=un)
            ts.append(time.perf_counter() - t1)
        u = un.astype(np.float64)
    dev_s, e2e_s = float(np.median(ms)) / 1e3, float(np.median(ts))
    return {"flops": int(flops), "device_s": dev_s, "e2e_s": e2e_s, "u": u,
            "device_gflops": flops / dev_s / 1e9, "e2e_gflops": flops / e2e_s / 1e9}


KERNEL_NAMES = {0: "Gaussian", 1: "Laplace", 2: "Polynomial", 4: "Exponential (Matern-1/2)"}
METRIC = "evaluate GFLOPS & % of FP64 peak (N=1M, r=512); sec per K~W; rel. error"


def ours_arm(args, world, rank, local):
    import torch

    from paper_1707_00164_b200 import Evaluator, synth

    torch.cuda.set_device(local)
    cfg = dict(synth.CONFIGS[args.config])
    if args.budget is not None:
        cfg["budget"] = args.budget
    if args.n:
        cfg["n"] = args.n
    r = args.r or cfg["r"]
    cfg["name"] = args.config
    t0 = time.perf_counter()
    tree, tree_info = workload_tree(cfg, cfg["n"], args.seed, args.tree)
    t_gen = time.perf_counter() - t0
    f32 = args.precision == "fp32"
    tdt = torch.float32 if f32 else torch.float64
    esz = 4 if f32 else 8
    t0 = time.perf_counter()
    ev = Evaluator(tree, device=local, precision=args.precision)
    t_create = time.perf_counter() - t0
    flops = ev.flops(r)
    pflops = ev.phase_flops(r)

    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    w = torch.randn((r, tree.n), dtype=tdt, device="cuda", generator=gen).t()  # N x r column-major
    u = torch.empty((r, tree.n), dtype=tdt, device="cuda").t()
    for _ in range(args.warmup):
        ev.evaluate_torch(w, out=u)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    # inputs smaller than 2x L2 (126 MB): flush L2 between steps (outside the per-step events)
    small = tree.n * r * esz < 2 * 126 * 2 ** 20
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda") if small else None
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        if small:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush.zero_()
                a.record(stream)
                ev.evaluate_torch(w, out=u)
                b.record(stream)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                ev.evaluate_torch(w, out=u)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
        barrier(world)
    ms = allmax(ms, world)
    value = world * flops / (ms * 1e-3) / 1e9  # whole-job GFLOP/s

    # per-phase and per-launch device times of one more evaluation (CUDA events on the stream the
    # kernels are launched on); the roofline reports the longest single launch
    _, ph = ev.evaluate_torch(w, out=u, sync_stats=True)
    torch.cuda.synchronize()
    peak, peak_src = tf32x3_peak_tflops() if f32 else fp64_peak_tflops()
    phases = {"upward": (pflops["upward"], ph["ms_upward"]), "downward": (pflops["downward"], ph["ms_downward"]),
              "output": (pflops["output"], ph["ms_output"])}
    launches = ev.launch_profile(r)
    dom = max(launches, key=lambda x: x["ms"])
    achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12 if dom["ms"] > 0 else 0.0
    kname = "grouped_gemm_tf32x3" if f32 else "grouped_gemm_f64"
    dom_name = f"{kname} {dom['phase']} launch (level {dom['level']})" if dom["level"] >= 0 else \
        f"{kname} output launch (L2L + leaf S2N)"
    traffic = None
    try:
        with open(NCU_SUMMARY_FILE) as f:
            nsum = json.load(f)
        for rec in nsum.get("launches", []):
            if (rec.get("config") == args.config and rec.get("phase") == dom["phase"]
                    and rec.get("precision", "fp64") == args.precision and rec.get("tree", "synth") == args.tree
                    and rec.get("level") == dom["level"] and rec.get("n") == tree.n and rec.get("r") == r):
                traffic = rec.get("dram_bytes")
    except Exception:
        pass

    # algorithmic bytes of the dominant launch (each operand once): output launch = W_perm read +
    # u written + the leaves' c and proj read; a downward / upward launch = its level's B rows
    # (what / c / W_perm) and outputs plus the proj it reads — leaf-level figures from the tree
    alg_bytes = None
    if dom["phase"] == "output":
        lv = np.flatnonzero(np.asarray(tree.left) < 0)
        rk = np.maximum(np.asarray(tree.rank)[lv], 0).astype(np.int64)
        cnt = (np.asarray(tree.end) - np.asarray(tree.start))[lv].astype(np.int64)
        alg_bytes = int(esz * (2 * tree.n * r + int(rk.sum()) * r + int((rk * cnt).sum())))

    # the BASELINE metric's "rel. error" on the timed tree itself: the reference's error_eps2
    # (evaluate.hpp:330-373; r = 1, 100 sampled rows, the reference Rng draws) computed by the
    # product — GPU evaluation + matrix-free exact rows on the GPU
    eps2 = None
    if not f32:
        eps2 = ev.error_eps2(1, 100, args.seed)["eps2"]

    # end-to-end through the host API (pinned host W and u; H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        w_h = torch.empty((r, tree.n), dtype=tdt, pin_memory=True)
        w_h.copy_(w.t())
        # the host-API leg owns the HBM a user's call would have: drop the device-resident W / u
        del w, u, flush
        torch.cuda.empty_cache()
        u_h = torch.empty((r, tree.n), dtype=tdt, pin_memory=True)
        wn, un = w_h.numpy().T, u_h.numpy().T  # Fortran-ordered N x r views of pinned memory
        ev.evaluate(wn, out=un)  # warm
        barrier(world)
        ts = []
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            p = ev.evaluate(wn, out=un)
            ts.append(time.perf_counter() - t1)
        barrier(world)
        sec = allmax(float(np.mean(ts)), world)
        e2e = {"value": round(world * flops / sec / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(tree.n * r * esz), "d2h_bytes_per_step": int(tree.n * r * esz),
               "sec_per_eval": round(sec, 5), "ms_h2d": round(p.stats["ms_h2d"], 3),
               "ms_d2h": round(p.stats["ms_d2h"], 3)}
        del w_h, u_h

    # CPU baseline (reference evaluate on a bounded sample, the reference arm's protocol) + the GPU
    # on exactly that tree and W (same-config ratio) + parity of the GPU on that tree
    cpu, same, rel_err, timed_parity = None, None, None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import refpy as R

            ref, stree = cpu_sample_tree(cfg, min(args.cpu_n, tree.n), seed=args.seed)
            threads = os.cpu_count() or 1
            ws = sample_rhs(stree.n, r)
            res = cpu_protocol(ref, ws, threads, reps=3, warmup=1)
            del ref
            cpu_sec = res["task_dag"]["median_s"]
            cpu_val = res["flops"] / cpu_sec / 1e9
            cpu = {"value": round(cpu_val, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                   "sample": f"{args.config} cloud at N={stree.n} compressed by the reference compress() (same "
                             f"d/kernel/m/s/budget, seed {args.seed}), r={r}; reference gfmm::evaluate, TaskDag "
                             f"x{threads} threads, median of 3 Potentials.seconds after 1 warm-up (the reference "
                             f"arm's protocol)",
                   "level_by_level_gflops": round(res["flops"] / res["level_by_level"]["median_s"] / 1e9, 3),
                   "runs_s": res["task_dag"]["runs_s"], "host": host_info()}
            sc = same_config_leg(Evaluator, stree, ws, args.precision, local)
            rel_err = float(np.linalg.norm(sc["u"] - res["u"]) / np.linalg.norm(res["u"]))
            same = {"tree": cpu["sample"].split(";")[0], "r": r, "flops": sc["flops"],
                    "gpu_device_gflops": round(sc["device_gflops"], 3), "gpu_e2e_gflops": round(sc["e2e_gflops"], 3),
                    "reference_gflops": round(cpu_val, 3),
                    "ratio_device": round(sc["device_gflops"] / cpu_val, 2),
                    "ratio_e2e": round(sc["e2e_gflops"] / cpu_val, 2),
                    "rel_error_vs_reference": rel_err,
                    "note": "GPU timed on the reference arm's exact tree and W (device: CUDA events, L2 flushed, "
                            "median of 5; e2e: gofmm_evaluate with pinned host buffers, median of >= 5 (up to 50 within 2 s))"}
            # parity ON THE TIMED TREE: the GPU's u rows of 8 sampled leaves vs the reference evaluate on
            # restrict_to_leaves(tree, leaves) (bit-identical to those rows of the full reference
            # evaluation, whose stored blocks would not fit host RAM; tests/_util.py)
            if not f32:
                from tests._util import pick_leaves, reference_rows_check

                wt = np.asfortranarray(np.random.default_rng(7).standard_normal((tree.n, r)))
                ut = ev.evaluate(wt).u
                leaves = pick_leaves(tree, 8, 0)
                chk = reference_rows_check(R, tree, wt, ut, leaves, threads, cols=min(r, 512))
                del wt, ut
                timed_parity = {k: chk[k] for k in ("rel_error", "leaves", "rows", "cols", "near_kept", "far_kept")}
        except Exception as exc:  # report, never hide
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {exc!r}"[:300]}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {KERNEL_NAMES.get(cfg['kernel'], 'kernel')} h={cfg['h']} N={tree.n} "
                               f"d={cfg['d']} m={cfg['m']} "
                               f"s={cfg['s']} budget={cfg['budget']} r={r} per GPU", "n": tree.n, "d": cfg["d"],
                   "m": cfg["m"], "s": cfg["s"], "budget": cfg["budget"], "r_per_gpu": r,
                   "near_pairs": int(len(tree.near_a)), "far_pairs": int(len(tree.far_a)),
                   **tree_info, "l2_flush": (f"L2 flushed between steps (256 MB write, outside the per-step events); W {tree.n * r * esz / 1e6:.1f} MB" if small else f"inputs larger than L2 (W {tree.n * r * esz / 1e9:.2f} GB)"),
                   "parallelism": "single GPU", "precision": args.precision,
                   "arithmetic": "3xTF32 on tcgen05 (FP32 accumulate in TMEM)" if f32 else "FP64 DMMA"},
        "sec_per_eval": round(ms / 1e3, 6),
        ("pct_3xtf32_peak" if f32 else "pct_fp64_peak"): round(100.0 * value / 1e3 / (peak * world), 2),
        "flops_per_eval": int(flops),
        "rel_error": (timed_parity or {}).get("rel_error", rel_err),
        "rel_error_tree": ("the timed tree: GPU u rows of 8 sampled leaves vs the reference evaluate on the "
                           "leaf-restricted HMatrix (bit-identical to the full reference's rows)") if timed_parity
        else (same or {}).get("tree"),
        "timed_tree_parity": timed_parity,
        "eps2_timed_tree": eps2,
        "phase_ms": {k: round(v[1], 3) for k, v in phases.items()} | {"permute": round(ph["ms_permute"], 3)},
        "roofline": {"bound": "tensor", "kernel": dom_name, "achieved": round(achieved, 3),
                     "algorithmic_bytes": alg_bytes,
                     "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_src, "launch_ms": round(dom["ms"], 3), "launch_flops": int(dom["flops"]),
                     "share_of_step": round(dom["ms"] / ms, 4)},
        "cpu_baseline": cpu,
        "same_config": same,
        "e2e": e2e,
        "gpu_launches": int(ev.launches_per_eval * args.steps),
        "setup_s": {"tree_gen": round(t_gen, 2), "create_upload": round(t_create, 2)},
    }
    if f32:
        line["pct_fp32_simt_peak"] = round(100.0 * value / 1e3 / (FP32_SIMT_PEAK * world), 2)
        line["tolerance"] = "rel. 2-norm 1e-5 vs the reference FP64 evaluate (north_star, fp32)"
    if rank == 0:
        line["clocks"] = clk.summary()
        print(json.dumps(line), flush=True)
    ev.close()
    return 0


def dist_arm(args, world, rank, local):
    """Subtree-split evaluation of one config over `world` GPUs (strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_1707_00164_b200 import Evaluator, gofmm, synth

    torch.cuda.set_device(local)
    cfg = dict(synth.CONFIGS[args.config])
    if args.budget is not None:
        cfg["budget"] = args.budget
    if args.n:
        cfg["n"] = args.n
    r = args.r or cfg["r"]
    cfg["name"] = args.config
    t0 = time.perf_counter()
    tree, tree_info = workload_tree(cfg, cfg["n"], args.seed, args.tree)
    t_gen = time.perf_counter() - t0
    if world > 1:  # every rank compressed the same cloud; the GPU compress is deterministic — check
        import hashlib

        hsh = hashlib.sha256()
        for f in ("iperm", "rank", "skel_idx", "proj", "near_a", "near_b", "far_a", "far_b"):
            hsh.update(np.ascontiguousarray(getattr(tree, f)).tobytes())
        digests = [None] * world
        dist.all_gather_object(digests, hsh.hexdigest())
        if len(set(digests)) != 1:
            raise RuntimeError(f"ranks built different trees: {digests}")
    t0 = time.perf_counter()
    f32 = args.precision == "fp32"
    tdt = torch.float32 if f32 else torch.float64
    esz = 4 if f32 else 8
    ev = Evaluator(tree, device=local, rank=rank, nranks=world, precision=args.precision)
    t_create = time.perf_counter() - t0
    info = ev.dist_info()
    full_flops = info["full_flops_per_rhs"] * r
    gen = torch.Generator(device="cuda").manual_seed(1000)  # every rank holds the same W
    w = torch.randn((r, tree.n), dtype=tdt, device="cuda", generator=gen).t()
    u = torch.zeros((r, tree.n), dtype=tdt, device="cuda").t()
    slot = ev.send_elems(r)
    if world > 1:
        # the library's own data plane: an NCCL communicator created from a unique id that rank 0
        # draws and torch.distributed broadcasts; one ncclAllGather per evaluation inside
        # gofmm_dist_evaluate, overlapped with the own leaves' D + near output terms
        uid = [gofmm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ev.init_comm(uid[0])

    def step():
        ev.dist_evaluate_torch(w, u)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = allmax(e0.elapsed_time(e1) / args.steps, world)
    value = full_flops / (ms * 1e-3) / 1e9
    peak, peak_src = tf32x3_peak_tflops() if f32 else fp64_peak_tflops()
    # one more evaluation with the library's event timing: stage 1 and the all-gather (on its own
    # stream, overlapping the own D + near output terms), max over ranks
    barrier(world)
    tm = ev.dist_evaluate_torch(w, u, timed=True)
    exchange = {k: round(allmax(v, world), 3) for k, v in tm.items()}

    # zero-communication baseline: the whole tree replicated on every GPU, each
    # evaluating r / N of the columns (evaluation is column-separable)
    rhs_shard = None
    if world > 1 or args.rhs_shard:
        rl = max(1, r // world)
        ev1 = Evaluator(tree, device=local, precision=args.precision)
        w1, u1 = w[:, :rl], torch.empty((rl, tree.n), dtype=tdt, device="cuda").t()
        ev1.evaluate_torch(w1, out=u1)
        torch.cuda.synchronize()
        barrier(world)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            ev1.evaluate_torch(w1, out=u1)
        f1.record(stream)
        torch.cuda.synchronize()
        ms1 = allmax(f0.elapsed_time(f1) / args.steps, world)
        rhs_shard = {"value": round(world * ev1.flops(rl) / (ms1 * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
                     "ms_per_step": round(ms1, 3), "r_per_gpu": rl,
                     "note": "zero-communication baseline: replicated tree, r/N columns per GPU"}
        ev1.close()
        del w1, u1

    # end to end: pinned host W -> device, evaluation, own rows of u -> pinned host
    e2e = None
    if not args.no_e2e:
        w_h = torch.empty((r, tree.n), dtype=tdt, pin_memory=True)
        w_h.copy_(w.t())
        own = slice(int(info["own_row_begin"]), int(info["own_row_end"]))
        u_h = torch.empty((r, own.stop - own.start), dtype=tdt, pin_memory=True)
        ts = []
        for it in range(args.e2e_steps + 1):
            barrier(world)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            w.t().copy_(w_h, non_blocking=True)
            step()
            u_h.copy_(u.t()[:, own], non_blocking=True)
            torch.cuda.synchronize()
            if it:
                ts.append(time.perf_counter() - t1)
        sec = allmax(float(np.mean(ts)), world)
        e2e = {"value": round(full_flops / sec / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": int(tree.n * r * esz), "d2h_bytes_per_step": int((own.stop - own.start) * r * esz),
               "sec_per_eval": round(sec, 5), "note": "per rank: full W in, own rows of u out"}
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if f32 else "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {KERNEL_NAMES.get(cfg['kernel'], 'kernel')} h={cfg['h']} N={tree.n} "
                               f"d={cfg['d']} m={cfg['m']} s={cfg['s']} budget={cfg['budget']} r={r} total",
                   "n": tree.n, "r": r, "budget": cfg["budget"], "parallelism": f"subtree split x{world}", **tree_info,
                   "split_level": info["split_level"], "allgather_bytes_per_rank": int(slot * esz),
                   "exchange": "in-library ncclAllGather (gofmm_dist_evaluate), W replicated, what only",
                   "l2_flush": f"inputs larger than L2 (W {tree.n * r * esz / 1e9:.2f} GB)",
                   "precision": args.precision},
        "sec_per_eval": round(ms / 1e3, 6),
        ("pct_3xtf32_peak" if f32 else "pct_fp64_peak"): round(100.0 * value / 1e3 / (peak * world), 2),
        "flops_per_eval": int(full_flops),
        "rank_flops_max": int(allmax(float(info["flops_per_rhs"] * r), world)),
        "rel_error": None,
        # whole rank step (the distributed stages do not time single launches): the busiest
        # rank's reference-counted flops over the step time, against one GPU's peak
        "roofline": {"bound": "tensor", "kernel": "whole subtree-split step (busiest rank)",
                     "achieved": round(allmax(float(info["flops_per_rhs"] * r), world) / (ms * 1e-3) / 1e12, 3),
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": round(allmax(float(info["flops_per_rhs"] * r), world) / (ms * 1e-3) / 1e12 / peak, 4),
                     "traffic": None, "peak_source": peak_src},
        "cpu_baseline": None,
        "rhs_shard_baseline": rhs_shard,
        "exchange_ms": exchange,
        "e2e": e2e,
        "gpu_launches": int((ev.launches_per_eval + 2) * args.steps),
        "setup_s": {"tree_gen": round(t_gen, 2), "create_upload": round(t_create, 2)},
    }
    if rank == 0:
        line["clocks"] = clk.summary()
        print(json.dumps(line), flush=True)
    ev.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--budget", type=float, default=None)
    ap.add_argument("--tree", default="compress", choices=["compress", "synth"],
                    help="timed tree: the product compress of the config's cloud (default) or synth.py's")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--r", type=int, default=None)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-n", type=int, default=1 << 16)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true", help="use the subtree-split path even on one GPU")
    ap.add_argument("--rhs-shard", action="store_true",
                    help="also time the zero-communication RHS-sharding baseline on one GPU (always on for N > 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        rc = reference_arm(args, world, rank)
    elif world > 1 or args.dist:
        rc = dist_arm(args, world, rank, local)
    else:
        rc = ours_arm(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
