#!/usr/bin/env python
"""bench.py — GOFMM evaluation phase u = K~ W on B200 (BASELINE.json metric, config 3 by default).

One "step" = one evaluation of the c3 workload (N = 2^20 COVTYPE-shaped d=8 points, Gaussian h=1,
m = s = 512, budget 0.03, r = 512 RHS, FP64) over a synthetic compressed tree of that shape
(paper_1707_00164_b200/synth.py; the reference compress needs hours at 1M and has no HMatrix file
format). Inputs (W, 4.3 GB) exceed L2 (126 MB), so no extra flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]

Under torchrun (N > 1, N a power of two) the SAME config-3 evaluation is split across the ranks
(strong scaling): the tree is cut at level log2(N), rank g owns the g-th subtree, nodes above the
cut are evaluated redundantly, and one NCCL all-gather per evaluation exchanges the skeleton
weights and W rows other ranks need (north_star (4)). The timed region is bracketed
by a barrier + synchronize and the max over ranks is used.
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
NCU_SUMMARY_FILE = os.path.join(HERE, "profiles", "r01_ncu_summary.json")


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
def cpu_sample_tree(cfg: dict, n_sample: int, seed: int):
    """A bounded sample of the workload: a c3-shaped tree (same d, m, s, budget, kernel) on
    n_sample points, imported into the reference HMatrix through the reference oracle."""
    from paper_1707_00164_b200 import synth

    tree, _ = synth.make_config_tree(cfg["name"], seed=seed, n=n_sample, budget=cfg["budget"])
    return tree


def run_reference_sample(tree, r: int, reps: int, threads: int):
    """Time the reference's own evaluate() (oracle/_ref: reference headers, unmodified) on the host."""
    from oracle import refpy as R

    ref = R.import_flat(tree, threads=threads)
    w = np.asfortranarray(np.random.default_rng(1).standard_normal((tree.n, r)))
    times, flops, u = [], 0, None
    for _ in range(reps):
        u, flops, sec = ref.evaluate(w, mode=R.TASK_DAG, threads=threads)
        times.append(sec)
    return dict(ref=ref, w=w, u=u, flops=flops, times=times)


def reference_arm(args, world, rank):
    """--impl reference: the reference CPU evaluate on this box's host cores."""
    if rank != 0:
        return 0
    from paper_1707_00164_b200 import synth

    cfg = dict(synth.CONFIGS[args.config])
    cfg["name"] = args.config
    r = args.r or cfg["r"]
    threads = os.cpu_count() or 1
    tree = cpu_sample_tree(cfg, min(args.cpu_n, cfg["n"]), seed=args.seed)
    from oracle import refpy as R

    ref = R.import_flat(tree, threads=threads)
    w = np.asfortranarray(np.random.default_rng(1).standard_normal((tree.n, r)))
    for _ in range(args.warmup):
        ref.evaluate(w, mode=R.TASK_DAG, threads=threads)
    secs, flops = [], 0
    for _ in range(args.steps):
        _, flops, sec = ref.evaluate(w, mode=R.TASK_DAG, threads=threads)
        secs.append(sec)
    ms = 1e3 * float(np.mean(secs))
    val = flops / (ms * 1e-3) / 1e9
    sample = (f"{args.config}-shaped tree at N={tree.n} (same d/m/s/budget/kernel), r={r}; reference "
              f"gfmm::evaluate (TaskDag) per step, Potentials.seconds")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} sample N={tree.n} r={r}", "n": tree.n, "r": r, "cpu_threads": threads},
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


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
    t0 = time.perf_counter()
    tree, cfg = synth.make_config_tree(args.config, seed=args.seed,
                                       **{k: cfg[k] for k in ("n", "budget")})
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
                    and rec.get("precision", "fp64") == args.precision
                    and rec.get("level") == dom["level"] and rec.get("n") == tree.n and rec.get("r") == r):
                traffic = rec.get("dram_bytes")
    except Exception:
        pass

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

    # CPU baseline (reference evaluate on a bounded sample) + parity of the GPU on that sample
    cpu = None
    rel_err = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cfg_s = dict(cfg)
            cfg_s["name"] = args.config
            stree = cpu_sample_tree(cfg_s, min(args.cpu_n, tree.n), seed=args.seed)
            threads = os.cpu_count() or 1
            res = run_reference_sample(stree, r, reps=2, threads=threads)
            cpu_sec = float(np.median(res["times"]))
            cpu = {"value": round(res["flops"] / cpu_sec / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
                   "kind": "reference",
                   "sample": f"{args.config}-shaped tree at N={stree.n} (same d/m/s/budget/kernel), r={r}, "
                             f"reference gfmm::evaluate TaskDag x{threads} threads, median of 2 Potentials.seconds"}
            with Evaluator(stree, device=local, precision=args.precision) as es:
                pu = es.evaluate(res["w"])
            rel_err = float(np.linalg.norm(pu.u.astype(np.float64) - res["u"]) / np.linalg.norm(res["u"]))
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
                   "tree": "synthetic saturated-rank tree (synth.py)", "l2_flush": (f"L2 flushed between steps (256 MB write, outside the per-step events); W {tree.n * r * esz / 1e6:.1f} MB" if small else f"inputs larger than L2 (W {tree.n * r * esz / 1e9:.2f} GB)"),
                   "parallelism": "single GPU", "precision": args.precision,
                   "arithmetic": "3xTF32 on tcgen05 (FP32 accumulate in TMEM)" if f32 else "FP64 DMMA"},
        "sec_per_eval": round(ms / 1e3, 6),
        ("pct_3xtf32_peak" if f32 else "pct_fp64_peak"): round(100.0 * value / 1e3 / (peak * world), 2),
        "flops_per_eval": int(flops),
        "rel_error": rel_err,
        "phase_ms": {k: round(v[1], 3) for k, v in phases.items()} | {"permute": round(ph["ms_permute"], 3)},
        "roofline": {"bound": "tensor", "kernel": dom_name, "achieved": round(achieved, 3),
                     "peak": peak, "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "peak_source": peak_src, "launch_ms": round(dom["ms"], 3), "launch_flops": int(dom["flops"]),
                     "share_of_step": round(dom["ms"] / ms, 4)},
        "cpu_baseline": cpu,
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

    from paper_1707_00164_b200 import Evaluator, synth

    torch.cuda.set_device(local)
    cfg = dict(synth.CONFIGS[args.config])
    if args.budget is not None:
        cfg["budget"] = args.budget
    if args.n:
        cfg["n"] = args.n
    r = args.r or cfg["r"]
    t0 = time.perf_counter()
    tree, cfg = synth.make_config_tree(args.config, seed=args.seed, **{k: cfg[k] for k in ("n", "budget")})
    t_gen = time.perf_counter() - t0
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
    send = torch.empty(slot, dtype=tdt, device="cuda")
    recv = torch.empty(slot * world, dtype=tdt, device="cuda")

    def step():
        ev.dist_stage1_torch(w, send)
        if slot and world > 1:
            dist.all_gather_into_tensor(recv, send)
        ev.dist_stage2_torch(recv, r, u)

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
                   "n": tree.n, "r": r, "budget": cfg["budget"], "parallelism": f"subtree split x{world}",
                   "split_level": info["split_level"], "allgather_bytes_per_rank": int(slot * esz),
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
