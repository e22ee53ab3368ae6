"""Latency probe for the small BASELINE configs (c1, c2): device time of one evaluation through
the CUDA-graph path (median of many, L2 flushed) and the per-launch CUDA-event times of a timed
(non-graph) evaluation, on the product-compress tree of the config's cloud.

  python tools/latency_probe.py c1 [--reps 50] [--tree compress|synth]   (GOFMM_NO_PDL=1: no PDL)
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1707_00164_b200 import Evaluator, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--tree", default="compress")
    ap.add_argument("--precision", default="fp64")
    a = ap.parse_args()
    cfg = dict(synth.CONFIGS[a.config])
    cfg["name"] = a.config
    tree, info = bench.workload_tree(cfg, cfg["n"], 0, a.tree)
    r = cfg["r"]
    ev = Evaluator(tree, precision=a.precision)
    dt = torch.float64 if a.precision == "fp64" else torch.float32
    w = torch.randn((r, tree.n), dtype=dt, device="cuda").t()
    u = torch.empty((r, tree.n), dtype=dt, device="cuda").t()
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")
    for _ in range(5):
        ev.evaluate_torch(w, out=u)
    st = torch.cuda.current_stream()
    ms = []
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ev.evaluate_torch(w, out=u)
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    flops = ev.flops(r)
    med = float(np.median(ms))
    out = {"config": a.config, "pdl": os.environ.get("GOFMM_NO_PDL", "0") != "1", "n": tree.n, "r": r, "tree": info.get("tree"), "flops": int(flops),
           "graph_ms_median": round(med, 4), "graph_ms_min": round(float(np.min(ms)), 4),
           "tflops": round(flops / med / 1e9, 3), "launches_per_eval": ev.launches_per_eval,
           "near_pairs": int(len(tree.near_a)), "far_pairs": int(len(tree.far_a)), "depth": int(tree.depth)}
    _, ph = ev.evaluate_torch(w, out=u, sync_stats=True)
    out["timed_phase_ms"] = {k: round(v, 4) for k, v in ph.items()}
    out["launches"] = [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in L.items()}
                       for L in ev.launch_profile(r)]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
