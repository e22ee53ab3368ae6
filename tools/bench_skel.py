"""Batched skeletonisation on one B200 vs the reference skeletonize_node on the
host cores: one c3-shaped level of interior nodes (2s+32 = 1056 sampled rows x 2s = 1024
candidates, Gaussian d=8, s=512, tau=1e-5). Prints one JSON line: GPU kernel time, nodes/s,
algorithmic GB/s against the HBM roofline (the kernel streams each trailing block three times per
pivot step), the CPU reference on a bounded sample of the same nodes, and the bitwise parity of
that sample."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1707_00164_b200 import skeletonize_batch  # noqa: E402


def gaussian_block(rng, rows, cols, d, h=1.0):
    xs = rng.standard_normal((rows, d))
    xc = rng.standard_normal((cols, d))
    d2 = ((xs[:, None, :] - xc[None, :, :]) ** 2).sum(-1)
    return np.exp(-d2 / (2 * h * h))


ap = argparse.ArgumentParser()
ap.add_argument("--nodes", type=int, default=1776)
ap.add_argument("--rows", type=int, default=1056)
ap.add_argument("--cols", type=int, default=1024)
ap.add_argument("--cpu-nodes", type=int, default=16)
a = ap.parse_args()
rng = np.random.default_rng(0)
uniq = [gaussian_block(rng, a.rows, a.cols, 8) for _ in range(8)]
blocks = [uniq[i % len(uniq)] for i in range(a.nodes)]
skeletonize_batch(blocks[:2], 512, 1e-5)  # warm (context, module load)
st = {}
t0 = time.perf_counter()
got = skeletonize_batch(blocks, 512, 1e-5, stats=st)
wall = time.perf_counter() - t0
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
gbs = st["bytes"] / (st["kernel_ms"] * 1e-3) / 1e9
line = {"what": "batched skeletonize_node (CPQR + ID), c3-shaped interior level", "nodes": a.nodes,
        "block": [a.rows, a.cols], "s": 512, "tau": 1e-5, "gpu_kernel_ms": round(st["kernel_ms"], 3),
        "gpu_call_s": round(wall, 3), "gpu_nodes_per_s": round(a.nodes / (st["kernel_ms"] * 1e-3), 1),
        "algorithmic_gbs": round(gbs, 1), "hbm_peak_gbs": peak,
        "hbm_frac": round(gbs / peak, 4) if peak else None,
        "householder_gflops": round(st["flops"] / (st["kernel_ms"] * 1e-3) / 1e9, 1)}
try:
    from oracle import refpy as R

    threads = os.cpu_count() or 1
    sample = blocks[:a.cpu_nodes]
    ref, sec = R.skeletonize_batch(sample, 512, 1e-5, threads=threads)
    same = all(g.rank == k and np.array_equal(g.skel, sk) and np.array_equal(g.proj, pj)
               for (k, sk, pj, _), g in zip(ref, got[:a.cpu_nodes]))
    line["cpu_reference"] = {"nodes": len(sample), "threads": threads, "seconds": round(sec, 3),
                             "nodes_per_s": round(len(sample) / sec, 2)}
    line["speedup_vs_cpu_nodes_per_s"] = round(line["gpu_nodes_per_s"] / (len(sample) / sec), 1)
    line["bitwise_equal_on_cpu_sample"] = bool(same)
except Exception as e:  # the oracle library may be absent
    line["cpu_reference"] = f"unavailable: {e}"
print(json.dumps(line))
