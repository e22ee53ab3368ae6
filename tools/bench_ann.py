"""ANN leaf pass on one B200 vs the reference ann_iteration on the host cores.
c3-shaped: N points d=8 (standard normal), leaves of m=512 from the reference's random tree,
kappa=32, geometric metric (bit-identical; checked here on the whole table). Prints one JSON line:
GPU kernel ms, candidate pairs/s, FP64 rate of the distance work (3d+1 ops per pair) against the
measured DFMA peak, and the reference iteration (its leaf loop, same tree) with all host threads."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import refpy as R  # noqa: E402  (reference side + the host-built random tree)
from paper_1707_00164_b200 import ann_leaf_merge  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 18)
ap.add_argument("--d", type=int, default=8)
ap.add_argument("--m", type=int, default=512)
ap.add_argument("--kappa", type=int, default=32)
a = ap.parse_args()
coords = R.points_gaussian(a.n, a.d, 3)
k = a.kappa
t0 = time.perf_counter()
off, idx = R.ann_leaves(coords, 0, 1.0, a.m, 7)
t_tree = time.perf_counter() - t0
tj, td, tl = np.full((a.n, k), -1, np.int32), np.zeros((a.n, k)), np.zeros(a.n, np.int32)
ann_leaf_merge(coords, 0, 1.0, k, off, idx, tj.copy(), td.copy(), tl.copy())  # warm
ms = ann_leaf_merge(coords, 0, 1.0, k, off, idx, tj, td, tl)
# a second iteration (another random tree) on the now-full table: most candidates are pruned
off2, idx2 = R.ann_leaves(coords, 0, 1.0, a.m, 8)
tj2, td2, tl2 = tj.copy(), td.copy(), tl.copy()
ms2 = ann_leaf_merge(coords, 0, 1.0, k, off2, idx2, tj2, td2, tl2)
sizes = np.diff(off).astype(np.int64)
pairs = int((sizes * (sizes - 1)).sum())
threads = os.cpu_count() or 1
rj, rd, rl = np.full((a.n, k), -1, np.int32), np.zeros((a.n, k)), np.zeros(a.n, np.int32)
sec = R.ann_iteration(coords, 0, 1.0, k, a.m, 7, rj, rd, rl, threads=threads)
same = bool(np.array_equal(rj, tj) and np.array_equal(rd, td) and np.array_equal(rl, tl))
sec2 = R.ann_iteration(coords, 0, 1.0, k, a.m, 8, rj, rd, rl, threads=threads)
same2 = bool(np.array_equal(rj, tj2) and np.array_equal(rd, td2) and np.array_equal(rl, tl2))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                   "r01_fp64_peak.json")))["dfma_b8_t256_tflops"]
gflops = pairs * (3 * a.d + 1) / (ms * 1e-3) / 1e9
print(json.dumps({"what": "ANN leaf pass (all-pairs in leaves + kappa merge), geometric metric",
                  "n": a.n, "d": a.d, "m": a.m, "kappa": k, "leaves": int(len(sizes)), "pairs": pairs,
                  "gpu_kernel_ms": round(ms, 3), "gpu_pairs_per_s": round(pairs / (ms * 1e-3), 1),
                  "fp64_gflops_distance_work": round(gflops, 1), "dfma_peak_tflops": peak,
                  "fp64_frac": round(gflops / 1e3 / peak, 4),
                  "cpu_reference": {"seconds": round(sec, 3), "threads": threads,
                                    "note": "ann_iteration incl. its own random-tree build"},
                  "host_tree_build_s": round(t_tree, 3), "speedup_vs_cpu_iteration": round(sec / (ms * 1e-3), 1),
                  "bitwise_equal_table": same,
                  "second_iteration": {"gpu_kernel_ms": round(ms2, 3), "cpu_reference_s": round(sec2, 3),
                                       "bitwise_equal_table": same2}}))
