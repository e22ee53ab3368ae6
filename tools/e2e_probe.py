"""Host-API (gofmm_evaluate) latency probe: wall time per call vs the C-level seconds and the
device phase times, to locate fixed per-call overhead."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1707_00164_b200 import Evaluator, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # > 0: the product compress of the config's cloud at n
if n:
    import bench

    c = dict(synth.CONFIGS[cfg], name=cfg)
    tree, _ = bench.workload_tree(c, n, 0, "compress")
else:
    tree, c = synth.make_config_tree(cfg)
r = c["r"]
dt = torch.float64 if prec == "fp64" else torch.float32
with Evaluator(tree, precision=prec) as ev:
    wh = torch.randn((r, tree.n), dtype=dt).pin_memory()
    uh = torch.empty((r, tree.n), dtype=dt).pin_memory()
    wn, un = wh.numpy().T, uh.numpy().T
    for i in range(6):
        t0 = time.perf_counter()
        p = ev.evaluate(wn, out=un)
        t1 = time.perf_counter()
        st = p.stats
        print(f"{cfg} {prec} call {i}: wall {1e3 * (t1 - t0):8.2f} ms  C {1e3 * st['seconds']:8.2f} ms  h2d {st['ms_h2d']:7.2f}"
              f"  d2h {st['ms_d2h']:7.2f}  dev {st['ms_permute'] + st['ms_upward'] + st['ms_downward'] + st['ms_output']:8.2f}"
              f"  [perm {st['ms_permute']:.1f} up {st['ms_upward']:.1f} down {st['ms_downward']:.1f} out {st['ms_output']:.1f}]")
