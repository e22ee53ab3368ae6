"""Profiling driver: a c3-shaped workload (default N=2^18, same d/m/s/budget/r) evaluated twice,
for `ncu` captures of the grouped GEMM launches (see profiles/README.md for the commands)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1707_00164_b200 import Evaluator, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--n", type=int, default=1 << 18)
ap.add_argument("--budget", type=float, default=None)
ap.add_argument("--evals", type=int, default=2)
ap.add_argument("--far-mode", type=int, default=0)
ap.add_argument("--near-mode", type=int, default=0)
ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
ap.add_argument("--tree", default="synth", choices=["synth", "compress"])
a = ap.parse_args()
over = {"n": a.n}
if a.budget is not None:
    over["budget"] = a.budget
if a.tree == "compress":  # the product compress of the config's cloud (bench.py's timed tree)
    import bench

    cfg = dict(synth.CONFIGS[a.config], name=a.config, **over)
    tree, _ = bench.workload_tree(cfg, cfg["n"], 0, "compress")
else:
    tree, cfg = synth.make_config_tree(a.config, **over)
ev = Evaluator(tree, near_mode=a.near_mode, far_mode=a.far_mode, precision=a.precision)
r = cfg["r"]
dt = torch.float64 if a.precision == "fp64" else torch.float32
w = torch.randn((r, tree.n), dtype=dt, device="cuda").t()
u = torch.empty((r, tree.n), dtype=dt, device="cuda").t()
for i in range(a.evals):
    _, st = ev.evaluate_torch(w, out=u, sync_stats=True)
    print(i, {k: round(v, 3) for k, v in st.items()}, ev.phase_flops(r), flush=True)
print("launches/eval", ev.launches_per_eval, "depth", tree.depth)
for L in ev.launch_profile(r):
    tf = L["flops"] / (L["ms"] * 1e-3) / 1e12 if L["ms"] > 0 else 0.0
    print(f"  {L['phase']:9s} level {L['level']:3d} ctas {L['ctas']:7d} gen {L['generated']} "
          f"ms {L['ms']:9.3f} TF/s {tf:6.2f}")
