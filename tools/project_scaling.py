"""Projected strong scaling of the subtree-split evaluation from ONE B200.

Every rank g of P is created in turn on the single device and its two stages are timed with CUDA
events: stage1 (own-subtree permutation + N2S + pack) and stage2 (unpack + top tree + downward +
output of its own rows, fed a zero receive buffer of the real size). The all-gather between them is
NOT measured here (one GPU): it is estimated from its byte count at an assumed NVLink-5 NCCL bus
bandwidth (--busbw, GB/s). Projected T_P = max_g stage1 + allgather + max_g stage2, efficiency =
T_1 / (P * T_P). This is a projection, not a multi-GPU measurement."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1707_00164_b200 import Evaluator, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--ranks", default="2,4,8")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--busbw", type=float, default=650.0)
ap.add_argument("--tree", default="compress", choices=["compress", "synth"])
a = ap.parse_args()
if a.tree == "compress":  # bench.py's timed tree: the product compress of the config's cloud
    import bench

    cfg = dict(synth.CONFIGS[a.config], name=a.config)
    tree, _ = bench.workload_tree(cfg, cfg["n"], 0, "compress")
else:
    tree, cfg = synth.make_config_tree(a.config)
r = cfg["r"]
w = torch.randn((r, tree.n), dtype=torch.float64, device="cuda").t()
u = torch.zeros((r, tree.n), dtype=torch.float64, device="cuda").t()
st = torch.cuda.current_stream()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


with Evaluator(tree) as ev:
    t1 = timed(lambda: ev.evaluate_torch(w, out=u))
    flops = ev.flops(r)
out = {"config": a.config, "tree": a.tree, "n": tree.n, "r": r, "t1_ms": round(t1, 3), "busbw_gbs_assumed": a.busbw, "ranks": {}}
for P in [int(x) for x in a.ranks.split(",")]:
    s1, s2, slot = [], [], 0
    for g in range(P):
        ev = Evaluator(tree, rank=g, nranks=P)
        slot = ev.send_elems(r)
        send = torch.empty(max(slot, 1), dtype=torch.float64, device="cuda")
        recv = torch.zeros(max(slot * P, 1), dtype=torch.float64, device="cuda")
        s1.append(timed(lambda: ev.dist_stage1_torch(w, send)))
        s2.append(timed(lambda: ev.dist_stage2_torch(recv, r, u)))
        ev.close()
        del send, recv
        torch.cuda.empty_cache()
    ag_bytes = slot * 8 * (P - 1)  # received per rank
    ag_ms = ag_bytes / (a.busbw * 1e9) * 1e3
    tp = max(s1) + ag_ms + max(s2)
    out["ranks"][P] = {"stage1_ms_max": round(max(s1), 3), "stage2_ms_max": round(max(s2), 3),
                       "stage1_ms": [round(x, 2) for x in s1], "stage2_ms": [round(x, 2) for x in s2],
                       "allgather_bytes_per_rank": int(ag_bytes), "allgather_ms_est": round(ag_ms, 3),
                       "projected_ms": round(tp, 3), "projected_tflops": round(flops / (tp * 1e-3) / 1e12, 2),
                       "projected_efficiency": round(t1 / (P * tp), 4)}
    print(json.dumps({P: out["ranks"][P]}), flush=True)
print(json.dumps(out))
