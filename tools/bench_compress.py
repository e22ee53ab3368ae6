"""Product compress (gofmm_compress, device entries) at the BASELINE configurations, with the
reference compress timed beside it where it finishes in minutes — SURVEY.md §8(f).3 evidence.

  python tools/bench_compress.py c3 [n] [--ref-n N]   -> one JSON line per run
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1707_00164_b200 as G  # noqa: E402
from paper_1707_00164_b200 import synth  # noqa: E402


def cloud(cfg, n, seed=0):
    fn = {"uniform": synth.uniform_cloud, "gaussian": synth.gaussian_cloud, "covtype": synth.covtype_like}[cfg["cloud"]]
    return fn(n, cfg["d"], seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="c3")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--ref-n", type=int, default=0, help="also time the reference compress at this N")
    ap.add_argument("--entries", default="device")
    a = ap.parse_args()
    cfg = dict(synth.CONFIGS[a.config])
    n = a.n or cfg["n"]
    pc = cloud(cfg, n)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    res = G.compress(pc, cfg["kernel"], (cfg["h"], 0.0), m=cfg["m"], s=cfg["s"], budget=cfg["budget"],
                     distance="kernel", seed=0, threads=threads, entries=a.entries)
    wall = time.perf_counter() - t0
    st = dict(res.stats)
    line = {"what": "product compress", "config": a.config, "n": n, "entries": a.entries, "wall_s": round(wall, 2),
            "threads": threads, "stats": st}
    with G.Evaluator(res.tree) as ev:
        line["eval_flops_per_rhs"] = ev.flops(1)
        line["eps2"] = ev.error_eps2(1, 100, 0)["eps2"]
    print(json.dumps(line), flush=True)
    if a.ref_n:
        from oracle import refpy as R

        pr = cloud(cfg, a.ref_n)
        t0 = time.perf_counter()
        h = R.compress_kernel(cfg["kernel"], pr, cfg["h"], 0.0, m=cfg["m"], s=cfg["s"], budget=cfg["budget"], seed=0,
                              threads=threads)
        tr = time.perf_counter() - t0
        t0 = time.perf_counter()
        r2 = G.compress(pr, cfg["kernel"], (cfg["h"], 0.0), m=cfg["m"], s=cfg["s"], budget=cfg["budget"],
                        distance="kernel", seed=0, threads=threads, entries=a.entries)
        tp = time.perf_counter() - t0
        print(json.dumps({"what": "reference vs product compress", "config": a.config, "n": a.ref_n,
                          "reference_s": round(tr, 2), "product_s": round(tp, 2), "speedup": round(tr / tp, 1),
                          "reference_stats": h.compress_stats(), "product_entries": r2.stats["entries_evaluated"],
                          "threads": threads}), flush=True)


if __name__ == "__main__":
    main()
