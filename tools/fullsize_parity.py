"""Full-size parity at the BASELINE configurations on the PRODUCT-compressed trees (the trees bench.py
times): GPU evaluate (host API) vs the reference evaluate() (oracle/_ref, unmodified headers) on the
same tree and W, compared on sampled leaves through restrict_to_leaves (tests/_util.py: those rows are
bit-identical to the full reference evaluation, whose ~100-300 GB of stored blocks do not fit host RAM).
Optionally (--eps2) the reference's error_eps2 on the timed tree, assembled from the reference's u rows
of every leaf holding a sampled row (batched restrictions) and the reference's exact rows.

  python tools/fullsize_parity.py c3 c4 c5 [--leaves 8] [--eps2] [--fp32] > gpurun_out/fullsize.jsonl
Test infrastructure (imports oracle/); writes one JSON line per config."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1707_00164_b200 as G  # noqa: E402
from oracle import refpy as R  # noqa: E402
from tests._util import (THREADS, pick_leaves, product_config_tree, reference_eps2_on_leaves,  # noqa: E402
                         reference_flops, reference_rows_check)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--leaves", type=int, default=8)
    ap.add_argument("--ref-cols", type=int, default=0, help="reference columns (0 = all r)")
    ap.add_argument("--eps2", action="store_true")
    ap.add_argument("--eps2-batch", type=int, default=16)
    ap.add_argument("--fp32", action="store_true")
    a = ap.parse_args()
    for name in a.configs:
        cfg, tree, t_comp = product_config_tree(name)
        r = cfg["r"]
        line = {"config": name, "n": tree.n, "r": r, "near_pairs": len(tree.near_a), "far_pairs": len(tree.far_a),
                "tree": "product compress (gofmm_compress, GPU entries)", "compress_s": round(t_comp, 1)}
        w = np.asfortranarray(np.random.default_rng(7).standard_normal((tree.n, r)))
        with G.Evaluator(tree) as ev:
            p = ev.evaluate(w)
            line["flops_gpu"], line["flops_reference_formula"] = int(p.flops), reference_flops(tree, r)
            gpu_eps2 = ev.error_eps2(1, 100, 0) if a.eps2 else None
        leaves = pick_leaves(tree, a.leaves, 0)
        cols = a.ref_cols or (r if r <= 512 else 128)
        t0 = time.perf_counter()
        chk = reference_rows_check(R, tree, w, p.u, leaves, THREADS, cols=cols)
        chk["wall_s"] = round(time.perf_counter() - t0, 1)
        line["fp64"] = chk
        if a.fp32:
            with G.Evaluator(tree, precision="fp32") as ev:
                p32 = ev.evaluate(w.astype(np.float32))
            chk32 = reference_rows_check(R, tree, w, p32.u, leaves, THREADS, cols=cols)
            line["fp32"] = {k: chk32[k] for k in ("rel_error", "rows", "cols")}
        if gpu_eps2 is not None:
            t0 = time.perf_counter()
            e = reference_eps2_on_leaves(tree, gpu_eps2, 1, 100, 0, a.eps2_batch)
            e["wall_s"] = round(time.perf_counter() - t0, 1)
            e["rel_diff"] = abs(e["eps2_gpu"] - e["eps2_reference"]) / e["eps2_reference"]
            line["eps2"] = e
        print(json.dumps(line), flush=True)
        del p, w


if __name__ == "__main__":
    main()
