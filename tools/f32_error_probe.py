"""FP32 path error budget on a c3-shaped tree: which part of the 3xTF32 evaluation dominates the
relative error vs the reference FP64 evaluate (matrix-free generation vs materialised blocks,
per phase). Test/diagnostic tooling: imports the oracle as the checker."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import refpy as R  # noqa: E402
from paper_1707_00164_b200 import BLOCKS_MATERIALIZE, Evaluator, synth  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 15
    cfgname = sys.argv[2] if len(sys.argv) > 2 else "c3"
    r = 64
    tree, cfg = synth.make_config_tree(cfgname, n=n)
    ref = R.import_flat(tree, threads=os.cpu_count() or 8)
    w = np.asfortranarray(np.random.default_rng(3).standard_normal((tree.n, r)))
    u_ref, _, _ = ref.evaluate(w, threads=os.cpu_count() or 8)
    out = {"n": n, "config": cfgname}
    w32 = w.astype(np.float32)
    for name, kw in [("matrix_free", {}), ("near_materialized", dict(near_mode=BLOCKS_MATERIALIZE)),
                     ("all_materialized", dict(near_mode=BLOCKS_MATERIALIZE, far_mode=BLOCKS_MATERIALIZE))]:
        with Evaluator(tree, precision="fp32", **kw) as ev:
            out[name] = rel(ev.evaluate(w32).u, u_ref)
    # the same W rounded to fp32, evaluated in fp64: the input-rounding floor
    with Evaluator(tree) as ev:
        out["fp64_of_fp32_input"] = rel(ev.evaluate(w32.astype(np.float64)).u, u_ref)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
