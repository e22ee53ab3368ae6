"""Field-by-field comparison of the product compress (entries="host") with the reference compress
on one configuration — a debugging aid for tests/test_compress_gpu.py (prints the first mismatch)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1707_00164_b200 as G  # noqa: E402
from oracle import refpy as R  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 1
pc = R.points_gaussian(n, 3, 5)
cfg = dict(m=64, s=48, tau=1e-7, kappa=16, budget=0.05, seed=7, threads=8)
h = R.compress_kernel(R.GAUSSIAN, pc, 1.0, 0.0, kind=kind, **cfg)
f = h.export(blocks=False)
st = h.compress_stats()
res = G.compress(pc, G.KERNEL_GAUSSIAN, (1.0, 0.0), distance={0: "geom", 1: "kernel", 2: "angle"}[kind],
                 entries="host", **cfg)
t = res.tree
print("ref stats", st)
print("our stats", {k: res.stats[k] for k in st if k in res.stats})
for fld in ("parent", "left", "right", "level", "start", "end", "iperm", "near_a", "near_b", "far_a", "far_b", "rank",
            "skel_off", "skel_idx", "proj_off", "proj"):
    a, b = np.asarray(getattr(f, fld)), np.asarray(getattr(t, fld))
    if a.shape != b.shape:
        print(f"{fld}: shape {a.shape} vs {b.shape}")
        continue
    bad = np.nonzero(a != b)[0]
    print(f"{fld}: {'OK' if bad.size == 0 else f'{bad.size} mismatches, first at {bad[0]}: {a[bad[0]]} vs {b[bad[0]]}'}")
