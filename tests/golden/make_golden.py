"""Generates the golden fixtures in tests/golden/ from the REFERENCE (the oracle: the reference
headers compiled unmodified, oracle/Makefile). Run where /root/reference exists:

    python tests/golden/make_golden.py

Each fixture = a GHMX compressed tree (paper_1707_00164_b200/hmx_io.py, the reference's own
compress() output, stored blocks + coordinates) and an .npz with the W it was evaluated on, the
reference evaluate()'s u (permuted order) and its flop counter. tests/test_golden.py replays them:
on the CPU against the oracle (pins it), on the GPU without the oracle (parity travels as data)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refpy as R  # noqa: E402
from paper_1707_00164_b200 import CompressedTree, hmx_io  # noqa: E402

FIXTURES = {
    # name: (kernel, n, d, p0, compress kwargs, r, seeds (points, w))
    "gauss_n1024_d3": (R.GAUSSIAN, 1024, 3, 1.0, dict(m=64, s=48, tau=1e-7, kappa=16, budget=0.05, seed=2), 7, (5, 9)),
    "expo_n768_d2": (R.EXPONENTIAL, 768, 2, 0.7, dict(m=64, s=32, tau=1e-6, kappa=8, budget=0.1, seed=4), 3, (6, 10)),
}


def main():
    for name, (kernel, n, d, p0, kw, r, (ps, ws)) in FIXTURES.items():
        pc = R.points_gaussian(n, d, ps)
        h = R.compress_kernel(kernel, pc, p0, **kw)
        flat = h.export()
        w = R.rng_gauss(flat.n, r, ws)
        u, flops, _ = h.evaluate(w)
        hmx_io.save(os.path.join(HERE, name + ".ghmx"), CompressedTree.from_any(flat))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), w=w, u=u, flops=np.int64(flops))
        print(name, flat.n, r, flops)


if __name__ == "__main__":
    main()
