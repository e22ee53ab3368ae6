"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py from the reference's own
compress() + evaluate()): GHMX trees with the W they were evaluated on, the reference u (permuted
order) and its flop counter. The CPU test replays them through the oracle (pins it: bit-identical);
the GPU test checks the product against the stored reference output WITHOUT the oracle, in all
three block modes."""
import os

import numpy as np
import pytest

from paper_1707_00164_b200 import hmx_io

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["gauss_n1024_d3", "expo_n768_d2"]


def rel2(a, b):  # local: the GPU test below must not import oracle/ at all
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def load(name):
    tree = hmx_io.load(os.path.join(HERE, name + ".ghmx"))
    z = np.load(os.path.join(HERE, name + ".npz"))
    return tree, np.asfortranarray(z["w"]), z["u"], int(z["flops"])


@pytest.mark.parametrize("name", NAMES)
def test_golden_oracle_replay(oracle, name):
    tree, w, u, flops = load(name)
    ref = oracle.import_flat(tree)
    u2, f2, _ = ref.evaluate(w)
    assert f2 == flops
    assert np.array_equal(u2, u)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_golden_gpu(gpu, name):
    tree, w, u, flops = load(name)
    for kw in (dict(), dict(stored=True), dict(near_mode=gpu.BLOCKS_MATERIALIZE, far_mode=gpu.BLOCKS_MATERIALIZE)):
        with gpu.Evaluator(tree, **kw) as ev:
            p = ev.evaluate(w)
        assert p.flops == flops, kw
        assert rel2(p.u, u) <= 1e-12, (kw, rel2(p.u, u))
