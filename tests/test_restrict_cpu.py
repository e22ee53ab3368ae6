"""CPU pin of the full-size parity machinery (tests/_util.py): the reference evaluate() on
restrict_to_leaves(tree, S) reproduces the full reference evaluate's u rows of the leaves in S BIT FOR
BIT (so the full-size GPU tests, which cannot hold the reference's ~280 GB of stored c3 blocks, still
compare against the reference's own numbers), and reference_flops restates the reference counter."""
import numpy as np
import pytest

from tests._util import leaf_rows, pick_leaves, reference_flops, restrict_to_leaves, to_tree


@pytest.mark.parametrize("kernel,budget,seed", [("GAUSSIAN", 0.1, 2), ("EXPONENTIAL", 0.2, 5), ("GAUSSIAN", 0.0, 7)])
def test_restricted_reference_rows_bitwise(oracle, kernel, budget, seed):
    R = oracle
    pc = R.points_gaussian(4096, 3, seed)
    h = R.compress_kernel(getattr(R, kernel), pc, 1.0, m=128, s=96, tau=1e-6, kappa=16, budget=budget, seed=seed,
                          threads=8)
    t = to_tree(h.export(blocks=False))
    w = R.rng_gauss(t.n, 5, 3)
    u, flops, _ = h.evaluate(w, threads=8)
    assert flops == reference_flops(t, 5)
    leaves = pick_leaves(t, 6, seed)
    sub = restrict_to_leaves(t, leaves)
    assert len(sub.far_a) < len(t.far_a) or budget == 0.0
    us, _, _ = R.import_flat(sub, threads=8).evaluate(w, threads=8)
    rows = leaf_rows(t, leaves)
    assert np.array_equal(us[rows], u[rows])


def test_reference_flops_golden(oracle):
    """The restated counter on the acceptance fixture equals the recorded 8,126,464 (test_output.txt:39)."""
    R = oracle
    pc = R.points_gaussian(2048, 6, 42)
    h = R.compress_kernel(R.GAUSSIAN, pc, 1.0, m=256, s=256, tau=1e-5, kappa=32, budget=0.03, kind=R.ANGLE, seed=42,
                          threads=8)
    assert reference_flops(to_tree(h.export(blocks=False)), 1) == 8126464
