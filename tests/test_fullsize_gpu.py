"""Full-size parity at BASELINE configs c3, c4 and c5 on the PRODUCT-compressed trees — c3 is exactly
the tree bench.py times (N = 2^20, d = 8, m = s = 512, b = .03, r = 512). The reference cannot hold
these HMatrices (stored near/far blocks: ~280 GB at c3), so the GPU's u is compared with the
reference evaluate() (oracle/_ref) on restrict_to_leaves(tree, S) — whose u rows of the sampled leaves
S are bit-identical to the full reference evaluation (tests/test_restrict_cpu.py pins this) — at
north_star's tolerances (1e-12 fp64, 1e-5 fp32). The flop counter must equal the reference's formula,
and error_eps2 must reproduce the reference's (assembled from the reference's own u rows and exact
rows) to 1e-10. Evidence from the same procedure: profiles/r02_fullsize_parity.jsonl."""
import numpy as np
import pytest

from tests._util import (THREADS, pick_leaves, product_config_tree, reference_eps2_on_leaves, reference_flops,
                         reference_rows_check)

pytestmark = pytest.mark.gpu

TOL64, TOL32 = 1e-12, 1e-5


def _run(gpu, oracle, name, ref_cols=None, fp32=True, eps2=True):
    cfg, tree, _ = product_config_tree(name)
    r = cfg["r"]
    w = np.asfortranarray(np.random.default_rng(7).standard_normal((tree.n, r)))
    with gpu.Evaluator(tree) as ev:
        p = ev.evaluate(w)
        assert p.flops == reference_flops(tree, r)
        rep = ev.error_eps2(1, 100, 0) if eps2 else None
    leaves = pick_leaves(tree, 8, 0)
    chk = reference_rows_check(oracle, tree, w, p.u, leaves, THREADS, cols=ref_cols)
    assert chk["rel_error"] <= TOL64, chk
    del p
    if fp32:
        with gpu.Evaluator(tree, precision="fp32") as ev:
            p32 = ev.evaluate(w.astype(np.float32))
        chk32 = reference_rows_check(oracle, tree, w, p32.u, leaves, THREADS, cols=ref_cols)
        assert chk32["rel_error"] <= TOL32, chk32
    if rep is not None:
        e = reference_eps2_on_leaves(tree, rep, 1, 100, 0, 16)
        assert e["same_rows"]
        assert abs(e["eps2_gpu"] - e["eps2_reference"]) <= 1e-10 * e["eps2_reference"], e


def test_c3_timed_tree_full_size(gpu, oracle):
    _run(gpu, oracle, "c3")


def test_c4_full_size(gpu, oracle):
    _run(gpu, oracle, "c4")


def test_c5_full_size(gpu, oracle):
    """N = 2^22, r = 1024 on the GPU; the reference restricted evaluation on the first 64 columns
    (evaluate is column-separable). FP32 at this size: profiles/r02_fullsize_parity.jsonl."""
    _run(gpu, oracle, "c5", ref_cols=64, fp32=False, eps2=False)
