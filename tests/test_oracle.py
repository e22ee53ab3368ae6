"""CPU tests: the oracle (reference GOFMM headers compiled unmodified against oracle/eigen_shim)
pinned to every golden value the reference's own recorded run holds (proj/test_output.txt), plus
the reference's evaluate-path properties (test_evaluate.cpp) restated on the oracle."""
import numpy as np
import pytest

# proj/test_output.txt:39-42 (acceptance fixture, criterion 3)
GOLDEN_FLOPS = {2048: 8126464, 4096: 17563648, 8192: 41156608, 16384: 119013376}
GOLDEN_ENTRIES = {2048: 9378886, 4096: 19606678, 8192: 41467190, 16384: 93306486}


def acceptance_fixture(R, n, seed=42, threads=8):
    """reference_fixture (test_acceptance.cpp:39-52)."""
    pc = R.points_gaussian(n, 6, seed)
    return R.compress_kernel(R.GAUSSIAN, pc, 1.0, m=256, s=256, tau=1e-5, kappa=32, budget=0.03,
                             kind=R.ANGLE, seed=seed, threads=threads)


@pytest.mark.parametrize("n", [2048, 4096, 8192, 16384])
def test_golden_eval_flops_and_entries(oracle, n):
    h = acceptance_fixture(oracle, n)
    _, flops, _ = h.evaluate(oracle.rng_gauss(n, 1, 3), threads=8)
    assert flops == GOLDEN_FLOPS[n]
    assert h.compress_stats()["entries_evaluated"] == GOLDEN_ENTRIES[n]


def test_golden_eps2_criterion2(oracle):
    """n=8192 eps2=0.34486 (test_output.txt:21; single-threaded by contract)."""
    h = acceptance_fixture(oracle, 8192, threads=1)
    rep = h.error_eps2(1, 100, 42)
    assert f"{rep['eps2']:.6g}" == "0.34486"
    assert rep["eval_flops"] == GOLDEN_FLOPS[8192]


@pytest.mark.slow
def test_golden_budget_switch_criterion4(oracle):
    """mean eps2: budget=3% 0.206133, budget=0 0.206153 (test_output.txt:56)."""
    R = oracle
    n, r = 4096, 4
    sf = sh = 0.0
    for seed in range(1, 6):
        pc = R.points_gaussian(n, 6, seed)
        kw = dict(m=256, s=256, tau=1e-5, kappa=32, kind=R.ANGLE, seed=seed, threads=8)
        sf += R.compress_kernel(R.GAUSSIAN, pc, 1.0, budget=0.03, **kw).error_eps2(r, n, seed, threads=8)["eps2"]
        hss = R.compress_kernel(R.GAUSSIAN, pc, 1.0, budget=0.0, **kw)
        assert hss.compress_stats()["near_field_entries"] == 0
        sh += hss.error_eps2(r, n, seed, threads=8)["eps2"]
    assert f"{sf / 5:.6g}" == "0.206133"
    assert f"{sh / 5:.6g}" == "0.206153"


def smooth_fixture(R, n, seed, budget=0.03):
    """test_evaluate.cpp:23-34"""
    pc = R.points_gaussian(n, 2, seed)
    return R.compress_kernel(R.GAUSSIAN, pc, 3.0, m=32, s=32, tau=1e-7, kappa=8, budget=budget, seed=seed)


def test_single_leaf_bitwise_dense(oracle):
    """test_evaluate.cpp:38-51"""
    h = oracle.compress_randspd(24, 3, m=32, s=16)
    assert h.sizes().num_nodes == 1
    w = oracle.rng_gauss(24, 3, 5)
    u, flops, _ = h.evaluate(w)
    assert np.array_equal(h.unpermute(u), h.dense() @ w) or np.allclose(h.unpermute(u), h.dense() @ w, rtol=1e-15)
    assert flops == 2 * 24 * 24 * 3


def test_linearity_and_symmetry(oracle):
    """test_evaluate.cpp:59-83"""
    h = smooth_fixture(oracle, 256, 9)
    x, y = oracle.rng_gauss(256, 1, 1), oracle.rng_gauss(256, 1, 2)
    ux, uy = h.evaluate(x)[0], h.evaluate(y)[0]
    uc = h.evaluate(2.25 * x - 0.5 * y)[0]
    assert np.linalg.norm(uc - 2.25 * ux + 0.5 * uy) <= 1e-12 * (np.linalg.norm(ux) + np.linalg.norm(uy))
    h = smooth_fixture(oracle, 300, 4, 0.05)
    x, y = oracle.rng_gauss(300, 1, 7), oracle.rng_gauss(300, 1, 8)
    kx, ky = h.unpermute(h.evaluate(x)[0]), h.unpermute(h.evaluate(y)[0])
    scale = np.linalg.norm(x) * np.linalg.norm(ky) + np.linalg.norm(y) * np.linalg.norm(kx)
    assert abs((x.T @ ky).item() - (kx.T @ y).item()) <= 1e-12 * scale


def test_modes_and_threads_bitwise(oracle):
    """test_evaluate.cpp:85-103"""
    h = smooth_fixture(oracle, 400, 13)
    w = oracle.rng_gauss(400, 2, 3)
    ref = h.evaluate(w, mode=oracle.LEVEL_BY_LEVEL, threads=1)[0]
    for mode in (oracle.LEVEL_BY_LEVEL, oracle.TASK_DAG):
        for threads in (1, 2, 4, 8):
            assert np.array_equal(h.evaluate(w, mode=mode, threads=threads)[0], ref)


def test_exact_representation_eps2(oracle):
    """test_evaluate.cpp:155-171"""
    h = oracle.compress_randspd(64, 2, m=32, s=32, kappa=8, budget=1.0)
    rep = h.error_eps2(2, 64, 11)
    assert rep["eps2"] <= 1e-13 and rep["mean_sample"] <= 1e-13
    assert len(rep["per_entry"]) == 10 and len(rep["sample_rows"]) == 64


def test_matvec_vs_dense(oracle):
    """test_evaluate.cpp:137-153"""
    pc = oracle.points_gaussian(384, 2, 2)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 3.0, m=32, s=32, tau=1e-7, kappa=8, budget=0.03)
    w = oracle.rng_gauss(384, 1, 6)
    u = h.unpermute(h.evaluate(w)[0])
    ex = h.dense() @ w
    assert np.linalg.norm(u - ex) / np.linalg.norm(ex) <= 1e-3


def test_malformed_input(oracle):
    """test_evaluate.cpp:193-199: std::invalid_argument -> code 2"""
    h = smooth_fixture(oracle, 64, 1)
    with pytest.raises(oracle.OracleError) as e:
        h.evaluate(np.zeros((63, 1)))
    assert e.value.code == 2


def test_reconstruct_exact_limits(oracle):
    """test_compress.cpp:265-280: budget=1 with two leaves reproduces K; near entries 2*32*32."""
    h = oracle.compress_randspd(64, 2, m=32, s=32, kappa=8, budget=1.0)
    f = h.export()
    assert len(f.far_a) == 0 and len(f.near_a) == 1
    assert h.compress_stats()["near_field_entries"] == 2 * 32 * 32


def test_zero_budget_is_hss(oracle):
    """test_compress.cpp:282-299: budget 0 -> one sibling coupling per internal node."""
    pc = oracle.points_gaussian(128, 3, 4)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 2.0, m=16, s=16, budget=0.0, kind=oracle.GEOM)
    f = h.export()
    assert len(f.near_a) == 0
    internal = int((f.left >= 0).sum())
    assert len(f.far_a) == internal
