"""GPU parity tests: the sm_100a path through the C-ABI vs the oracle (the reference's own
evaluate(), compiled unmodified) on the SAME compressed trees. Tolerance: relative 2-norm
<= 1e-12 in fp64 (BASELINE.json north_star); flop counts must match the reference counter
exactly; eps2 must reproduce the reference's."""
import numpy as np
import pytest

from tests._util import rel2, to_tree

pytestmark = pytest.mark.gpu

TOL = 1e-12  # north_star: relative 2-norm vs the reference evaluate, fp64


def check_parity(G, R, h, r=3, seed=5, modes=None, tol=TOL):
    flat = h.export()
    tree = to_tree(flat)
    w = R.rng_gauss(flat.n, r, seed)
    u_ref, flops_ref, _ = h.evaluate(w)
    if modes is None:
        modes = [dict(stored=True)]
        if flat.coords is not None:
            modes += [dict(stored=False), dict(stored=False, near_mode=G.BLOCKS_MATERIALIZE,
                                               far_mode=G.BLOCKS_MATERIALIZE)]
    out = []
    for kw in modes:
        with G.Evaluator(tree, **kw) as ev:
            p = ev.evaluate(w)
            assert p.flops == flops_ref, (kw, p.flops, flops_ref)
            err = rel2(p.u, u_ref)
            assert err <= tol, (kw, err)
            out.append(p.u)
    return out, u_ref, w


def test_single_leaf_matches_dense(gpu, oracle):
    """test_evaluate.cpp:38-51 (randspd N=24 m=32): one leaf, u = D w; flops = 2*24*24*3."""
    h = oracle.compress_randspd(24, 3, m=32, s=16)
    (u,), u_ref, w = check_parity(gpu, oracle, h, r=3)
    assert np.allclose(h.unpermute(u), h.dense() @ w, rtol=1e-14, atol=1e-14)


def test_exact_representation_two_leaves(gpu, oracle):
    """test_compress.cpp:265-280 / test_evaluate.cpp:155-171: budget 1, D + S only."""
    h = oracle.compress_randspd(64, 2, m=32, s=32, kappa=8, budget=1.0)
    (u,), _, w = check_parity(gpu, oracle, h, r=2)
    ex = h.dense() @ w
    assert rel2(h.unpermute(u), ex) <= 1e-13


@pytest.mark.parametrize("n,budget,seed", [(200, 0.03, 1), (300, 0.05, 4), (400, 0.03, 13), (512, 0.0, 7)])
def test_smooth_gaussian_fixtures(gpu, oracle, n, budget, seed):
    """smooth_fixture (test_evaluate.cpp:23-34), all block modes."""
    pc = oracle.points_gaussian(n, 2, seed)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 3.0, m=32, s=32, tau=1e-7, kappa=8, budget=budget, seed=seed)
    check_parity(gpu, oracle, h, r=4)


@pytest.mark.parametrize("n", [2048, 4096])
def test_acceptance_fixture_parity_and_golden_flops(gpu, oracle, n):
    """reference_fixture (test_acceptance.cpp:39-52); eval_flops golden (test_output.txt:39-42)."""
    golden = {2048: 8126464, 4096: 17563648}
    pc = oracle.points_gaussian(n, 6, 42)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
    flat = h.export()
    with gpu.Evaluator(to_tree(flat)) as ev:
        assert ev.flops(1) == golden[n]
    check_parity(gpu, oracle, h, r=8)


def test_config1_tree_from_reference_compress(gpu, oracle):
    """BASELINE config 1: Gaussian N=8192 uniform d=6, h=1, m=s=128, budget .03, r=64."""
    rng = np.random.default_rng(0)
    pc = np.asfortranarray(rng.random((6, 8192)))
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=128, s=128, tau=1e-5, kappa=32, budget=0.03,
                               seed=0, threads=8)
    check_parity(gpu, oracle, h, r=64, modes=[dict(stored=False), dict(stored=True)])


@pytest.mark.parametrize("kernel,p0,p1", [("LAPLACE", -1.0, 0.0), ("EXPONENTIAL", 1.0, 0.0),
                                          ("POLYNOMIAL", 1.0, 2.0)])
def test_other_kernels(gpu, oracle, kernel, p0, p1):
    pc = oracle.points_gaussian(1000, 3, 7)
    h = oracle.compress_kernel(getattr(oracle, kernel), pc, p0, p1, m=64, s=48, budget=0.1, seed=1, threads=8)
    check_parity(gpu, oracle, h, r=5)


def test_odd_ranks_and_sizes(gpu, oracle):
    """Odd leaf sizes / odd ranks exercise the padded layouts (pad2 offsets, zero columns)."""
    pc = oracle.points_gaussian(777, 3, 11)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.3, m=37, s=23, tau=1e-9, kappa=8, budget=0.07, seed=2)
    f = h.export()
    assert (f.rank[1:] % 2 == 1).any() and ((f.end - f.start)[f.left < 0] % 2 == 1).any()
    check_parity(gpu, oracle, h, r=7)


@pytest.mark.parametrize("r", [1, 3, 127, 130, 300])
def test_rhs_counts(gpu, oracle, r):
    """Column counts that do not fill a tile (r % BN != 0) and r = 1."""
    pc = oracle.points_gaussian(600, 3, 3)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=40, budget=0.05, seed=3)
    check_parity(gpu, oracle, h, r=r, modes=[dict(stored=False)])


def test_rhs_chunking_matches(gpu, oracle):
    """Column chunking (max_rhs_chunk) is invisible: evaluation is column-separable."""
    pc = oracle.points_gaussian(700, 3, 5)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=40, budget=0.05, seed=5)
    tree = to_tree(h.export())
    w = oracle.rng_gauss(700, 37, 1)
    u_ref, _, _ = h.evaluate(w)
    with gpu.Evaluator(tree, max_rhs_chunk=8) as ev:
        p = ev.evaluate(w)
    assert rel2(p.u, u_ref) <= TOL
    with gpu.Evaluator(tree) as ev:
        assert np.array_equal(ev.evaluate(w).u, p.u)


def test_eps2_reproduces_reference(gpu, oracle):
    """error_eps2 (evaluate.hpp:330-373) on the criterion-2 fixture: 0.34486 (test_output.txt:21)."""
    n = 8192
    pc = oracle.points_gaussian(n, 6, 42)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
    rep = h.error_eps2(1, 100, 42)
    rows, w = oracle.eps2_draw(n, 1, 100, 42)
    with gpu.Evaluator(to_tree(h.export())) as ev:
        u = ev.unpermute(ev.evaluate(w).u)
    exact = h.exact_rows(rows, w)
    d = u[rows] - exact
    eps2 = float(np.sqrt((d ** 2).sum() / (exact ** 2).sum()))
    assert abs(eps2 - rep["eps2"]) <= 1e-10 * rep["eps2"]
    assert f"{eps2:.6g}" == "0.34486"


def test_zero_linearity_symmetry_determinism(gpu, oracle):
    """test_evaluate.cpp:53-83 restated on the GPU path."""
    pc = oracle.points_gaussian(900, 3, 4)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=48, tau=1e-7, kappa=8, budget=0.05, seed=4)
    with gpu.Evaluator(to_tree(h.export())) as ev:
        assert np.abs(ev.evaluate(np.zeros((900, 2))).u).max() == 0.0
        x, y = oracle.rng_gauss(900, 1, 1), oracle.rng_gauss(900, 1, 2)
        ux, uy = ev.evaluate(x).u, ev.evaluate(y).u
        uc = ev.evaluate(2.25 * x - 0.5 * y).u
        assert np.linalg.norm(uc - 2.25 * ux + 0.5 * uy) <= 1e-12 * (np.linalg.norm(ux) + np.linalg.norm(uy))
        kx, ky = ev.unpermute(ux), ev.unpermute(uy)
        scale = np.linalg.norm(x) * np.linalg.norm(ky) + np.linalg.norm(y) * np.linalg.norm(kx)
        assert abs((x.T @ ky).item() - (kx.T @ y).item()) <= 1e-12 * scale
        w = oracle.rng_gauss(900, 9, 3)
        assert np.array_equal(ev.evaluate(w).u, ev.evaluate(w).u)  # no atomics: bitwise repeatable


def test_malformed_input_errors(gpu, oracle):
    """evaluate.hpp:288-289 -> std::invalid_argument -> GOFMM_ERR_INVALID (2)."""
    pc = oracle.points_gaussian(200, 2, 1)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 3.0, m=32, s=32, budget=0.03, seed=1)
    with gpu.Evaluator(to_tree(h.export())) as ev:
        with pytest.raises(gpu.InvalidArgument) as e:
            ev.evaluate(np.zeros((199, 1)))
        assert e.value.code == 2
        with pytest.raises(gpu.InvalidArgument):
            ev.evaluate(np.zeros((200, 0)))


def test_device_api_and_unpermute(gpu, oracle):
    """gofmm_evaluate_device / gofmm_unpermute_device agree with the host API."""
    import torch

    from paper_1707_00164_b200 import _lib as L

    pc = oracle.points_gaussian(1500, 3, 9)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=48, budget=0.05, seed=9)
    w = oracle.rng_gauss(1500, 6, 2)
    with gpu.Evaluator(to_tree(h.export())) as ev:
        uh = ev.evaluate(w).u
        wd = torch.from_numpy(np.ascontiguousarray(w.T)).cuda().t()
        ud, _ = ev.evaluate_torch(wd)
        torch.cuda.synchronize()
        assert np.array_equal(ud.cpu().numpy(), uh)
        uo = torch.empty_like(ud)
        L.check(L.lib().gofmm_unpermute_device(ev._h, ud.data_ptr(), ud.stride(1), 6, uo.data_ptr(), uo.stride(1),
                                               None))
        torch.cuda.synchronize()
        assert np.array_equal(uo.cpu().numpy(), ev.unpermute(uh))


def test_graph_replay_recapture(gpu, oracle, monkeypatch):
    """Device evaluations replay one captured CUDA graph; new buffers / r re-capture it. Every replay
    is bitwise equal to the same evaluation with graphs disabled (GOFMM_NO_GRAPH=1)."""
    import torch

    pc = oracle.points_gaussian(2000, 3, 4)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=48, budget=0.05, seed=4)
    tree = to_tree(h.export())
    ws = [oracle.rng_gauss(2000, r, 7 + r) for r in (5, 5, 70, 300)]
    outs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("GOFMM_NO_GRAPH", flag)
        with gpu.Evaluator(tree) as ev:
            res = []
            for k in (0, 1, 0, 2, 3, 2):  # A, B, A again (pointer change back), other r's
                wd = torch.from_numpy(np.ascontiguousarray(ws[k].T)).cuda().t()
                ud, _ = ev.evaluate_torch(wd)
                ud2, _ = ev.evaluate_torch(wd, out=ud)  # same buffers: replay
                torch.cuda.synchronize()
                res.append(ud2.cpu().numpy().copy())
        outs[flag] = res
    for a, b in zip(outs["0"], outs["1"]):
        assert np.array_equal(a, b)
    u_ref, _, _ = h.evaluate(ws[3])
    assert rel2(outs["0"][4], u_ref) <= TOL


def test_c3_shaped_sample_parity(gpu, oracle):
    """A c3-shaped tree (d=8, m=s=512, budget .03, r=512) at N=2^15 through the reference evaluate."""
    from paper_1707_00164_b200 import synth

    tree, cfg = synth.make_config_tree("c3", n=1 << 15)
    ref = oracle.import_flat(tree, threads=8)
    w = np.asfortranarray(np.random.default_rng(3).standard_normal((tree.n, 512)))
    u_ref, flops_ref, _ = ref.evaluate(w, threads=8)
    with gpu.Evaluator(tree) as ev:
        p = ev.evaluate(w)
    assert p.flops == flops_ref
    assert rel2(p.u, u_ref) <= TOL


def test_full_size_c3_linearity(gpu):
    """Size-independent property at BASELINE config-3 scale (N=2^20, r=512, budget .03)."""
    import torch

    from paper_1707_00164_b200 import synth

    tree, cfg = synth.make_config_tree("c3")
    with gpu.Evaluator(tree) as ev:
        g = torch.Generator(device="cuda").manual_seed(7)
        x = torch.randn((512, tree.n), dtype=torch.float64, device="cuda", generator=g).t()
        y = torch.randn((512, tree.n), dtype=torch.float64, device="cuda", generator=g).t()
        ux = ev.evaluate_torch(x)[0].clone()
        uy = ev.evaluate_torch(y)[0].clone()
        uc = ev.evaluate_torch((2.25 * x - 0.5 * y).t().contiguous().t())[0]
        torch.cuda.synchronize()
        num = torch.linalg.norm(uc - 2.25 * ux + 0.5 * uy).item()
        den = torch.linalg.norm(ux).item() + torch.linalg.norm(uy).item()
        assert num <= 1e-12 * den


def simulate_subtree_split(G, tree, w_np, nranks):
    """All nranks of the subtree-split evaluation on ONE device: stage1 per rank, the all-gather
    as a concatenation of the send buffers, stage2 per rank (each writes its own rows of u)."""
    import torch

    r = w_np.shape[1]
    evs = [G.Evaluator(tree, rank=g, nranks=nranks) for g in range(nranks)]
    infos = [e.dist_info() for e in evs]
    slot = infos[0]["max_send_rows"] * r
    w = torch.from_numpy(np.ascontiguousarray(w_np.T)).cuda().t()
    sends = [torch.zeros(slot, dtype=torch.float64, device="cuda") for _ in evs]
    for e, sb in zip(evs, sends):
        e.dist_stage1_torch(w, sb)
    recv = torch.cat(sends) if slot else torch.zeros(0, dtype=torch.float64, device="cuda")
    u = torch.full((r, tree.n), float("nan"), dtype=torch.float64, device="cuda").t()
    for e in evs:
        e.dist_stage2_torch(recv, r, u)
    torch.cuda.synchronize()
    out = u.cpu().numpy()
    for e in evs:
        e.close()
    return out, infos


@pytest.mark.parametrize("nranks", [1, 2, 4, 8])
def test_subtree_split_matches_single_gpu(gpu, oracle, nranks):
    """north_star (4): subtree split + one all-gather reproduces the single-GPU / reference result."""
    from paper_1707_00164_b200 import synth

    tree, _ = synth.make_config_tree("c3", n=1 << 15, seed=1)
    w = np.asfortranarray(np.random.default_rng(5).standard_normal((tree.n, 24)))
    with gpu.Evaluator(tree) as ev:
        single = ev.evaluate(w)
    u, infos = simulate_subtree_split(gpu, tree, w, nranks)
    assert not np.isnan(u).any(), "some rows of u were not written by their owner"
    assert rel2(u, single.u) <= TOL
    assert all(i["full_flops_per_rhs"] * 24 == single.flops for i in infos)
    assert sum(i["own_row_end"] - i["own_row_begin"] for i in infos) == tree.n


def test_subtree_split_reference_tree(gpu, oracle):
    """Same on a tree from the reference compress (acceptance fixture, N=4096, 4 ranks) vs the oracle."""
    pc = oracle.points_gaussian(4096, 6, 42)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
    tree = to_tree(h.export())
    w = oracle.rng_gauss(4096, 8, 2)
    u_ref, _, _ = h.evaluate(w)
    u, _ = simulate_subtree_split(gpu, tree, w, 4)
    assert rel2(u, u_ref) <= TOL


def test_gpu_error_eps2_matches_reference(gpu, oracle):
    """error_eps2 computed entirely by the product (reference RNG restated in the C-ABI, exact rows
    matrix-free on the GPU) equals the reference's eps2 on the criterion-2 fixture (0.34486)."""
    pc = oracle.points_gaussian(8192, 6, 42)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
    rep_ref = h.error_eps2(1, 100, 42)
    with gpu.Evaluator(to_tree(h.export())) as ev:
        rep = ev.error_eps2(1, 100, 42)
        rows, w = oracle.eps2_draw(8192, 3, 50, 5)
        ex_gpu = ev.exact_rows(rows, w)
    assert rep["sample_rows"] == rep_ref["sample_rows"]
    assert abs(rep["eps2"] - rep_ref["eps2"]) <= 1e-10 * rep_ref["eps2"]
    assert np.allclose(rep["per_entry"], rep_ref["per_entry"], rtol=1e-9)
    assert rel2(ex_gpu, h.exact_rows(rows, w)) <= 1e-13
