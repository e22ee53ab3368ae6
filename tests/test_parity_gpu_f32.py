"""GPU parity of the FP32 path (3xTF32 on tcgen05) against the reference's own FP64 evaluate()
(the oracle, compiled unmodified) on the same compressed trees. Tolerance: relative 2-norm
<= 1e-5 (BASELINE.json north_star, fp32); the flop counter is precision-independent and must
match exactly."""
import numpy as np
import pytest

from tests._util import rel2, to_tree

pytestmark = pytest.mark.gpu

TOL32 = 1e-5  # north_star: relative 2-norm vs the reference evaluate, fp32


def check_parity32(G, R, h, r=3, seed=5, modes=None, tol=TOL32):
    flat = h.export()
    tree = to_tree(flat)
    w = R.rng_gauss(flat.n, r, seed)
    u_ref, flops_ref, _ = h.evaluate(w)
    if modes is None:
        modes = [dict(stored=True)]
        if flat.coords is not None:
            modes += [dict(stored=False), dict(stored=False, near_mode=G.BLOCKS_MATERIALIZE,
                                               far_mode=G.BLOCKS_MATERIALIZE)]
    errs = []
    for kw in modes:
        with G.Evaluator(tree, precision="fp32", **kw) as ev:
            p = ev.evaluate(w.astype(np.float32))
            assert p.u.dtype == np.float32
            assert p.flops == flops_ref, (kw, p.flops, flops_ref)
            err = rel2(p.u.astype(np.float64), u_ref)
            assert err <= tol, (kw, err)
            errs.append(err)
    return errs


def test_f32_single_leaf(gpu, oracle):
    """test_evaluate.cpp:38-51 shape (one leaf, u = D w) through the stored-block FP32 path."""
    h = oracle.compress_randspd(24, 3, m=32, s=16)
    check_parity32(gpu, oracle, h, r=3)


def test_f32_exact_two_leaves(gpu, oracle):
    h = oracle.compress_randspd(64, 2, m=32, s=32, kappa=8, budget=1.0)
    check_parity32(gpu, oracle, h, r=2)


@pytest.mark.parametrize("n,budget,seed", [(200, 0.03, 1), (400, 0.03, 13), (512, 0.0, 7)])
def test_f32_smooth_gaussian_fixtures(gpu, oracle, n, budget, seed):
    """smooth_fixture (test_evaluate.cpp:23-34), stored / matrix-free / materialised blocks."""
    pc = oracle.points_gaussian(n, 2, seed)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 3.0, m=32, s=32, tau=1e-7, kappa=8, budget=budget, seed=seed)
    check_parity32(gpu, oracle, h, r=4)


def test_f32_acceptance_fixture(gpu, oracle):
    """reference_fixture (test_acceptance.cpp:39-52), N=4096 d=6 m=s=256."""
    pc = oracle.points_gaussian(4096, 6, 42)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
    check_parity32(gpu, oracle, h, r=8)


def test_f32_config1_tree(gpu, oracle):
    """BASELINE config 1 (N=8192 uniform d=6, h=1, m=s=128, budget .03, r=64) in fp32."""
    rng = np.random.default_rng(0)
    pc = np.asfortranarray(rng.random((6, 8192)))
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=128, s=128, tau=1e-5, kappa=32, budget=0.03,
                               seed=0, threads=8)
    check_parity32(gpu, oracle, h, r=64, modes=[dict(stored=False), dict(stored=True)])


@pytest.mark.parametrize("kernel,p0,p1", [("LAPLACE", -1.0, 0.0), ("EXPONENTIAL", 1.0, 0.0),
                                          ("POLYNOMIAL", 1.0, 2.0)])
def test_f32_other_kernels(gpu, oracle, kernel, p0, p1):
    pc = oracle.points_gaussian(1000, 3, 7)
    h = oracle.compress_kernel(getattr(oracle, kernel), pc, p0, p1, m=64, s=48, budget=0.1, seed=1, threads=8)
    check_parity32(gpu, oracle, h, r=5)


def test_f32_odd_ranks_and_sizes(gpu, oracle):
    pc = oracle.points_gaussian(777, 3, 11)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.3, m=37, s=23, tau=1e-9, kappa=8, budget=0.07, seed=2)
    check_parity32(gpu, oracle, h, r=7)


@pytest.mark.parametrize("r", [1, 64, 65, 128, 129, 300])
def test_f32_rhs_counts(gpu, oracle, r):
    """Column counts around the N-tile choices (64 / 128 / 256)."""
    pc = oracle.points_gaussian(600, 3, 3)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=40, budget=0.05, seed=3)
    check_parity32(gpu, oracle, h, r=r, modes=[dict(stored=False)])


def test_f32_chunking_zero_linearity(gpu, oracle):
    """Column chunking is invisible; zero in -> zero out; linear; bitwise repeatable."""
    pc = oracle.points_gaussian(700, 3, 5)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=40, budget=0.05, seed=5)
    tree = to_tree(h.export())
    w = oracle.rng_gauss(700, 37, 1).astype(np.float32)
    with gpu.Evaluator(tree, precision="fp32", max_rhs_chunk=8) as ev:
        pc8 = ev.evaluate(w).u
    with gpu.Evaluator(tree, precision="fp32") as ev:
        full = ev.evaluate(w).u
        assert np.array_equal(full, pc8)
        assert np.array_equal(ev.evaluate(w).u, full)
        assert np.abs(ev.evaluate(np.zeros((700, 3), np.float32)).u).max() == 0.0
        x, y = w[:, :1], w[:, 1:2]
        ux, uy = ev.evaluate(x).u.astype(np.float64), ev.evaluate(y).u.astype(np.float64)
        uc = ev.evaluate((2.25 * x - 0.5 * y).astype(np.float32)).u.astype(np.float64)
        assert np.linalg.norm(uc - 2.25 * ux + 0.5 * uy) <= 1e-5 * (np.linalg.norm(ux) + np.linalg.norm(uy))


def test_f32_precision_mismatch_errors(gpu, oracle):
    """An fp32 handle rejects the fp64 entry points (and vice versa) with GOFMM_ERR_INVALID."""
    import ctypes as C

    from paper_1707_00164_b200 import _lib as L

    pc = oracle.points_gaussian(200, 2, 1)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 3.0, m=32, s=32, budget=0.03, seed=1)
    tree = to_tree(h.export())
    w64 = np.zeros((200, 1))
    u64 = np.zeros((200, 1))
    w32 = np.zeros((200, 1), np.float32)
    with gpu.Evaluator(tree, precision="fp32") as ev:
        assert L.lib().gofmm_precision(ev._h) == L.PRECISION_F32
        rc = L.lib().gofmm_evaluate(ev._h, w64.ctypes.data_as(C.c_void_p), 200, 1, u64.ctypes.data_as(C.c_void_p),
                                    200, None)
        assert rc == L.GOFMM_ERR_INVALID
        with pytest.raises(gpu.InvalidArgument):
            ev.evaluate(np.zeros((199, 1), np.float32))
    with gpu.Evaluator(tree) as ev:
        rc = L.lib().gofmm_evaluate_f32(ev._h, w32.ctypes.data_as(C.c_void_p), 200, 1,
                                        w32.ctypes.data_as(C.c_void_p), 200, None)
        assert rc == L.GOFMM_ERR_INVALID


def test_f32_device_api(gpu, oracle):
    """gofmm_evaluate_device_f32 / gofmm_unpermute_device_f32 agree with the host API."""
    import torch

    from paper_1707_00164_b200 import _lib as L

    pc = oracle.points_gaussian(1500, 3, 9)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=48, budget=0.05, seed=9)
    w = oracle.rng_gauss(1500, 6, 2).astype(np.float32)
    with gpu.Evaluator(to_tree(h.export()), precision="fp32") as ev:
        uh = ev.evaluate(w).u
        wd = torch.from_numpy(np.ascontiguousarray(w.T)).cuda().t()
        ud, _ = ev.evaluate_torch(wd)
        torch.cuda.synchronize()
        assert np.array_equal(ud.cpu().numpy(), uh)
        uo = torch.empty_like(ud)
        L.check(L.lib().gofmm_unpermute_device_f32(ev._h, ud.data_ptr(), ud.stride(1), 6, uo.data_ptr(),
                                                   uo.stride(1), None))
        torch.cuda.synchronize()
        assert np.array_equal(uo.cpu().numpy(), ev.unpermute(uh))


def test_f32_graph_replay_recapture(gpu, oracle, monkeypatch):
    """FP32 device evaluations through the captured CUDA graph (replays and re-captures on new
    buffers / r) are bitwise equal to the same evaluations with graphs disabled."""
    import torch

    pc = oracle.points_gaussian(2000, 3, 4)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=64, s=48, budget=0.05, seed=4)
    tree = to_tree(h.export())
    ws = [oracle.rng_gauss(2000, r, 7 + r).astype(np.float32) for r in (5, 5, 70, 300)]
    outs = {}
    for flag in ("0", "1"):
        monkeypatch.setenv("GOFMM_NO_GRAPH", flag)
        with gpu.Evaluator(tree, precision="fp32") as ev:
            res = []
            for k in (0, 1, 0, 2, 3, 2):
                wd = torch.from_numpy(np.ascontiguousarray(ws[k].T)).cuda().t()
                ud, _ = ev.evaluate_torch(wd)
                ud2, _ = ev.evaluate_torch(wd, out=ud)
                torch.cuda.synchronize()
                res.append(ud2.cpu().numpy().copy())
        outs[flag] = res
    for a, b in zip(outs["0"], outs["1"]):
        assert np.array_equal(a, b)
    u_ref, _, _ = h.evaluate(ws[3].astype(np.float64))
    assert rel2(outs["0"][4].astype(np.float64), u_ref) <= TOL32


def test_f32_c3_shaped_sample(gpu, oracle):
    """A c3-shaped tree (d=8, m=s=512, budget .03, r=512) at N=2^15 vs the reference evaluate."""
    from paper_1707_00164_b200 import synth

    tree, _ = synth.make_config_tree("c3", n=1 << 15)
    ref = oracle.import_flat(tree, threads=8)
    w = np.asfortranarray(np.random.default_rng(3).standard_normal((tree.n, 512)))
    u_ref, flops_ref, _ = ref.evaluate(w, threads=8)
    with gpu.Evaluator(tree, precision="fp32") as ev:
        p = ev.evaluate(w.astype(np.float32))
    assert p.flops == flops_ref
    assert rel2(p.u.astype(np.float64), u_ref) <= TOL32


def test_f32_eps2_close_to_reference(gpu, oracle):
    """error_eps2 with an fp32 evaluation: the compression error (0.34486) dominates fp32 rounding."""
    pc = oracle.points_gaussian(8192, 6, 42)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
    rep_ref = h.error_eps2(1, 100, 42)
    with gpu.Evaluator(to_tree(h.export()), precision="fp32") as ev:
        rep = ev.error_eps2(1, 100, 42)
    assert abs(rep["eps2"] - rep_ref["eps2"]) <= 1e-4 * rep_ref["eps2"]


def simulate_subtree_split32(G, tree, w_np, nranks):
    """All nranks of the FP32 subtree-split evaluation on ONE device (see test_parity_gpu.py):
    stage1 per rank, the all-gather as a concatenation of the hi/lo send slots, stage2 per rank."""
    import torch

    r = w_np.shape[1]
    evs = [G.Evaluator(tree, rank=g, nranks=nranks, precision="fp32") for g in range(nranks)]
    slot = evs[0].send_elems(r)
    w = torch.from_numpy(np.ascontiguousarray(w_np.T.astype(np.float32))).cuda().t()
    sends = [torch.zeros(slot, dtype=torch.float32, device="cuda") for _ in evs]
    for e, sb in zip(evs, sends):
        e.dist_stage1_torch(w, sb)
    recv = torch.cat(sends) if slot else torch.zeros(0, dtype=torch.float32, device="cuda")
    u = torch.full((r, tree.n), float("nan"), dtype=torch.float32, device="cuda").t()
    for e in evs:
        e.dist_stage2_torch(recv, r, u)
    torch.cuda.synchronize()
    out = u.cpu().numpy()
    for e in evs:
        e.close()
    return out


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_f32_subtree_split_matches_single_gpu(gpu, oracle, nranks):
    """north_star (4) in FP32: subtree split + one all-gather equals the single-GPU FP32 result
    and stays within 1e-5 of the reference FP64 evaluate."""
    from paper_1707_00164_b200 import synth

    tree, _ = synth.make_config_tree("c3", n=1 << 15, seed=1)
    w = np.asfortranarray(np.random.default_rng(5).standard_normal((tree.n, 24)))
    ref = oracle.import_flat(tree, threads=8)
    u_ref, _, _ = ref.evaluate(w, threads=8)
    with gpu.Evaluator(tree, precision="fp32") as ev:
        single = ev.evaluate(w.astype(np.float32)).u
    u = simulate_subtree_split32(gpu, tree, w, nranks)
    assert not np.isnan(u).any(), "some rows of u were not written by their owner"
    assert rel2(u.astype(np.float64), single.astype(np.float64)) <= 1e-6
    assert rel2(u.astype(np.float64), u_ref) <= TOL32


def test_f32_two_pass_permutation_bitwise(gpu, oracle, monkeypatch):
    """The two-pass permutation (transpose + coalesced row gather, used for W >= 4 GB) forced on a
    small tree: u bitwise equal to the one-pass gather (both split the same W values)."""
    pc = oracle.points_gaussian(3000, 3, 4)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=128, s=64, tau=1e-7, kappa=16, budget=0.05, seed=3,
                               threads=8)
    tree = to_tree(h.export(blocks=False))
    w = oracle.rng_gauss(tree.n, 300, 6).astype(np.float32)
    outs = []
    for v in ("0", "1"):
        monkeypatch.setenv("GOFMM_PERM2", v)
        with gpu.Evaluator(tree, precision="fp32") as ev:
            outs.append(ev.evaluate(w).u)
    assert np.array_equal(outs[0], outs[1])
    u_ref, _, _ = h.evaluate(w.astype(np.float64), threads=8)
    assert rel2(outs[1].astype(np.float64), u_ref) <= TOL32
