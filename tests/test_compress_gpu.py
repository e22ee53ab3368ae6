"""The product compress (gofmm_compress, csrc/gofmm_compress.cu) against the
reference compress() (compress.hpp:331-434, compiled unmodified in oracle/_ref).

* entries="host": bit-identical HMatrix structure — tree (nodes, permutation), near / far lists,
  skeleton ranks and indices, proj — and identical statistics (entries_evaluated, compress_flops,
  near_field_entries, max / mean skeleton) for every distance kind and kernel;
* the reference's recorded acceptance runs (test_output.txt:39-42): entries_evaluated
  9,378,886 / 19,606,678 / 41,467,190 / 93,306,486 and eval_flops 8,126,464 / 17,563,648 /
  41,156,608 / 119,013,376 at N = 2048 ... 16384;
* entries="device" (ANN distances and sampled blocks on the GPU): the same metric tree, nearly the
  same near field and ranks, an operator of the same accuracy (eps2), and — as for any tree — the
  GPU evaluation matches the reference evaluate on it to 1e-12."""
import numpy as np
import pytest

from tests._util import rel2, to_tree

pytestmark = pytest.mark.gpu

FIELDS = ("parent", "left", "right", "level", "start", "end", "iperm", "rank", "skel_off", "skel_idx", "proj_off",
          "near_a", "near_b", "far_a", "far_b")


def _ref(oracle, kernel, pc, p0, p1, **cfg):
    h = oracle.compress_kernel(kernel, pc, p0, p1, **cfg)
    return h, h.export(blocks=False), h.compress_stats()


def _ours(G, kernel, pc, p0, p1, entries="host", **cfg):
    kind = {0: "geom", 1: "kernel", 2: "angle"}[cfg.pop("kind", 1)]
    return G.compress(pc, kernel, (p0, p1), distance=kind, entries=entries, **cfg)


def assert_same_hmatrix(flat, res, st_ref):
    t = res.tree
    for f in FIELDS:
        a, b = np.asarray(getattr(flat, f)), np.asarray(getattr(t, f))
        assert a.shape == b.shape and np.array_equal(a, b), f
    assert np.array_equal(flat.proj, t.proj), "proj"
    for k in ("entries_evaluated", "compress_flops", "near_field_entries", "max_skeleton"):
        assert res.stats[k] == st_ref[k], (k, res.stats[k], st_ref[k])
    assert res.stats["mean_skeleton"] == pytest.approx(st_ref["mean_skeleton"], rel=1e-15)


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_host_entries_bit_identical_gaussian(gpu, oracle, kind):
    pc = oracle.points_gaussian(3000, 3, 5)
    cfg = dict(m=64, s=48, tau=1e-7, kappa=16, budget=0.05, kind=kind, seed=7, threads=8)
    _, flat, st = _ref(oracle, oracle.GAUSSIAN, pc, 1.0, 0.0, **cfg)
    res = _ours(gpu, gpu.KERNEL_GAUSSIAN, pc, 1.0, 0.0, **cfg)
    assert_same_hmatrix(flat, res, st)


@pytest.mark.parametrize("kernel,p0,p1", [("LAPLACE", None, 0.0), ("EXPONENTIAL", 1.0, 0.0), ("POLYNOMIAL", 1.0, 2.0)])
def test_host_entries_bit_identical_other_kernels(gpu, oracle, kernel, p0, p1):
    pc = oracle.points_gaussian(1500, 3, 9)
    if p0 is None:
        p0 = oracle.default_laplace_floor(pc)
    cfg = dict(m=64, s=40, tau=1e-6, kappa=12, budget=0.08, kind=1, seed=3, threads=8)
    _, flat, st = _ref(oracle, getattr(oracle, kernel), pc, p0, p1, **cfg)
    res = _ours(gpu, getattr(oracle, kernel), pc, p0, p1, **cfg)
    assert_same_hmatrix(flat, res, st)


@pytest.mark.parametrize("n,entries,flops", [(2048, 9378886, 8126464), (4096, 19606678, 17563648),
                                             (8192, 41467190, 41156608), (16384, 93306486, 119013376)])
def test_acceptance_golden_counts(gpu, oracle, n, entries, flops):
    """reference_fixture (test_acceptance.cpp:39-52): normal d=6 (seed 42), Gaussian h=1, angle
    distance, m=s=256 — the counts the reference recorded (test_output.txt:39-42)."""
    pc = oracle.points_gaussian(n, 6, 42)
    res = gpu.compress(pc, gpu.KERNEL_GAUSSIAN, (1.0, 0.0), m=256, s=256, tau=1e-5, kappa=32, budget=0.03,
                       distance="angle", seed=42, threads=8, entries="host")
    assert res.stats["entries_evaluated"] == entries
    with gpu.Evaluator(res.tree) as ev:
        assert ev.flops(1) == flops
    if n <= 4096:  # and the whole HMatrix equals the reference's
        _, flat, st = _ref(oracle, oracle.GAUSSIAN, pc, 1.0, 0.0, m=256, s=256, kind=oracle.ANGLE, seed=42, threads=8)
        assert_same_hmatrix(flat, res, st)


def test_device_entries_c3_shaped(gpu, oracle):
    """c3-shaped (COVTYPE-like d=8, m=s=512, b=.03) at N=2^16 with entries on the GPU."""
    from paper_1707_00164_b200 import synth

    pc = synth.covtype_like(1 << 16, 8, 0)
    kw = dict(m=512, s=512, tau=1e-5, kappa=32, budget=0.03, distance="kernel", seed=0, threads=16)
    dev = gpu.compress(pc, gpu.KERNEL_GAUSSIAN, (1.0, 0.0), entries="device", **kw)
    host = gpu.compress(pc, gpu.KERNEL_GAUSSIAN, (1.0, 0.0), entries="host", **kw)
    td, th = dev.tree, host.tree
    for f in ("parent", "left", "right", "level", "start", "end", "iperm"):  # metric tree: host in both
        assert np.array_equal(getattr(td, f), getattr(th, f)), f
    nd = set(zip(td.near_a.tolist(), td.near_b.tolist()))
    nh = set(zip(th.near_a.tolist(), th.near_b.tolist()))
    assert len(nd & nh) >= 0.95 * max(len(nh), 1)
    assert abs(dev.stats["mean_skeleton"] - host.stats["mean_skeleton"]) <= 0.02 * host.stats["mean_skeleton"]
    # any tree: the GPU evaluation equals the reference evaluate on it
    ref = oracle.import_flat(td, threads=16)
    w = oracle.rng_gauss(td.n, 64, 3)
    u_ref, flops, _ = ref.evaluate(w, threads=16)
    with gpu.Evaluator(td) as ev:
        p = ev.evaluate(w)
        e_dev = ev.error_eps2(2, 100, 0)["eps2"]
    assert p.flops == flops and rel2(p.u, u_ref) <= 1e-12
    with gpu.Evaluator(th) as ev:
        e_host = ev.error_eps2(2, 100, 0)["eps2"]
    assert abs(e_dev - e_host) <= 0.2 * e_host + 1e-12, (e_dev, e_host)


def test_compress_validation(gpu):
    pc = np.random.default_rng(0).standard_normal((3, 100))
    for bad in (dict(m=0), dict(s=300, m=256), dict(tau=0.0), dict(budget=1.5), dict(kappa=-1)):
        with pytest.raises(gpu.InvalidArgument):
            gpu.compress(pc, gpu.KERNEL_GAUSSIAN, (1.0, 0.0), **bad)
    with pytest.raises(gpu.InvalidArgument):
        gpu.compress(pc, gpu.KERNEL_GAUSSIAN, (-1.0, 0.0))
