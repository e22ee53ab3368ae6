"""CPU tests of the boundary and host logic: the C-ABI library loads and exports every symbol
include/gofmm_b200.h declares, descriptor validation mirrors the reference's errors, the product
fails loudly without a device, and the synthetic workload trees satisfy the reference invariants."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1707_00164_b200 import _lib as L
from paper_1707_00164_b200 import synth

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gofmm_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(gofmm_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = L.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(L.EXPORTS)
    assert lib.gofmm_abi_version() == 2  # 2: gofmm_options.precision + the *_f32 entry points


def _desc_from_tree(t, keep):
    def p(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a.ctypes.data_as(C.c_void_p)

    d = L.TreeDesc()
    d.n, d.num_nodes = t.n, t.num_nodes
    for f in ("parent", "left", "right", "level", "start", "end", "iperm", "rank"):
        setattr(d, f, p(getattr(t, f), np.int32))
    d.skel_offset, d.skel_idx = p(t.skel_off, np.int64), p(np.append(t.skel_idx, 0), np.int32)
    d.proj_offset, d.proj = p(t.proj_off, np.int64), p(np.append(t.proj, 0), np.float64)
    d.num_near, d.near_a, d.near_b = len(t.near_a), p(np.append(t.near_a, 0), np.int32), p(np.append(t.near_b, 0), np.int32)
    d.num_far, d.far_a, d.far_b = len(t.far_a), p(np.append(t.far_a, 0), np.int32), p(np.append(t.far_b, 0), np.int32)
    d.source, d.kernel, d.dim = L.SOURCE_KERNEL, 0, t.coords.shape[0]
    d.coords = p(np.asfortranarray(t.coords).ravel(order="F"), np.float64)
    d.kparam[0] = 1.0
    return d


def _create(d):
    h = C.c_void_p()
    rc = L.lib().gofmm_create(C.byref(d), None, C.byref(h))
    return rc, h


def test_create_validates_before_touching_a_device():
    t, _ = synth.make_config_tree("c1", n=1024)
    keep = []
    d = _desc_from_tree(t, keep)
    d.n = 0
    assert _create(d)[0] == L.GOFMM_ERR_INVALID
    d = _desc_from_tree(t, keep)
    bad_right = np.ascontiguousarray(t.right, dtype=np.int32).copy()
    bad_right[0] += 1  # children must be consecutive ids (tree.hpp:213-217)
    keep.append(bad_right)
    d.right = bad_right.ctypes.data_as(C.c_void_p)
    assert _create(d)[0] == L.GOFMM_ERR_INVALID
    assert b"consecutive" in L.lib().gofmm_last_error()


def test_no_cpu_fallback_without_device():
    """A valid descriptor on a box without a GPU must fail loudly (code 5), not compute on CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present; the GPU suite covers creation")
    t, _ = synth.make_config_tree("c1", n=1024)
    keep = []
    rc, _ = _create(_desc_from_tree(t, keep))
    assert rc == L.GOFMM_ERR_CUDA
    assert b"no CUDA device" in L.lib().gofmm_last_error()


def coverage(t):
    """audit_coverage (test_compress.cpp:62-83) on a flattened tree."""
    n = t.n
    cov = np.zeros((n, n), dtype=np.int32)
    idx = lambda a: t.iperm[t.start[a]:t.end[a]]  # noqa: E731
    for a in np.nonzero(t.left < 0)[0]:
        i = idx(a)
        cov[np.ix_(i, i)] += 1
    for a, b in list(zip(t.near_a, t.near_b)) + list(zip(t.far_a, t.far_b)):
        ia, ib = idx(a), idx(b)
        cov[np.ix_(ia, ib)] += 1
        cov[np.ix_(ib, ia)] += 1
    return cov


@pytest.mark.parametrize("budget", [0.0, 0.05, 0.3, 1.0])
def test_synthetic_tree_invariants(budget):
    coords = synth.gaussian_cloud(700, 3, 5)
    t = synth.synthetic_tree(coords, m=40, s=24, budget=budget, kernel=0)
    # BFS order, consecutive children, balanced split (left = ceil(n/2))
    for i in range(t.num_nodes):
        if t.left[i] >= 0:
            assert t.right[i] == t.left[i] + 1
            cnt = t.end[i] - t.start[i]
            assert t.end[t.left[i]] - t.start[t.left[i]] == cnt - cnt // 2
        else:
            assert t.end[i] - t.start[i] <= 40
    assert sorted(t.iperm.tolist()) == list(range(700))
    assert t.rank[0] == -1
    # nestedness (test_compress.cpp:326-332)
    for i in range(1, t.num_nodes):
        sk = set(t.skel_idx[t.skel_off[i]:t.skel_off[i + 1]].tolist())
        if t.left[i] >= 0:
            ch = set(t.skel_idx[t.skel_off[t.left[i]]:t.skel_off[t.left[i] + 1]].tolist())
            ch |= set(t.skel_idx[t.skel_off[t.right[i]]:t.skel_off[t.right[i] + 1]].tolist())
            assert sk <= ch
        else:
            assert sk <= set(t.iperm[t.start[i]:t.end[i]].tolist())
    cov = coverage(t)
    assert np.array_equal(cov, np.ones((700, 700), dtype=np.int32)), "exactly-once coverage"
    if budget == 0.0:
        assert len(t.near_a) == 0 and len(t.far_a) == int((t.left >= 0).sum())
    # pairs stored once, a < b, sorted
    assert all(a < b for a, b in zip(t.near_a, t.near_b))
    assert list(zip(t.far_a, t.far_b)) == sorted(zip(t.far_a, t.far_b))


def test_synthetic_tree_runs_through_reference_evaluate(oracle):
    """The oracle imports a synthetic tree and the reference evaluate agrees with the dense
    assembly D + S + U V^T of that same tree (an independent check of both)."""
    coords = synth.covtype_like(300, 4, seed=3)
    t = synth.synthetic_tree(coords, m=32, s=20, budget=0.1, kernel=0, kparams=(1.5, 0.0))
    ref = oracle.import_flat(t)
    w = np.random.default_rng(0).standard_normal((300, 2))
    u, flops, _ = ref.evaluate(w)
    f = ref.export()
    # dense reconstruct (test_compress.cpp:19-59) in original order
    K = np.zeros((300, 300))
    idx = lambda a: f.iperm[f.start[a]:f.end[a]]  # noqa: E731

    def proj(a):
        k, o = f.rank[a], f.proj_off[a]
        c = (f.proj_off[a + 1] - o) // k
        return f.proj[o:o + k * c].reshape((k, c), order="F")

    def transfer(a):
        if f.left[a] < 0:
            return proj(a)
        tl, tr = transfer(f.left[a]), transfer(f.right[a])
        blk = np.zeros((tl.shape[0] + tr.shape[0], tl.shape[1] + tr.shape[1]))
        blk[:tl.shape[0], :tl.shape[1]] = tl
        blk[tl.shape[0]:, tl.shape[1]:] = tr
        return proj(a) @ blk

    for a in np.nonzero(f.left < 0)[0]:
        d0 = f.diag_off[a]
        na = f.end[a] - f.start[a]
        K[np.ix_(idx(a), idx(a))] += f.diag[d0:d0 + na * na].reshape((na, na), order="F")
    for q, (a, b) in enumerate(zip(f.near_a, f.near_b)):
        na, nb = f.end[a] - f.start[a], f.end[b] - f.start[b]
        blk = f.near_blk[f.near_off[q]:f.near_off[q] + na * nb].reshape((na, nb), order="F")
        K[np.ix_(idx(a), idx(b))] += blk
        K[np.ix_(idx(b), idx(a))] += blk.T
    for q, (a, b) in enumerate(zip(f.far_a, f.far_b)):
        ka, kb = f.rank[a], f.rank[b]
        blk = f.far_blk[f.far_off[q]:f.far_off[q] + ka * kb].reshape((ka, kb), order="F")
        full = transfer(a).T @ blk @ transfer(b)
        K[np.ix_(idx(a), idx(b))] += full
        K[np.ix_(idx(b), idx(a))] += full.T
    dense = K @ w
    got = ref.unpermute(u)
    assert np.linalg.norm(got - dense) / np.linalg.norm(dense) <= 1e-12


def test_reference_rng_draws_match_oracle(oracle):
    """gofmm_rng_eps2_draw reproduces error_eps2's RNG consumption (evaluate.hpp:336-346)."""
    from paper_1707_00164_b200 import gofmm

    for n, r, k, seed in [(500, 3, 100, 7), (64, 2, 64, 11), (1000, 1, 10, 42)]:
        rows, w = gofmm.rng_eps2_draw(seed, n, r, k)
        rows_ref, w_ref = oracle.eps2_draw(n, r, k, seed)
        assert np.array_equal(rows, rows_ref)
        assert np.array_equal(w, w_ref)


def test_ghmx_roundtrip_reference_tree(oracle, tmp_path):
    """GHMX file format (hmx_io): a reference-compressed tree with stored blocks and coordinates
    survives save/load bit for bit, and the reloaded tree evaluates identically in the oracle."""
    from paper_1707_00164_b200 import CompressedTree, hmx_io

    pc = oracle.points_gaussian(400, 3, 2)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.2, m=32, s=24, budget=0.05, seed=2)
    t = CompressedTree.from_any(h.export())
    path = str(tmp_path / "tree.ghmx")
    hmx_io.save(path, t)
    t2 = hmx_io.load(path)
    for name in ("parent", "left", "right", "level", "start", "end", "iperm", "rank", "skel_off", "skel_idx",
                 "proj_off", "proj", "near_a", "near_b", "far_a", "far_b", "coords", "diag_off", "diag",
                 "near_off", "near_blk", "far_off", "far_blk"):
        assert np.array_equal(np.asarray(getattr(t, name)), np.asarray(getattr(t2, name))), name
    assert t2.kernel == t.kernel and tuple(t2.kparams) == tuple(t.kparams)
    w = np.random.default_rng(0).standard_normal((400, 3))
    u1 = oracle.import_flat(t).evaluate(w)[0]
    u2 = oracle.import_flat(t2).evaluate(w)[0]
    assert np.array_equal(u1, u2)
    with pytest.raises(ValueError):
        open(path, "r+b").write(b"XXXX")
        hmx_io.load(path)
