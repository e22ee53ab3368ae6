"""GPU batched skeletonisation vs the reference skeletonize_node
(compress.hpp:149-187, compiled unmodified in the oracle) on the SAME sampled blocks: ranks,
skeleton pivots, proj and achieved_tol must be bit-identical (the GPU issues the reference's
floating-point operations in the reference's order)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def gaussian_block(rng, rows, cols, d, h=1.0, scale=1.0):
    """K(sample points, candidate points) of the Gaussian kernel (oracle.hpp:148-159 form)."""
    xs = rng.standard_normal((rows, d)) * scale
    xc = rng.standard_normal((cols, d)) * scale
    d2 = ((xs[:, None, :] - xc[None, :, :]) ** 2).sum(-1)
    return np.exp(-d2 / (2 * h * h))


def blocks_suite():
    rng = np.random.default_rng(11)
    bl = [
        gaussian_block(rng, 60, 40, 3),
        gaussian_block(rng, 30, 50, 3),              # rows < cols: size = rows
        gaussian_block(rng, 288, 128, 6, 1.0, 0.5),  # c1 leaf shape (2s+32 samples, m candidates)
        gaussian_block(rng, 200, 256, 8),
        rng.standard_normal((70, 9)) @ rng.standard_normal((9, 45)),  # exact rank 9
        np.zeros((12, 7)),                            # all-zero: tau = 0 Householder branch
        np.ones((10, 6)),                             # identical columns: norm ties at every step
        rng.standard_normal((1, 5)),
        rng.standard_normal((5, 1)),
        rng.standard_normal((1, 1)),
    ]
    a = rng.standard_normal((40, 30))
    a[:, 5] = a[:, 2]                                 # duplicated column (pivot ties after the first)
    a[:, 11] = 0.0                                    # zero column (upd = 0 skips the downdate)
    bl.append(a)
    return bl


@pytest.mark.parametrize("s,tau", [(16, 1e-5), (64, 1e-7), (512, 0.0), (3, 1e-2)])
def test_skeletonize_bitwise_vs_reference(gpu, oracle, s, tau):
    from paper_1707_00164_b200 import skeletonize_batch

    blocks = blocks_suite()
    ref, _ = oracle.skeletonize_batch(blocks, s, tau, threads=4)
    got = skeletonize_batch(blocks, s, tau)
    for t, (b, (k, skel, proj, ach), g) in enumerate(zip(blocks, ref, got)):
        assert g.rank == k, (t, g.rank, k)
        assert np.array_equal(g.skel, skel), t
        assert np.array_equal(g.proj, proj), (t, np.abs(g.proj - proj).max())
        assert g.achieved_tol == ach, (t, g.achieved_tol, ach)
        # interpolation property of an ID: B ~= B[:, skel] proj
        if k < min(b.shape) and ach < 1e-6:
            assert np.linalg.norm(b - b[:, skel] @ proj) <= 1e-4 * np.linalg.norm(b)


def test_skeletonize_c3_shaped_nodes(gpu, oracle):
    """Two c3-shaped interior nodes (2s+32 = 1056 sampled rows x 2s = 1024 candidates, d=8) and a
    leaf (1056 x 512): bit-identical to the reference."""
    from paper_1707_00164_b200 import skeletonize_batch

    rng = np.random.default_rng(5)
    blocks = [gaussian_block(rng, 1056, 1024, 8), gaussian_block(rng, 1056, 512, 8, 1.0, 0.7)]
    ref, _ = oracle.skeletonize_batch(blocks, 512, 1e-5, threads=2)
    st = {}
    got = skeletonize_batch(blocks, 512, 1e-5, stats=st)
    for (k, skel, proj, ach), g in zip(ref, got):
        assert g.rank == k and np.array_equal(g.skel, skel) and np.array_equal(g.proj, proj)
        assert g.achieved_tol == ach
    assert st["kernel_ms"] > 0 and st["bytes"] > 0


def test_skeletonize_errors(gpu):
    from paper_1707_00164_b200 import InvalidArgument, skeletonize_batch

    with pytest.raises(InvalidArgument):
        skeletonize_batch([np.ones((3, 3))], 0, 1e-5)
    with pytest.raises(InvalidArgument):
        skeletonize_batch([np.ones((3, 3))], 4, -1.0)
    assert skeletonize_batch([], 4, 1e-5) == []
