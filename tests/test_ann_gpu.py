"""GPU ANN leaf pass vs the reference ann_iteration (neighbors.hpp:88-106,
compiled unmodified in the oracle) on the same random trees and tables. Geometric distances:
bit-identical tables. Kernel distances (Gaussian entries through the device exp, <= 1-2 ulp from
glibc's): same list lengths, distances to 1e-14 relative, neighbor sets equal except at ties."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_both(oracle, ann_leaf_merge, coords, kind, h, kappa, m, seeds):
    d, n = coords.shape
    k = min(kappa, n - 1)  # NeighborTable::k
    ref = [np.full((n, k), -1, np.int32), np.zeros((n, k)), np.zeros(n, np.int32)]
    gpu = [a.copy() for a in ref]
    for seed in seeds:
        oracle.ann_iteration(coords, kind, h, k, m, seed, *ref, threads=4)
        off, idx = oracle.ann_leaves(coords, kind, h, m, seed)
        ann_leaf_merge(coords, kind, h, k, off, idx, *gpu)
    return ref, gpu


@pytest.mark.parametrize("d,n,m,kappa", [(3, 3000, 128, 16), (8, 2500, 256, 32), (6, 700, 64, 8), (5, 300, 40, 12)])
def test_ann_geometric_bitwise(gpu, oracle, d, n, m, kappa):
    from paper_1707_00164_b200 import ann_leaf_merge

    coords = oracle.points_gaussian(n, d, 17 + d)
    ref, got = run_both(oracle, ann_leaf_merge, coords, 0, 1.0, kappa, m, [11, 12, 13])
    assert np.array_equal(ref[2], got[2])
    assert np.array_equal(ref[0], got[0])
    assert np.array_equal(ref[1], got[1])
    assert (ref[2] == min(kappa, n - 1)).mean() > 0.5


def test_ann_kernel_metric(gpu, oracle):
    from paper_1707_00164_b200 import ann_leaf_merge

    coords = oracle.points_gaussian(3000, 3, 5)
    ref, got = run_both(oracle, ann_leaf_merge, coords, 1, 1.0, 16, 128, [21, 22])
    assert np.array_equal(ref[2], got[2])
    mask = np.arange(16)[None, :] < ref[2][:, None]
    assert np.allclose(got[1][mask], ref[1][mask], rtol=1e-14, atol=1e-15)
    same = [set(ref[0][i, :ref[2][i]]) == set(got[0][i, :got[2][i]]) for i in range(3000)]
    assert np.mean(same) >= 0.99


def test_ann_errors(gpu):
    from paper_1707_00164_b200 import InvalidArgument, ann_leaf_merge

    c = np.zeros((3, 10))
    tj, td, tl = np.zeros((10, 4), np.int32), np.zeros((10, 4)), np.zeros(10, np.int32)
    with pytest.raises(InvalidArgument):
        ann_leaf_merge(c, 0, 1.0, 40, np.array([0, 10]), np.arange(10), tj, td, tl)  # kappa > 32
    with pytest.raises(InvalidArgument):
        ann_leaf_merge(c, 2, 1.0, 4, np.array([0, 10]), np.arange(10), tj, td, tl)   # unknown kind
