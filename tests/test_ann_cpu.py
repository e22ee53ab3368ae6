"""CPU side of the ANN leaf pass: the oracle's reference ann_iteration and
random-tree leaves behave as neighbors.hpp documents (sorted, self-free, duplicate-free lists;
leaves partition the indices), and the GPU entry point fails loudly without a device."""
import numpy as np
import pytest


def test_reference_ann_tables(oracle):
    coords = oracle.points_gaussian(800, 3, 2)
    n, k = 800, 10
    tj, td, tl = np.full((n, k), -1, np.int32), np.zeros((n, k)), np.zeros(n, np.int32)
    for seed in (1, 2):
        oracle.ann_iteration(coords, 0, 1.0, k, 64, seed, tj, td, tl)
        off, idx = oracle.ann_leaves(coords, 0, 1.0, 64, seed)
        assert np.array_equal(np.sort(idx), np.arange(n))          # leaves partition the indices
        assert np.all(np.diff(off) > 0)
    for i in range(n):
        js, ds = tj[i, :tl[i]], td[i, :tl[i]]
        assert i not in js and len(set(js.tolist())) == len(js)
        assert np.all(np.diff(ds) >= 0)
        exact = np.linalg.norm(coords[:, js] - coords[:, [i]], axis=0)
        assert np.allclose(ds, exact, rtol=1e-14)


def test_gpu_ann_no_cpu_fallback():
    import torch

    from paper_1707_00164_b200 import GofmmError, ann_leaf_merge

    if torch.cuda.is_available():
        pytest.skip("a device is present; tests/test_ann_gpu.py covers the GPU path")
    tj, td, tl = np.zeros((10, 4), np.int32), np.zeros((10, 4)), np.zeros(10, np.int32)
    with pytest.raises(GofmmError) as e:
        ann_leaf_merge(np.zeros((3, 10)), 0, 1.0, 4, np.array([0, 10]), np.arange(10), tj, td, tl)
    assert e.value.code == 5
