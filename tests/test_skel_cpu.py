"""CPU side of the batched skeletonisation: the oracle's reference
skeletonize_node on given blocks honours the ID contract of compress.hpp:149-187, and the GPU
entry point fails loudly (never computes on the CPU) when no device is present."""
import numpy as np
import pytest


def test_reference_skeletonize_exact_low_rank(oracle):
    rng = np.random.default_rng(2)
    b = rng.standard_normal((70, 9)) @ rng.standard_normal((9, 45))
    (k, skel, proj, ach), = oracle.skeletonize_batch([b], 32, 1e-10)[0]
    assert k == 9 and len(set(skel.tolist())) == 9
    assert np.allclose(proj[:, skel], np.eye(9))               # proj(l, perm[l]) = 1
    assert np.linalg.norm(b - b[:, skel] @ proj) <= 1e-10 * np.linalg.norm(b)
    assert ach < 1e-10


def test_reference_skeletonize_clamps_rank(oracle):
    rng = np.random.default_rng(3)
    out, _ = oracle.skeletonize_batch([rng.standard_normal((20, 15)), np.zeros((6, 4))], 5, 0.0)
    assert out[0][0] == 5          # clamp to s (compress.hpp:170)
    assert out[1][0] == 1          # all-zero block: clamp to 1, lead = 0 so proj is the unit pivot row
    assert out[1][2].shape == (1, 4)


def test_gpu_skeletonize_no_cpu_fallback():
    import torch

    from paper_1707_00164_b200 import GofmmError, skeletonize_batch

    if torch.cuda.is_available():
        pytest.skip("a device is present; tests/test_skel_gpu.py covers the GPU path")
    with pytest.raises(GofmmError) as e:
        skeletonize_batch([np.ones((4, 3))], 2, 1e-5)
    assert e.value.code == 5
