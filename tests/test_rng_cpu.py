"""error_eps2's draws (evaluate.hpp:336-346, Rng common.hpp:40-104) restated in the C-ABI, incl.
the redraws: W of attempt a continues the same stream after attempts 0..a-1 (evaluate.hpp:343-372),
so it equals columns [a*r, (a+1)*r) of a single (a+1)*r-column draw by the reference. Host code
only (no device needed)."""
import numpy as np
import pytest

from paper_1707_00164_b200 import gofmm


@pytest.mark.parametrize("n,r,rows,seed", [(500, 3, 100, 42), (64, 2, 100, 7), (1000, 1, 37, 11)])
def test_eps2_draw_attempts_follow_reference_stream(oracle, n, r, rows, seed):
    ref_rows, ref_w = oracle.eps2_draw(n, 3 * r, rows, seed)
    for a in range(3):
        got_rows, got_w = gofmm.rng_eps2_draw(seed, n, r, rows, attempt=a)
        assert np.array_equal(got_rows, ref_rows)
        assert np.array_equal(got_w, ref_w[:, a * r:(a + 1) * r])


def test_eps2_draw_rejects_bad_attempt():
    from paper_1707_00164_b200 import InvalidArgument

    with pytest.raises(InvalidArgument):
        gofmm.rng_eps2_draw(1, 10, 1, 5, attempt=3)


# ------------------------------------------------------------------ the CLI's point sources (host C-ABI)
def _lib():
    from paper_1707_00164_b200 import _lib

    return _lib.lib()


@pytest.mark.parametrize("n,d,seed", [(100, 3, 0), (513, 6, 42), (7, 1, 9)])
def test_points_gaussian_matches_reference(oracle, n, d, seed):
    """PointCloud::random_gaussian (oracle.hpp:18-25)."""
    import ctypes as C

    out = np.empty((d, n), order="F")
    assert _lib().gofmm_points_gaussian(n, d, seed, out.ctypes.data_as(C.c_void_p)) == 0
    assert np.array_equal(out, oracle.points_gaussian(n, d, seed))


@pytest.mark.parametrize("n,d,seed", [(2000, 3, 0), (2000, 3, 11), (50, 6, 4), (1, 2, 0)])
def test_default_laplace_floor_matches_reference(oracle, n, d, seed):
    """default_laplace_floor (oracle.hpp:274-288), bit for bit."""
    import ctypes as C

    pc = oracle.points_gaussian(n, d, seed + 1)
    got = C.c_double()
    assert _lib().gofmm_default_laplace_floor(d, n, pc.ctypes.data_as(C.c_void_p), seed, C.byref(got)) == 0
    assert got.value == oracle.default_laplace_floor(pc, seed)


@pytest.mark.parametrize("seed,stream", [(1, 0xbe7c), (0, 0), (5, 0x9f)])
def test_rng_gauss_stream_matches_reference(oracle, seed, stream):
    import ctypes as C

    n, r = 300, 3
    w = np.empty((n, r), order="F")
    assert _lib().gofmm_rng_gauss_stream(seed, stream, n, r, w.ctypes.data_as(C.c_void_p), n) == 0
    assert np.array_equal(w, oracle.rng_gauss(n, r, seed, stream))
