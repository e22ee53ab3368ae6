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
