"""The header-only C++ adapter (include/gofmm_b200_gfmm.hpp) over the reference API, compiled with
the reference headers into oracle/_ref/adapter_test (oracle/Makefile, target `adapter`): the
reference's own compress() + evaluate() + error_eps2() next to the adapter on the same HMatrix —
gfmm::evaluate_b200(h, w, opts) (evaluate()'s signature, cached per HMatrix), the stored and the
matrix-free evaluators (Gaussian, Laplace, Exponential) within 1e-12 with equal flop counters,
error_eps2_b200 == error_eps2, the distributed evaluator (B200Evaluator::distributed +
evaluate_dist over gofmm_dist_evaluate_host) on one rank, 4 threads calling evaluate_b200 on one HMatrix concurrently
bitwise equal to serial calls, and std::invalid_argument on a wrong-sized W
(evaluate.hpp:288-289)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


@pytest.mark.parametrize("n,r", [(2048, 16), (3000, 5)])
def test_cpp_adapter_matches_reference_evaluate(gpu, n, r):
    assert os.path.exists(BIN), "oracle/_ref/adapter_test missing (make -C oracle adapter where /root/reference exists)"
    p = subprocess.run([BIN, str(n), str(r)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "ok=1" in p.stdout, p.stdout
