"""The drop-in boundary's contract beyond single-call parity:
* concurrent evaluate() calls on one HMatrix with different w are allowed: host
  threads calling the host-buffer API, and device-buffer calls on different CUDA streams, give
  results bitwise equal to the same calls made one after another;
* a subtree-split handle (nranks > 1) is rejected by the whole-matrix entry points;
* a caller-supplied device `out` is validated (shape, dtype, device, layout) before any launch;
* the in-library data plane (gofmm_dist_evaluate: stage 1 -> ncclAllGather -> stage 2, with the
  own D + near output terms overlapping the all-gather) on a one-rank NCCL communicator equals
  the single-GPU evaluation bitwise; a multi-rank handle without a communicator is rejected."""
import threading

import numpy as np
import pytest

from tests._util import rel2, to_tree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tree_and_ref(oracle):
    pc = oracle.points_gaussian(3000, 3, 21)
    h = oracle.compress_kernel(oracle.GAUSSIAN, pc, 1.0, m=128, s=64, tau=1e-7, kappa=16, budget=0.05, seed=4,
                               threads=8)
    return to_tree(h.export()), h


def test_concurrent_host_calls_bitwise_equal_serial(gpu, oracle, tree_and_ref):
    tree, h = tree_and_ref
    ws = [oracle.rng_gauss(tree.n, r, 50 + r) for r in (3, 17, 64, 130)]
    with gpu.Evaluator(tree) as ev:
        serial = [ev.evaluate(w).u.copy() for w in ws]
        out = [[None] * 3 for _ in ws]
        errs = []

        def work(i):
            try:
                for rep in range(3):
                    out[i][rep] = ev.evaluate(ws[i]).u
            except Exception as e:  # surfaced below
                errs.append(e)

        th = [threading.Thread(target=work, args=(i,)) for i in range(len(ws))]
        for t in th:
            t.start()
        for t in th:
            t.join()
    assert not errs, errs
    for i, w in enumerate(ws):
        for rep in range(3):
            assert np.array_equal(out[i][rep], serial[i]), (i, rep)
    u_ref, _, _ = h.evaluate(ws[1])
    assert rel2(serial[1], u_ref) <= 1e-12


def test_concurrent_device_calls_on_two_streams(gpu, oracle, tree_and_ref):
    """Device-buffer evaluations enqueued on two streams race on nothing: the handle's workspace
    is handed from one enqueue to the next by an event, whatever stream each was issued on."""
    import torch

    tree, _ = tree_and_ref
    ws = [torch.from_numpy(np.ascontiguousarray(oracle.rng_gauss(tree.n, 40, 70 + i).T)).cuda().t() for i in range(2)]
    with gpu.Evaluator(tree) as ev:
        ref = []
        for w in ws:
            u, _ = ev.evaluate_torch(w)
            torch.cuda.synchronize()
            ref.append(u.cpu().numpy())
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        outs = [[torch.empty((40, tree.n), dtype=torch.float64, device="cuda").t() for _ in range(4)] for _ in ws]
        torch.cuda.synchronize()
        for rep in range(4):  # interleave: A on s0, B on s1, A on s0 ...
            for i, w in enumerate(ws):
                with torch.cuda.stream(streams[i]):
                    ev.evaluate_torch(w, out=outs[i][rep])
        torch.cuda.synchronize()
    for i in range(2):
        for rep in range(4):
            assert np.array_equal(outs[i][rep].cpu().numpy(), ref[i]), (i, rep)


def test_dist_handle_rejected_by_whole_matrix_entry_points(gpu, oracle, tree_and_ref):
    import torch

    tree, _ = tree_and_ref
    w = oracle.rng_gauss(tree.n, 2, 1)
    with gpu.Evaluator(tree, rank=0, nranks=2) as ev:
        with pytest.raises(gpu.InvalidArgument) as e:
            ev.evaluate(w)
        assert "subtree split" in str(e.value)
        wd = torch.from_numpy(np.ascontiguousarray(w.T)).cuda().t()
        with pytest.raises(gpu.InvalidArgument):
            ev.evaluate_torch(wd)
        out = torch.empty((2, tree.n), dtype=torch.float64, device="cuda").t()
        with pytest.raises(gpu.InvalidArgument) as e:  # no communicator attached
            ev.dist_evaluate_torch(wd, out)
        assert "communicator" in str(e.value)


def test_device_out_validation(gpu, oracle, tree_and_ref):
    import torch

    tree, _ = tree_and_ref
    w = torch.from_numpy(np.ascontiguousarray(oracle.rng_gauss(tree.n, 8, 2).T)).cuda().t()
    with gpu.Evaluator(tree) as ev:
        bad = [torch.empty((8, tree.n), dtype=torch.float32, device="cuda").t(),  # dtype
               torch.empty((4, tree.n), dtype=torch.float64, device="cuda").t(),  # too few columns
               torch.empty((tree.n, 8), dtype=torch.float64, device="cuda"),     # row-major
               torch.empty((8, tree.n), dtype=torch.float64).t()]                # host tensor
        for out in bad:
            with pytest.raises(gpu.InvalidArgument):
                ev.evaluate_torch(w, out=out)
        with pytest.raises(gpu.InvalidArgument):  # too many rows: the reference throws, no truncation
            ev.evaluate_torch(torch.zeros((tree.n + 1, 2), dtype=torch.float64, device="cuda"))


def test_library_nccl_data_plane_single_rank(gpu, oracle, tree_and_ref):
    """gofmm_dist_evaluate on a one-rank NCCL communicator created by the library from a unique
    id (the multi-rank path differs only in the all-gather's rank count)."""
    import torch

    from paper_1707_00164_b200 import gofmm

    tree, h = tree_and_ref
    w_np = oracle.rng_gauss(tree.n, 33, 9)
    w = torch.from_numpy(np.ascontiguousarray(w_np.T)).cuda().t()
    with gpu.Evaluator(tree) as ev:
        single, _ = ev.evaluate_torch(w)
        torch.cuda.synchronize()
        single = single.cpu().numpy()
    with gpu.Evaluator(tree, rank=0, nranks=1) as ev:
        ev.init_comm(gofmm.nccl_unique_id())
        out = torch.full((33, tree.n), float("nan"), dtype=torch.float64, device="cuda").t()
        t = ev.dist_evaluate_torch(w, out, timed=True)
        torch.cuda.synchronize()
        assert t["total_ms"] > 0
        assert np.array_equal(out.cpu().numpy(), single)
        ev.dist_evaluate_torch(w, out)  # untimed, repeated
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), single)
