"""The command-line driver (csrc/gofmm_cli.cpp) on the GPU: the reference CLI's own tests
(proj/tests/test_cli.cpp) restated, plus the report's values against the reference compress() +
error_eps2() (oracle/_ref) for --entries host (the bit-identical compress)."""
import subprocess

import numpy as np
import pytest

from paper_1707_00164_b200 import _lib

pytestmark = pytest.mark.gpu
CLI = _lib.CLI_PATH


def run(args):
    p = subprocess.run([CLI, *args.split()], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout


def keys_in_order(out):
    return [ln.split("=", 1)[0] for ln in out.splitlines() if "=" in ln]


def value_of(out, key):
    for ln in out.splitlines():
        if ln.startswith(key + "="):
            return ln[len(key) + 1:]
    return ""


def test_compress_report_keys_in_order(gpu):
    """test_cli.cpp:61-80."""
    rc, out = run("compress --gen gaussian --n 512 --d 2 --h 3 --m 64 --s 64 --k 8 --budget 0.03 --dist kernel "
                  "--seed 1 --iters 3")
    assert rc == 0, out
    assert keys_in_order(out) == [
        "ann_recall_iter_1", "ann_recall_iter_2", "ann_recall_iter_3", "tree_seconds", "entries_evaluated",
        "compress_flops", "compress_seconds", "near_field_entries", "max_skeleton", "mean_skeleton", "eval_flops",
        "eval_seconds", "eps2", "eps2_first10", "eps2_mean100"]
    assert float(value_of(out, "eps2")) <= 1e-2
    assert int(value_of(out, "entries_evaluated")) > 0
    assert value_of(out, "eps2_first10").count(",") == 9


def test_zero_budget_empty_near_field(gpu):
    rc, out = run("compress --gen gaussian --n 256 --d 2 --m 32 --s 32 --budget 0 --seed 2")
    assert rc == 0 and value_of(out, "near_field_entries") == "0"


@pytest.mark.parametrize("entries", ["host", "device"])
def test_reproducible_and_modes_identical(gpu, entries):
    base = f"compress --gen gaussian --n 400 --d 3 --m 32 --s 32 --seed 4 --entries {entries}"
    a, b = run(base + " --mode levels"), run(base + " --mode tasks")
    c = run(base + " --threads 2")
    assert a[0] == b[0] == c[0] == 0
    for k in ("eps2", "entries_evaluated", "eval_flops", "eps2_first10"):
        assert value_of(a[1], k) == value_of(b[1], k) == value_of(c[1], k), k


def test_numeric_degeneracy_exit_4(gpu, tmp_path):
    """Duplicate points with a zero Laplace floor make the kernel singular (test_cli.cpp:128-138)."""
    import struct

    pts = tmp_path / "dup.pts"
    pts.write_bytes(b"GPTS" + struct.pack("<IQQ", 1, 32, 3) + bytes(8 * 32 * 3))
    rc, _ = run(f"compress --gen laplace --points {pts} --delta 0 --m 8 --s 8")
    assert rc == 4


def test_bench_csv(gpu):
    rc, out = run("bench --gen gaussian --d 2 --m 32 --s 32 --n-list 128,256 --r-list 4 --seed 1")
    assert rc == 0, out
    lines = [ln for ln in out.splitlines() if ln]
    assert lines[0] == "N,r,dense_seconds,compress_seconds,eval_seconds,speedup"
    assert len(lines) == 3 and all(ln.count(",") == 5 for ln in lines[1:])
    assert run("bench --gen gaussian --n-list 20000 --r-list 1")[0] == 3  # desk-scale cap (io_error)


def test_f32_rounds_reported_errors(gpu):
    args = "compress --gen gaussian --n 128 --d 2 --m 32 --s 32 --seed 6"
    base, f32 = run(args), run(args + " --f32")
    assert base[0] == f32[0] == 0
    assert float(value_of(f32[1], "eps2")) == pytest.approx(float(np.float32(float(value_of(base[1], "eps2")))),
                                                             rel=1e-5)


@pytest.mark.parametrize("gen,extra,kernel", [("gaussian", "--h 1.5", "GAUSSIAN"), ("laplace", "", "LAPLACE"),
                                              ("poly", "--shift 1 --degree 2", "POLYNOMIAL")])
def test_report_matches_reference(gpu, oracle, gen, extra, kernel):
    """--entries host: every compress statistic equals the reference compress's, and eval_flops / eps2
    equal the reference error_eps2's (6 significant digits, as both print)."""
    R = oracle
    n, d, seed = 2000, 3, 11
    rc, out = run(f"compress --gen {gen} {extra} --n {n} --d {d} --m 64 --s 48 --k 16 --budget 0.05 --seed {seed} "
                  f"--r 2 --threads 4 --entries host")
    assert rc == 0, out
    pc = np.asfortranarray(R.points_gaussian(n, d, seed))
    p0, p1 = {"gaussian": (1.5, 0.0), "laplace": (-1.0, 0.0), "poly": (1.0, 2.0)}[gen]
    if gen == "laplace":
        p0 = R.default_laplace_floor(pc, seed)
    h = R.compress_kernel(getattr(R, kernel), pc, p0, p1, m=64, s=48, tau=1e-5, kappa=16, budget=0.05, seed=seed,
                          threads=4)
    st = h.compress_stats()
    for k in ("entries_evaluated", "compress_flops", "near_field_entries", "max_skeleton"):
        assert int(value_of(out, k)) == st[k], k
    assert value_of(out, "mean_skeleton") == f"{st['mean_skeleton']:g}"
    rep = h.error_eps2(2, 100, seed, threads=4)
    assert int(value_of(out, "eval_flops")) == rep["eval_flops"]
    assert float(value_of(out, "eps2")) == pytest.approx(rep["eps2"], rel=2e-6)

