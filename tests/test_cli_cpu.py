"""CPU tests of the command-line driver (paper_1707_00164_b200/_lib/gofmm_b200_cli, csrc/gofmm_cli.cpp):
the reference CLI's exit-code contract for bad flags and bad files (tests/test_cli.cpp:106-126), which
fires before any device work."""
import os
import subprocess

import pytest

from paper_1707_00164_b200 import _lib

CLI = _lib.CLI_PATH


def run(args, **kw):
    return subprocess.run([CLI, *args.split()], capture_output=True, text=True, timeout=60, **kw)


@pytest.fixture(scope="module", autouse=True)
def built():
    _lib.build()
    assert os.access(CLI, os.X_OK)


@pytest.mark.parametrize("args", [
    "compress --gen nope --n 64",
    "compress --n 64",                       # no source
    "compress --gen gaussian --n 64 --budget 2",
    "compress --gen gaussian --n 64 --mode sideways",
    "compress --gen invsqlap --n 63",
    "compress --gen gaussian --n 64 --dist diagonal",
    "frobnicate",
    "",
    "compress --gen gaussian --n 64 --s 300 --m 256",  # s > m (RunConfig::validate)
    "compress --gen gaussian --n 64 --r 0",
    "bench --gen gaussian --n-list 128,x",
    "compress --gen gaussian --n 64 --seed abc",
])
def test_bad_flags_exit_2(args):
    assert run(args).returncode == 2


def test_missing_or_malformed_files_exit_3(tmp_path):
    assert run("compress --matrix /no/such/file.bin --m 16 --s 16").returncode == 3
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXX garbage")
    assert run(f"compress --matrix {bad}").returncode == 3
    assert run(f"compress --gen gaussian --points {bad}").returncode == 3
    assert run("compress --gen gaussian --points /no/such/points.bin").returncode == 3
