"""Shared helpers for the parity tests (test infrastructure; may import oracle/)."""
from __future__ import annotations

import numpy as np

from oracle import refpy as R
from paper_1707_00164_b200 import CompressedTree


def to_tree(flat) -> CompressedTree:
    """oracle Flat export -> product CompressedTree (same field names)."""
    return CompressedTree.from_any(flat)


def rel2(a: np.ndarray, b: np.ndarray) -> float:
    """relative 2-norm (Frobenius) error ||a-b|| / ||b|| (north_star: 1e-12 fp64)."""
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def uniform_points(n: int, d: int, seed: int) -> np.ndarray:
    """Uniform [0,1]^d cloud (BASELINE config 1) from the reference RNG stream layout:
    Rng(seed, 0x9f), point-major fill like PointCloud::random_gaussian (oracle.hpp:18-25)."""
    g = R.rng_gauss(1, 1, seed)  # touch the library (build check)
    del g
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.random((d, n)))
