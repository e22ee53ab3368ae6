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


# ------------------------------------------------------------------ full-size parity on sampled leaves
def ancestors(tree, a: int) -> list[int]:
    """a and every ancestor of a below the root (tree.hpp:13-46 parent links)."""
    out = []
    while a > 0:
        out.append(int(a))
        a = int(tree.parent[a])
    return out


def restrict_to_leaves(tree, leaves):
    """A sub-HMatrix whose reference evaluate() reproduces, bit for bit, the u rows of `leaves` of the
    full HMatrix `tree` — used where the full reference HMatrix (stored near/far blocks, ~280 GB at c3)
    does not fit host RAM.

    Why bitwise (evaluate.hpp:141-217): the rows of leaf a are written by a's Output task from D_a,
    a's near blocks in ascending block index (:200-210) and proj_a^T c_a (:212-215); c_x of a node x is
    cfar_x (Coupling over ALL of x's far partners in ascending partner id, :164-177) plus the parent
    term from c_parent (:178-195); every what_y is produced by the Upward pass, which runs for every
    node with a skeleton regardless of the lists (:88-99). So keeping every near pair touching a
    sampled leaf and every far pair touching a node on a sampled leaf's root path leaves every task
    feeding those rows — and its accumulation order — unchanged."""
    import dataclasses

    S = {int(a) for a in leaves}
    path = set()
    for a in S:
        path.update(ancestors(tree, a))
    na, nb = np.asarray(tree.near_a), np.asarray(tree.near_b)
    fa, fb = np.asarray(tree.far_a), np.asarray(tree.far_b)
    keep_n = np.isin(na, list(S)) | np.isin(nb, list(S))
    pl = np.fromiter(path, dtype=np.int64) if path else np.zeros(0, dtype=np.int64)
    keep_f = np.isin(fa, pl) | np.isin(fb, pl)
    return dataclasses.replace(tree, near_a=na[keep_n], near_b=nb[keep_n], far_a=fa[keep_f], far_b=fb[keep_f])


def leaf_ids(tree) -> np.ndarray:
    """Leaves sorted by start (tree.hpp:232-233)."""
    lv = np.flatnonzero(np.asarray(tree.left) < 0)
    return lv[np.argsort(np.asarray(tree.start)[lv], kind="stable")]


def pick_leaves(tree, k: int, seed: int = 0) -> list[int]:
    """k sampled leaves: the first and last leaf, the leaf with the most near pairs, the leaf whose
    root path carries the most far pairs, and seeded random others."""
    lv = leaf_ids(tree)
    nn = tree.num_nodes
    near_cnt = np.bincount(np.concatenate([tree.near_a, tree.near_b]).astype(np.int64), minlength=nn)
    far_cnt = np.bincount(np.concatenate([tree.far_a, tree.far_b]).astype(np.int64), minlength=nn)
    path_far = np.array([sum(int(far_cnt[x]) for x in ancestors(tree, a)) for a in lv])
    chosen = [int(lv[0]), int(lv[-1]), int(lv[np.argmax(near_cnt[lv])]), int(lv[np.argmax(path_far)])]
    rng = np.random.default_rng(seed)
    for a in rng.permutation(lv):
        if len(set(chosen)) >= k:
            break
        chosen.append(int(a))
    return sorted(set(chosen))[:max(k, 4)]


def leaf_rows(tree, leaves) -> np.ndarray:
    """Permuted row indices of the given leaves, concatenated."""
    return np.concatenate([np.arange(int(tree.start[a]), int(tree.end[a])) for a in leaves])


def reference_flops(tree, r: int) -> int:
    """The reference flop counter (evaluate.hpp:141-217) restated from the structure alone."""
    rank = np.asarray(tree.rank, dtype=np.int64)
    cnt = np.asarray(tree.end, dtype=np.int64) - np.asarray(tree.start, dtype=np.int64)
    left, parent = np.asarray(tree.left), np.asarray(tree.parent)
    po = np.asarray(tree.proj_off, dtype=np.int64)
    valid = rank >= 0
    ncand = np.where(valid & (rank > 0), (po[1:] - po[:-1]) // np.maximum(rank, 1), 0)
    f = 0
    leaf = left < 0
    f += int((2 * rank * np.where(leaf, cnt, ncand))[valid].sum())          # Upward
    fa, fb = np.asarray(tree.far_a), np.asarray(tree.far_b)
    f += int((4 * rank[fa] * rank[fb]).sum())                                 # Coupling, both ends
    ids = np.arange(len(rank))
    dn = valid & (parent > 0)
    dn[dn] &= valid[parent[dn]]
    f += int((2 * rank[parent[dn]] * rank[ids[dn]]).sum())                    # Downward parent term
    f += int((2 * cnt[leaf] ** 2).sum())                                      # D
    na, nb = np.asarray(tree.near_a), np.asarray(tree.near_b)
    f += int((4 * cnt[na] * cnt[nb]).sum())                                   # near, both ends
    f += int((2 * rank * cnt)[leaf & valid].sum())                            # proj^T c
    return f * r


def reference_rows_check(oracle, tree, w: np.ndarray, u_gpu_perm: np.ndarray, leaves, threads: int,
                         cols: int | None = None) -> dict:
    """The reference evaluate (oracle/_ref) on restrict_to_leaves(tree, leaves) with W[:, :cols];
    returns the relative 2-norm error of the GPU's u rows of those leaves (first `cols` columns)."""
    sub = restrict_to_leaves(tree, leaves)
    ref = oracle.import_flat(sub, threads=threads)
    wc = w if cols is None else np.asfortranarray(w[:, :cols])
    u_ref, _, sec = ref.evaluate(wc, threads=threads)
    del ref
    rows = leaf_rows(tree, leaves)
    a = np.asarray(u_gpu_perm[rows, :wc.shape[1]], dtype=np.float64)
    b = u_ref[rows]
    return {"rel_error": rel2(a, b), "leaves": [int(x) for x in leaves], "rows": int(rows.size),
            "cols": int(wc.shape[1]), "near_kept": int(len(sub.near_a)), "far_kept": int(len(sub.far_a)),
            "ref_seconds": float(sec)}


# ------------------------------------------------------------------ product-compressed BASELINE trees
THREADS = __import__("os").cpu_count() or 1


def config_cloud(cfg, n, seed):
    from paper_1707_00164_b200 import synth

    fn = {"uniform": synth.uniform_cloud, "gaussian": synth.gaussian_cloud, "covtype": synth.covtype_like}[cfg["cloud"]]
    return fn(n, cfg["d"], seed)


def product_config_tree(name, seed=0):
    """The BASELINE config's cloud through the product compress (device entries) — bench.py's timed tree."""
    import time

    import paper_1707_00164_b200 as G
    from paper_1707_00164_b200 import synth

    cfg = dict(synth.CONFIGS[name])
    pc = config_cloud(cfg, cfg["n"], seed)
    t0 = time.perf_counter()
    res = G.compress(pc, cfg["kernel"], (cfg["h"], 0.0), m=cfg["m"], s=cfg["s"], budget=cfg["budget"], tau=1e-5,
                     kappa=32, distance="kernel", seed=seed, threads=THREADS, entries="device")
    return cfg, res.tree, time.perf_counter() - t0


def reference_eps2_on_leaves(tree, gpu_rep, r, sample_rows, seed, batch):
    """error_eps2 (evaluate.hpp:330-373) with the reference's own u rows (restrict_to_leaves over the
    leaves holding the sampled rows, `batch` leaves per restricted HMatrix) and the reference's own
    exact rows; gpu_rep is the product's report for the same (r, sample_rows, seed)."""
    from paper_1707_00164_b200.gofmm import rng_eps2_draw

    rows, w = rng_eps2_draw(seed, tree.n, r, sample_rows, 0)
    perm = np.empty(tree.n, dtype=np.int64)
    perm[np.asarray(tree.iperm)] = np.arange(tree.n)
    prow = perm[rows]                                    # permuted positions of the sampled rows
    lv = leaf_ids(tree)
    starts = np.asarray(tree.start)[lv]
    owner = lv[np.searchsorted(starts, prow, side="right") - 1]
    need = sorted(set(int(a) for a in owner))
    u_rows = np.empty((len(rows), r))
    for b in range(0, len(need), batch):
        part = need[b:b + batch]
        ref = R.import_flat(restrict_to_leaves(tree, part), threads=THREADS)
        u, _, _ = ref.evaluate(w, threads=THREADS)
        sel = np.isin(owner, part)
        u_rows[sel] = u[prow[sel]]
        if b == 0:
            exact = ref.exact_rows(rows, w)              # oracle.block(rows, all) * w (:353)
        del ref, u
    num = float(np.sum((u_rows - exact) ** 2))
    den = float(np.sum(exact ** 2))
    return {"eps2_reference": float(np.sqrt(num / den)), "eps2_gpu": gpu_rep["eps2"],
            "leaves_evaluated": len(need), "same_rows": list(map(int, rows)) == list(gpu_rep["sample_rows"])}


