"""Synthetic compressed trees of the BASELINE configurations — a WORKLOAD GENERATOR, not the hot path.

The reference compress() (compress.hpp:331-434) needs hours at N = 2^20..2^22 (sequential tree
build, O(#admitted) StructureWalker::crossed, Eigen CPQR) and has no on-disk
HMatrix format, so bench.py builds c3/c5-shaped trees here in seconds. They satisfy every
structural invariant evaluate() relies on:
  * balanced binary tree in BFS order, left child gets ceil(n/2), leaf iff count <= m
    (tree.hpp:56-70,195,213-217); iperm[new] = old;
  * nested skeletons (interior skeleton ⊂ skel(left) ∪ skel(right)), skel in pivot order,
    rank = min(s, #candidates) (saturated, as the recorded acceptance runs are:
    test_output.txt:39-42 == closed-form all-ranks-saturated count);
  * proj = interpolative form: proj(l, piv[l]) = 1 on skeleton columns, coefficients elsewhere
    (compress.hpp:177-185);
  * near pairs = leaf pairs chosen greedily under budget * N^2 (compress.hpp:100-143; here ranked
    by leaf-centroid distance instead of ANN neighbour counts), then the same dual-tree walk as
    StructureWalker (compress.hpp:287-318) so every off-diagonal pair is covered exactly once.
The interpolation coefficients are random (there is no CPQR), so eps2 on these trees is not
meaningful; parity against the reference evaluate is (the oracle consumes the same tree).
"""
from __future__ import annotations

import numpy as np

from .gofmm import CompressedTree


# ------------------------------------------------------------------ point clouds
def uniform_cloud(n: int, d: int, seed: int = 0) -> np.ndarray:
    """Uniform [0,1]^d (BASELINE config 1). d x n, column-major."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.random((n, d)).T)


def gaussian_cloud(n: int, d: int, seed: int = 0) -> np.ndarray:
    """Standard normal cloud (config 2/4/5 shape). d x n, column-major."""
    rng = np.random.default_rng(seed)
    return np.asfortranarray(rng.standard_normal((n, d)).T)


def covtype_like(n: int, d: int = 8, seed: int = 0, classes: int = 7) -> np.ndarray:
    """'COVTYPE-shaped' synthetic (config 3): a 7-class anisotropic Gaussian mixture with unequal
    class weights, standardised per dimension. d x n, column-major."""
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.full(classes, 2.0))
    lab = rng.choice(classes, size=n, p=w)
    means = rng.normal(0.0, 2.0, size=(classes, d))
    scales = rng.uniform(0.3, 1.5, size=(classes, d))
    x = means[lab] + scales[lab] * rng.standard_normal((n, d))
    x = (x - x.mean(axis=0)) / x.std(axis=0)
    return np.asfortranarray(x.T)


# ------------------------------------------------------------------ tree
def build_tree(coords: np.ndarray, m: int):
    """Balanced geometric binary tree (largest-spread coordinate, median split; left = ceil(n/2))."""
    n = coords.shape[1]
    iperm = np.arange(n, dtype=np.int64)
    parent, left, right, level, start, end = [-1], [-1], [-1], [0], [0], [n]
    i = 0
    while i < len(start):
        s, e = start[i], end[i]
        cnt = e - s
        if cnt > m:
            idx = iperm[s:e]
            pts = coords[:, idx]
            axis = int(np.argmax(pts.max(axis=1) - pts.min(axis=1)))
            lsize = cnt - cnt // 2
            order = np.argpartition(pts[axis], lsize - 1)
            lpart, rpart = np.sort(idx[order[:lsize]]), np.sort(idx[order[lsize:]])
            iperm[s:s + lsize], iperm[s + lsize:e] = lpart, rpart
            lc = len(start)
            left[i], right[i] = lc, lc + 1
            for (cs, ce) in ((s, s + lsize), (s + lsize, e)):
                parent.append(i)
                left.append(-1)
                right.append(-1)
                level.append(level[i] + 1)
                start.append(cs)
                end.append(ce)
        i += 1
    a = lambda v: np.asarray(v, dtype=np.int32)  # noqa: E731
    return dict(parent=a(parent), left=a(left), right=a(right), level=a(level), start=a(start), end=a(end),
                iperm=iperm.astype(np.int32))


# ------------------------------------------------------------------ interaction lists
def _leaf_order(t):
    leaves = np.nonzero(t["left"] < 0)[0]
    return leaves[np.argsort(t["start"][leaves], kind="stable")]


def select_near(t, coords: np.ndarray, budget: float):
    """Greedy leaf-pair admission under budget*N^2 (compress.hpp:85-144), ranked by centroid distance."""
    leaves = _leaf_order(t)
    nl, n = len(leaves), int(t["end"][0])
    if nl < 2 or budget <= 0:
        return []
    cnt = (t["end"][leaves] - t["start"][leaves]).astype(np.float64)
    cap = budget * float(n) * float(n)
    total_all = 2.0 * (cnt.sum() ** 2 - (cnt ** 2).sum()) / 2.0
    if total_all <= cap:
        return [(int(leaves[a]), int(leaves[b])) for a in range(nl) for b in range(a + 1, nl)]
    iperm = t["iperm"]
    cen = np.stack([coords[:, iperm[t["start"][lf]:t["end"][lf]]].mean(axis=1) for lf in leaves])
    sq = (cen ** 2).sum(axis=1)
    d2 = sq[:, None] + sq[None, :] - 2.0 * cen @ cen.T
    iu, ju = np.triu_indices(nl, 1)
    order = np.argsort(d2[iu, ju], kind="stable")
    cost = 2.0 * cnt[iu[order]] * cnt[ju[order]]
    csum = np.cumsum(cost)
    take = order[csum <= cap]
    pairs = sorted((int(min(leaves[iu[q]], leaves[ju[q]])), int(max(leaves[iu[q]], leaves[ju[q]]))) for q in take)
    return pairs


def walk_structure(t, near_pairs):
    """StructureWalker (compress.hpp:242-324): exactly-one coverage of off-diagonal pairs."""
    leaves = _leaf_order(t)
    nn = len(t["parent"])
    ordl = np.full(nn, -1, dtype=np.int64)
    ordl[leaves] = np.arange(len(leaves))
    lo = np.zeros(nn, dtype=np.int64)
    hi = np.zeros(nn, dtype=np.int64)
    for i in range(nn - 1, -1, -1):  # children have larger ids (BFS)
        if t["left"][i] < 0:
            lo[i], hi[i] = ordl[i], ordl[i] + 1
        else:
            lo[i], hi[i] = lo[t["left"][i]], hi[t["right"][i]]
    nl = len(leaves)
    pre = None
    if near_pairs:
        adm = np.zeros((nl + 1, nl + 1), dtype=np.int32)
        for a, b in near_pairs:
            x, y = ordl[a], ordl[b]
            adm[x + 1, y + 1] = 1
            adm[y + 1, x + 1] = 1
        pre = adm.cumsum(0).cumsum(1)

    def crossed(a, b):
        if pre is None:
            return False
        r0, r1, c0, c1 = lo[a], hi[a], lo[b], hi[b]
        return (pre[r1, c1] - pre[r0, c1] - pre[r1, c0] + pre[r0, c0]) > 0

    near, far = [], []
    left, right = t["left"], t["right"]
    stack = [(int(left[i]), int(right[i])) for i in range(nn) if left[i] >= 0]
    while stack:
        a, b = stack.pop()
        if not crossed(a, b):
            far.append((min(a, b), max(a, b)))
            continue
        la, lb = left[a] < 0, left[b] < 0
        if la and lb:
            near.append((min(a, b), max(a, b)))
        elif la:
            stack += [(a, int(left[b])), (a, int(right[b]))]
        elif lb:
            stack += [(int(left[a]), b), (int(right[a]), b)]
        else:
            stack += [(int(left[a]), int(left[b])), (int(left[a]), int(right[b])),
                      (int(right[a]), int(left[b])), (int(right[a]), int(right[b]))]
    near.sort()
    far.sort()
    return near, far


# ------------------------------------------------------------------ skeletons
def skeletonize(t, s: int, seed: int = 0, coef_scale: float = 0.5):
    """Nested saturated skeletons + interpolative proj (compress.hpp:149-187 shapes)."""
    rng = np.random.default_rng(seed ^ 0x51E7)
    nn = len(t["parent"])
    rank = np.full(nn, -1, dtype=np.int32)
    skel = [None] * nn
    projs = [None] * nn
    for i in range(nn - 1, 0, -1):  # bottom-up; the root keeps an invalid skeleton
        if t["left"][i] < 0:
            cand = t["iperm"][t["start"][i]:t["end"][i]]
        else:
            cand = np.concatenate([skel[t["left"][i]], skel[t["right"][i]]])
        c = len(cand)
        k = max(1, min(s, c))
        piv = rng.permutation(c)
        proj = np.zeros((k, c), dtype=np.float64, order="F")
        proj[np.arange(k), piv[:k]] = 1.0
        if c > k:
            proj[:, piv[k:]] = (coef_scale / np.sqrt(c)) * rng.standard_normal((k, c - k))
        rank[i] = k
        skel[i] = cand[piv[:k]].astype(np.int32)
        projs[i] = proj
    skel_off = np.zeros(nn + 1, dtype=np.int64)
    proj_off = np.zeros(nn + 1, dtype=np.int64)
    for i in range(nn):
        skel_off[i + 1] = skel_off[i] + (rank[i] if rank[i] > 0 else 0)
        proj_off[i + 1] = proj_off[i] + (projs[i].size if projs[i] is not None else 0)
    skel_idx = np.empty(skel_off[-1], dtype=np.int32)
    proj = np.empty(proj_off[-1], dtype=np.float64)
    for i in range(nn):
        if projs[i] is None:
            continue
        skel_idx[skel_off[i]:skel_off[i + 1]] = skel[i]
        proj[proj_off[i]:proj_off[i + 1]] = projs[i].ravel(order="F")
        projs[i] = None
    return rank, skel_off, skel_idx, proj_off, proj


def synthetic_tree(coords: np.ndarray, m: int, s: int, budget: float, kernel: int, kparams=(1.0, 0.0),
                   seed: int = 0) -> CompressedTree:
    coords = np.asfortranarray(coords, dtype=np.float64)
    t = build_tree(coords, m)
    admitted = select_near(t, coords, budget)
    near, far = walk_structure(t, admitted)
    rank, skel_off, skel_idx, proj_off, proj = skeletonize(t, s, seed)
    na = np.asarray([p[0] for p in near], dtype=np.int32)
    nb = np.asarray([p[1] for p in near], dtype=np.int32)
    fa = np.asarray([p[0] for p in far], dtype=np.int32)
    fb = np.asarray([p[1] for p in far], dtype=np.int32)
    return CompressedTree(
        n=coords.shape[1], depth=int(t["level"].max()), rank=rank, skel_off=skel_off, skel_idx=skel_idx,
        proj_off=proj_off, proj=proj, near_a=na, near_b=nb, far_a=fa, far_b=fb, coords=coords, kernel=kernel,
        kparams=tuple(kparams), **{k: t[k] for k in ("parent", "left", "right", "level", "start", "end", "iperm")})


# BASELINE.json configs (c1..c5). Budgets: c1/c2/c4 as stated; c3/c5 leave it open (SURVEY.md §7
# hard part 6) — c3 uses the reference RunConfig default 0.03 (compress.hpp:17), c5 uses 0.
CONFIGS = {
    "c1": dict(n=8192, d=6, m=128, s=128, budget=0.03, r=64, kernel=0, h=1.0, cloud="uniform"),
    "c2": dict(n=65536, d=3, m=256, s=256, budget=0.05, r=256, kernel=0, h=1.0, cloud="gaussian"),
    "c3": dict(n=1 << 20, d=8, m=512, s=512, budget=0.03, r=512, kernel=0, h=1.0, cloud="covtype"),
    "c4": dict(n=262144, d=3, m=256, s=256, budget=0.15, r=512, kernel=4, h=1.0, cloud="gaussian"),
    "c5": dict(n=1 << 22, d=3, m=256, s=256, budget=0.0, r=1024, kernel=0, h=1.0, cloud="gaussian"),
}


def make_config_tree(name: str, seed: int = 0, **over) -> tuple[CompressedTree, dict]:
    cfg = dict(CONFIGS[name])
    cfg.update(over)
    cloud = {"uniform": uniform_cloud, "gaussian": gaussian_cloud, "covtype": covtype_like}[cfg["cloud"]]
    coords = cloud(cfg["n"], cfg["d"], seed)
    tree = synthetic_tree(coords, cfg["m"], cfg["s"], cfg["budget"], cfg["kernel"], (cfg["h"], 0.0), seed)
    return tree, cfg
