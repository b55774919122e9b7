"""Synthetic instance generators for the benchmark configurations.

Raw COO (u, v, cost) as numpy arrays, before canonicalisation; feed them
to ``WeightedGraph`` (which canonicalises on the GPU) or to the oracle.
Shapes follow SURVEY.md section 8(d); C1 and C5 are exactly
``parcut.grid_graph`` (generate.py:28-62) and ``random_graph`` mirrors
generate.py:8-25.
"""

import numpy as np


def grid_coo(height, width, stride=0, seed=0):
    """parcut.grid_graph (generate.py:28-62): 4-connected row-major grid,
    optional coarse lattice edges (right block, then down block)."""
    if height < 1 or width < 1:
        raise ValueError("grid dimensions must be positive")
    if stride < 0 or stride == 1:
        raise ValueError("stride must be 0 (disabled) or at least 2")
    ids = np.arange(height * width, dtype=np.int64).reshape(height, width)
    us = [ids[:, :-1].ravel(), ids[:-1, :].ravel()]
    vs = [ids[:, 1:].ravel(), ids[1:, :].ravel()]
    if stride >= 2:
        r, c = np.meshgrid(np.arange(0, height, stride), np.arange(0, width, stride), indexing="ij")
        ok = c + stride < width
        us.append(ids[r[ok], c[ok]])
        vs.append(ids[r[ok], c[ok] + stride])
        ok = r + stride < height
        us.append(ids[r[ok], c[ok]])
        vs.append(ids[r[ok] + stride, c[ok]])
    u, v = np.concatenate(us), np.concatenate(vs)
    cost = np.random.default_rng(seed).standard_normal(u.size)
    return height * width, u, v, cost


def random_coo(num_nodes, p, seed=0):
    """parcut.random_graph (generate.py:8-25): Erdos-Renyi, N(0,1) costs."""
    if num_nodes < 0:
        raise ValueError("num_nodes must be non-negative")
    if not (0.0 <= p <= 1.0):
        raise ValueError("edge_probability must be in [0, 1]")
    rng = np.random.default_rng(seed)
    iu, iv = np.triu_indices(num_nodes, k=1)
    keep = rng.random(iu.size) < p
    u, v = iu[keep].astype(np.int64), iv[keep].astype(np.int64)
    return num_nodes, u, v, rng.standard_normal(u.size)


def grid8_coo(height=1024, width=2048, strides=(2, 3), seed=0):
    """C2: 8-connected row-major grid + coarse lattice edges at each stride
    (down block, then right block).  1024x2048 -> 9,892,581 edges."""
    ids = np.arange(height * width, dtype=np.int64).reshape(height, width)
    us = [ids[:, :-1].ravel(), ids[:-1, :].ravel(), ids[:-1, :-1].ravel(), ids[:-1, 1:].ravel()]
    vs = [ids[:, 1:].ravel(), ids[1:, :].ravel(), ids[1:, 1:].ravel(), ids[1:, :-1].ravel()]
    for s in strides:
        r, c = np.meshgrid(np.arange(0, height, s), np.arange(0, width, s), indexing="ij")
        ok = r + s < height
        us.append(ids[r[ok], c[ok]])
        vs.append(ids[r[ok] + s, c[ok]])
        ok = c + s < width
        us.append(ids[r[ok], c[ok]])
        vs.append(ids[r[ok], c[ok] + s])
    u, v = np.concatenate(us), np.concatenate(vs)
    cost = np.random.default_rng(seed).standard_normal(u.size)
    return height * width, u, v, cost


def grid3d_coo(depth=128, height=256, width=256, stride=2, seed=0):
    """C3: z-major 6-connected 3-D grid + stride lattice along z, y, x.
    128x256x256 -> 28,147,712 edges."""
    ids = np.arange(depth * height * width, dtype=np.int64).reshape(depth, height, width)
    us = [ids[:-1].ravel(), ids[:, :-1].ravel(), ids[:, :, :-1].ravel()]
    vs = [ids[1:].ravel(), ids[:, 1:].ravel(), ids[:, :, 1:].ravel()]
    if stride >= 2:
        s = stride
        sub = ids[::s, ::s, ::s]
        z, y, x = np.meshgrid(np.arange(0, depth, s), np.arange(0, height, s), np.arange(0, width, s),
                              indexing="ij")
        for ok, dz, dy, dx in ((z + s < depth, s, 0, 0), (y + s < height, 0, s, 0), (x + s < width, 0, 0, s)):
            us.append(sub[ok])
            vs.append(ids[z[ok] + dz, y[ok] + dy, x[ok] + dx])
    u, v = np.concatenate(us), np.concatenate(vs)
    cost = np.random.default_rng(seed).standard_normal(u.size)
    return depth * height * width, u, v, cost


def chung_lu_coo(n=1_000_000, alpha=2.1, draws=26_000_000, seed=0):
    """C4: Chung-Lu power-law graph, w_i = (i+1)^(-1/(alpha-1)); hubs have
    the lowest ids.  Duplicates are left for canonicalisation to sum."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (alpha - 1.0))
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rng = np.random.default_rng(seed)
    u = np.searchsorted(cdf, rng.random(draws))
    v = np.searchsorted(cdf, rng.random(draws))
    keep = u != v
    u, v = u[keep].astype(np.int64), v[keep].astype(np.int64)
    return n, u, v, rng.standard_normal(u.size)


CONFIGS = {
    "c1": dict(fn=grid_coo, kw=dict(height=64, width=64, stride=0), mode="P"),
    "c2": dict(fn=grid8_coo, kw=dict(height=1024, width=2048, strides=(2, 3)), mode="PD"),
    "c3": dict(fn=grid3d_coo, kw=dict(depth=128, height=256, width=256, stride=2), mode="PD"),
    "c4": dict(fn=chung_lu_coo, kw=dict(n=1_000_000, alpha=2.1, draws=26_000_000), mode="PD"),
    "c5": dict(fn=grid_coo, kw=dict(height=512, width=512, stride=0), mode="PD"),
}


def make(config, seed=0, **override):
    """Raw COO for a named config ('c1'..'c5'), optional shape overrides."""
    spec = CONFIGS[config]
    kw = dict(spec["kw"])
    kw.update(override)
    return spec["fn"](seed=seed, **kw)
