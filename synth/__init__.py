"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module generates INPUTS ONLY: graphs (COO edge indices), feature matrices,
upstream gradients.  It holds none of the method's arithmetic (no gather, no
reduction, no normalisation, no collate), so both the CUDA path and the CPU
oracle can consume the same arrays (task rule ③).  The recipes are stated in
DESIGN.md "Input recipe" and SURVEY.md §8(d).

Shapes follow PAPER.md Table 5: Cora 2,708 nodes / 5,278 undirected
edges, PubMed 19,717 / 44,324 / 500 features; the point clouds follow Table 3's
ModelNet setting (1,024 points) with k-NN graphs; Reddit uses the
public Reddit edge count (~114.6M, BASELINE config 4); R-MAT uses the Graph500
parameters (BASELINE config 5).

Small generators use numpy ``default_rng``; the large ones (configs 4, 5) use a
seeded ``torch.Generator`` on the requested device so that a B200 box generates
them in well under a second.  The generators are deterministic for a fixed
(seed, device type); host copies of the same arrays feed the oracle.
"""
from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# config shapes (BASELINE.json "configs")
CORA = dict(N=2708, E=10556, F=16)
PUBMED = dict(N=19717, pairs=44324, F=500)
CLOUDS = dict(G=64, P=1024, k=16, F=64)
REDDIT = dict(N=232965, E=114615892, F=602)
RMAT = dict(N=10_000_000, E=200_000_000, F=128, scale=24, abcd=(0.57, 0.19, 0.19, 0.05))


def uniform_edges(N, E, seed, no_loops=False, n_dst=None):
    """E iid uniform (src, dst) pairs; duplicates kept; optionally resample src == dst."""
    rng = np.random.default_rng(seed)
    n_dst = N if n_dst is None else n_dst
    src = rng.integers(0, N, E, dtype=np.int64)
    dst = rng.integers(0, n_dst, E, dtype=np.int64)
    if no_loops:
        bad = src == dst
        while bad.any():
            src[bad] = rng.integers(0, N, int(bad.sum()), dtype=np.int64)
            bad = src == dst
    return np.stack([src, dst])


def features(n, F, seed, signed=False, ld=None, dtype=np.float32):
    """X ~ U[0,1) (default, like bag-of-words / TF-IDF inputs) or U(-1,1).

    With ``ld > F`` returns a strided row view into an (n, ld) zero-padded buffer.
    """
    rng = np.random.default_rng(seed)
    x = rng.random((n, F), dtype=np.float64)
    if signed:
        x = 2.0 * x - 1.0
    x = x.astype(dtype)
    if ld is not None and ld > F:
        buf = np.zeros((n, ld), dtype)
        buf[:, :F] = x
        return buf[:, :F]
    return x


def cora_like(seed=1):
    """Config 1: N=2708, E=10556 iid uniform directed edges, no self-loops, F=16."""
    c = CORA
    ei = uniform_edges(c["N"], c["E"], seed, no_loops=True)
    x = features(c["N"], c["F"], 100 + seed)
    return ei, x


def symmetric_pairs(N, pairs, seed):
    """`pairs` distinct unordered pairs u != v, both directions, seeded shuffle."""
    rng = np.random.default_rng(seed)
    chosen = set()
    us, vs = [], []
    while len(us) < pairs:
        m = pairs - len(us)
        u = rng.integers(0, N, 2 * m, dtype=np.int64)
        v = rng.integers(0, N, 2 * m, dtype=np.int64)
        for a, b in zip(u.tolist(), v.tolist()):
            if a == b:
                continue
            key = (a, b) if a < b else (b, a)
            if key in chosen:
                continue
            chosen.add(key)
            us.append(key[0])
            vs.append(key[1])
            if len(us) == pairs:
                break
    u = np.array(us, np.int64)
    v = np.array(vs, np.int64)
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    order = rng.permutation(src.size)
    return np.stack([src[order], dst[order]])


def pubmed_like(seed=2):
    """Config 2: symmetric, loop-free, duplicate-free PubMed-shaped graph; X ~ U[0,1), F=500;
    grad_out ~ U(-1,1) for the backward."""
    c = PUBMED
    ei = symmetric_pairs(c["N"], c["pairs"], seed)
    x = features(c["N"], c["F"], 100 + seed)
    g = features(c["N"], c["F"], 200 + seed, signed=True)
    return ei, x, g


def knn_cloud_edges(G=64, P=1024, k=16, seed=3):
    """Config 3 inputs: G clouds of P points ~ U[0,1)^3 and, per cloud, the k nearest
    neighbours of every point (squared L2 in fp64, self excluded, ties -> lower index).
    Edges j -> i for j in kNN(i); per cloud ordered by (i, rank).

    Returns (num_nodes[G], edge_ptr[G+1], local_edge_index[2 x G*P*k]) -- the per-graph
    lists that the mini-batch collate consumes.  kNN is input generation only
    (P:80); it is not on the timed path.
    """
    rng = np.random.default_rng(seed)
    srcs, dsts = [], []
    for _ in range(G):
        pos = rng.random((P, 3))
        d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(-1)
        np.fill_diagonal(d2, np.inf)
        nbr = np.argsort(d2, axis=1, kind="stable")[:, :k]  # ties -> lower index
        dsts.append(np.repeat(np.arange(P, dtype=np.int64), k))
        srcs.append(nbr.reshape(-1).astype(np.int64))
    local = np.stack([np.concatenate(srcs), np.concatenate(dsts)])
    num_nodes = np.full(G, P, np.int64)
    edge_ptr = np.arange(G + 1, dtype=np.int64) * (P * k)
    return num_nodes, edge_ptr, local


def clouds_like(seed=3):
    c = CLOUDS
    num_nodes, edge_ptr, local = knn_cloud_edges(c["G"], c["P"], c["k"], seed)
    x = features(c["G"] * c["P"], c["F"], 100 + seed, signed=True)
    return num_nodes, edge_ptr, local, x


def random_graph_list(G, seed, n_range=(1, 40), deg=3.0):
    """Small random graphs for collate / batching-equivalence tests."""
    rng = np.random.default_rng(seed)
    nn = rng.integers(n_range[0], n_range[1] + 1, G).astype(np.int64)
    locs, eptr = [], [0]
    for n in nn.tolist():
        e = int(rng.poisson(deg * n))
        s = rng.integers(0, n, e, dtype=np.int64)
        d = rng.integers(0, n, e, dtype=np.int64)
        locs.append(np.stack([s, d]))
        eptr.append(eptr[-1] + e)
    local = np.concatenate(locs, axis=1) if locs else np.zeros((2, 0), np.int64)
    return nn, np.array(eptr, np.int64), local


def erdos_renyi(n, avg_degree, seed, directed=True):
    """G(n, p) with p = avg_degree / (n - 1) (Fig. 3 caption P:266)."""
    rng = np.random.default_rng(seed)
    p = avg_degree / (n - 1)
    m = rng.binomial(n * (n - 1), p)
    # sample m distinct ordered pairs (u != v) uniformly
    flat = rng.choice(n * (n - 1), size=m, replace=False)
    u = flat // (n - 1)
    v = flat % (n - 1)
    v = v + (v >= u)
    ei = np.stack([u, v]).astype(np.int64)
    if not directed:
        ei = np.concatenate([ei, ei[::-1]], axis=1)
    return ei


def rmat_edges_np(scale, E, N, seed, abcd=(0.57, 0.19, 0.19, 0.05)):
    """Graph500 R-MAT (numpy; small scales only): reject ids >= N, then a seeded relabel."""
    rng = np.random.default_rng(seed)
    a, b, c, _ = abcd
    out_s, out_d, have = [], [], 0
    while have < E:
        m = int((E - have) * 1.3) + 16
        s = np.zeros(m, np.int64)
        d = np.zeros(m, np.int64)
        for lvl in range(scale):
            r = rng.random(m)
            bit = np.int64(1) << np.int64(scale - 1 - lvl)
            s |= np.where(r >= a + b, bit, 0)
            d |= np.where(((r >= a) & (r < a + b)) | (r >= a + b + c), bit, 0)
        ok = (s < N) & (d < N)
        out_s.append(s[ok])
        out_d.append(d[ok])
        have += int(ok.sum())
    s = np.concatenate(out_s)[:E]
    d = np.concatenate(out_d)[:E]
    relabel = rng.permutation(N).astype(np.int64)
    return np.stack([relabel[s], relabel[d]])


# ---------------------------------------------------------------------------
# large generators (torch; GPU on the box)

def _torch_gen(device, seed):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def reddit_like_torch(device, seed=4, ld=None, N=None, E=None, F=None):
    """Config 4: E iid uniform (src, dst) over N nodes (loops/dups kept => in-degree ~
    Poisson(492)); X ~ U[0,1) with row stride ld (>= F).  Returns (edge_index [2,E] int64,
    X [N, F] float32 possibly a strided view)."""
    import torch

    c = REDDIT
    N = N or c["N"]
    E = E or c["E"]
    F = F or c["F"]
    g = _torch_gen(device, seed)
    ei = torch.randint(0, N, (2, E), generator=g, device=device, dtype=torch.int64)
    gx = _torch_gen(device, 100 + seed)
    ld = ld or F
    buf = torch.zeros((N, ld), dtype=torch.float32, device=device)
    buf[:, :F] = torch.rand((N, F), generator=gx, device=device, dtype=torch.float32)
    return ei, buf[:, :F]


def rmat_torch(device, seed=5, scale=None, N=None, E=None, abcd=None, chunk=1 << 25):
    """Config 5: Graph500 R-MAT (a,b,c,d) at `scale`, reject ids >= N (accept ~0.80), then a
    seeded random relabel of [0, N); exactly E edges, loops/dups kept."""
    import torch

    c = RMAT
    scale = scale or c["scale"]
    N = N or c["N"]
    E = E or c["E"]
    a, b, cc, _ = abcd or c["abcd"]
    g = _torch_gen(device, seed)
    src = torch.empty(E, dtype=torch.int64, device=device)
    dst = torch.empty(E, dtype=torch.int64, device=device)
    have = 0
    while have < E:
        m = min(chunk, int((E - have) * 1.3) + 1024)
        s = torch.zeros(m, dtype=torch.int64, device=device)
        d = torch.zeros(m, dtype=torch.int64, device=device)
        for lvl in range(scale):
            r = torch.rand(m, generator=g, device=device)
            bit = 1 << (scale - 1 - lvl)
            s += (r >= a + b).to(torch.int64) * bit
            d += (((r >= a) & (r < a + b)) | (r >= a + b + cc)).to(torch.int64) * bit
        ok = (s < N) & (d < N)
        s = s[ok]
        d = d[ok]
        take = min(E - have, s.numel())
        src[have:have + take] = s[:take]
        dst[have:have + take] = d[:take]
        have += take
    relabel = torch.randperm(N, generator=g, device=device)
    return torch.stack([relabel[src], relabel[dst]])
