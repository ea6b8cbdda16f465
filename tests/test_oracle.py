"""Pins for the CPU oracle (task rule ③): each oracle function is checked against
something other than itself -- printed worked examples (tests/golden/, each cited),
closed forms, dense brute force, an independent library routine, or invariants.

Runs without a GPU (-m "not gpu").
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerance import check_close, check_exact

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def rand_graph(rng, n_src, n_dst, E):
    return np.stack([rng.integers(0, n_src, E), rng.integers(0, n_dst, E)]).astype(np.int64)


def dense_adj(ei, n_src, n_dst, w=None):
    """A[i, j] = sum of w over edges j -> i, built as onehot(dst)^T diag(w) onehot(src)
    (a dense matrix product, independent of the oracle's edge loop)."""
    E = ei.shape[1]
    w = np.ones(E) if w is None else np.asarray(w, np.float64)
    Od = (ei[1][:, None] == np.arange(n_dst)[None, :]).astype(np.float64)  # E x n_dst
    Os = (ei[0][:, None] == np.arange(n_src)[None, :]).astype(np.float64)  # E x n_src
    return Od.T @ (w[:, None] * Os)


def brute_max(M, dst, n_dst):
    """Per-column max over each target's messages and the FIRST (lowest k) index
    attaining it, via np.argmax on the ascending edge list (empty -> 0, E)."""
    E, Fo = M.shape
    out = np.zeros((n_dst, Fo), np.float32)
    arg = np.full((n_dst, Fo), E, np.int64)
    for i in range(n_dst):
        ks = np.nonzero(dst == i)[0]
        if ks.size == 0:
            continue
        sub = M[ks]
        a = np.argmax(sub, axis=0)
        out[i] = sub[a, np.arange(Fo)]
        arg[i] = ks[a]
    return out, arg


# --------------------------------------------------------------------------- printed examples

def test_scatter_printed_examples():
    for c in gold("scatter_spec_examples.json")["cases"]:
        res = oracle.scatter(np.array(c["src"], np.float32), c["index"], c["dim_size"], c["reduce"])
        out = res[0] if isinstance(res, tuple) else res
        check_exact(out, np.array(c["out"], np.float32), c["reduce"])


def test_argmax_ties_and_empty():
    g = gold("argmax_ties.json")
    out, arg = oracle.scatter(np.array(g["src"], np.float32), g["index"], g["dim_size"], "max")
    check_exact(out, np.array(g["out"], np.float32))
    check_exact(arg, np.array(g["arg"], np.int64))


def test_structure_printed_examples():
    g = gold("structure_examples.json")
    c = g["collate"]
    ei, batch, node_ptr = oracle.collate(c["num_nodes"], c["edge_ptr"], [c["local_src"], c["local_dst"]])
    check_exact(ei, np.array([c["src"], c["dst"]]))
    check_exact(batch, np.array(c["batch"]))
    check_exact(node_ptr, np.array(c["node_ptr"]))

    d = g["degree"]
    ei = np.array(d["edges"]).T
    check_exact(oracle.degree(ei[1], d["N"]), np.array(d["deg"]))
    check_exact(oracle.degree(np.zeros(0, np.int64), 3), np.zeros(3, np.int64))

    t = g["to_csr"]
    ei = np.array(t["edges"]).T
    rowptr, perm = oracle.csr(ei[1], t["N"])
    check_exact(rowptr, np.array(t["rowptr"]))
    check_exact(ei[0][perm], np.array(t["col"]))
    rowptr, perm = oracle.csr(np.zeros(0, np.int64), 3)
    check_exact(rowptr, np.zeros(4, np.int64))

    s = g["spmm"]
    out = oracle.propagate(np.array(s["x"], np.float32), np.array(s["edges"]).T, reduce="sum")
    check_exact(out, np.array(s["out"], np.float32))

    gi = g["gin_sum"]
    x = np.array(gi["x"], np.float32)
    out = oracle.propagate(x, np.array(gi["edges"]).T, reduce="sum")
    check_exact(x + out, np.array(gi["out"], np.float32))

    gb = g["gather_backward"]
    # gather(x, index) is propagate's x_j block with edges (index[k] -> k); its backward
    # w.r.t. x is the scatter-add of the upstream gradient.
    x = np.array(gb["x"], np.float32)
    idx = np.array(gb["index"])
    ei = np.stack([idx, np.arange(idx.size)])
    gr = oracle.propagate_backward(x, ei, np.ones((idx.size, 2), np.float32), n_dst=idx.size)
    check_exact(gr["x_src"], np.array(gb["grad_x"], np.float32))

    gp = g["global_pool"]
    out = oracle.global_pool(np.array(gp["x"], np.float32), gp["batch"], gp["G"], "sum")
    check_exact(out, np.array(gp["out"], np.float32))

    ps = g["propagate_self_loop"]
    x = np.array(ps["x"], np.float32)
    for red in ("sum", "mean"):
        check_exact(oracle.propagate(x, np.array(ps["edges"]).T, reduce=red), x)
    check_exact(oracle.propagate(x, np.array(ps["edges"]).T, reduce="max")[0], x)


def test_empty_edge_set_gives_zero():
    # S:370 empty edge set -> all-zero output; S:159/S:189 empty segments give 0
    x = synth.features(5, 3, 0)
    ei = np.zeros((2, 0), np.int64)
    for red in ("sum", "mean"):
        check_exact(oracle.propagate(x, ei, reduce=red), np.zeros((5, 3), np.float32))
    out, arg = oracle.propagate(x, ei, reduce="max")
    check_exact(out, np.zeros((5, 3), np.float32))
    check_exact(arg, np.zeros((5, 3), np.int64))  # arg = E = 0


# --------------------------------------------------------------------------- GCN closed forms

def test_gcn_closed_forms():
    g = gold("gcn_closed_forms.json")
    X = np.array(g["X"], np.float32)
    for key in ("path_P4", "star_K13"):
        und = np.array(g[key]["undirected_edges"]).T
        ei = np.concatenate([und, und[::-1]], axis=1)
        ei2, w = oracle.gcn_norm(ei, 4)
        out = oracle.propagate(X, ei2, reduce="sum", edge_weight=w)
        check_close(out, np.array(g[key]["SX"]), atol=2e-7, rtol=2e-7, what=key)
    for c in g["spec_gcn_norm"]:
        ei = np.array(c["edges"]).T
        ei2, w = oracle.gcn_norm(ei, c["N"])
        check_close(w, np.array(c["weights"]), rtol=0, atol=1e-7)
    c = g["spec_gcn_layer"]
    ei2, w = oracle.gcn_norm(np.array(c["edges"]).T, c["N"])
    out = oracle.propagate(np.array(c["x"], np.float32), ei2, reduce="sum", edge_weight=w)
    check_close(out, np.array(c["out"]), rtol=0, atol=1e-7)
    c = g["spec_add_self_loops"]
    ei2, _ = oracle.gcn_norm(np.array(c["edges"]).T, c["N"])
    check_exact(ei2, np.array(c["edges_out"]).T)


@pytest.mark.parametrize("seed", range(4))
def test_gcn_dense_formula(seed):
    """propagate(gcn_norm) == dense D^-1/2 (A+I) D^-1/2 X (reading Q7: in-degree,
    existing self-loops kept, missing ones added with weight 1)."""
    rng = np.random.default_rng(seed)
    N, E = 30, 90
    ei = rand_graph(rng, N, N, E)
    if seed % 2:
        ei[:, :5] = np.array([[3, 3, 7, 7, 7], [3, 3, 7, 7, 7]])  # duplicated existing loops kept
    X = synth.features(N, 6, seed, signed=True)
    A = dense_adj(ei, N, N)
    loops = np.diag(A) > 0
    Ahat = A + np.diag((~loops).astype(np.float64))
    d = Ahat.sum(1)
    S = np.diag(d ** -0.5) @ Ahat @ np.diag(d ** -0.5)
    ref = S @ X.astype(np.float64)
    ei2, w = oracle.gcn_norm(ei, N)
    assert ei2.shape[1] == E + int((~loops).sum())
    out, ab = oracle.propagate(X, ei2, reduce="sum", edge_weight=w, with_abs=True)
    check_close(out, ref, abs_sum=np.abs(S) @ np.abs(X.astype(np.float64)), rtol=1e-6)
    # weights are the dense S entries
    check_close(w, S[ei2[1], ei2[0]] / np.maximum(1, A[ei2[1], ei2[0]] + (ei2[0] == ei2[1]) * (~loops)[ei2[0]]),
                rtol=1e-6, atol=0)


# --------------------------------------------------------------------------- sum / mean

@pytest.mark.parametrize("seed", range(6))
def test_sum_equals_dense_brute_force(seed):
    """out = A X (special case -> textbook matmul); bipartite, weighted and unweighted."""
    rng = np.random.default_rng(seed)
    n_src, n_dst, E, F = int(rng.integers(1, 64)), int(rng.integers(1, 64)), int(rng.integers(0, 300)), 5
    ei = rand_graph(rng, n_src, n_dst, E)
    X = synth.features(n_src, F, seed)
    w = rng.random(E).astype(np.float32) if seed % 2 else None
    A = dense_adj(ei, n_src, n_dst, w)
    out = oracle.propagate(X, ei, n_dst=n_dst, reduce="sum", edge_weight=w)
    check_close(out, A @ X.astype(np.float64), rtol=1e-6, atol=1e-7)
    # mean divides by the integer in-degree (Q6), not by sum of weights
    deg = dense_adj(ei, n_src, n_dst).sum(1)
    mean = oracle.propagate(X, ei, n_dst=n_dst, reduce="mean", edge_weight=w)
    ref = np.where(deg[:, None] > 0, (A @ X.astype(np.float64)) / np.maximum(deg, 1)[:, None], 0)
    check_close(mean, ref, rtol=1e-6, atol=1e-7)


def test_integer_sums_are_exact():
    """Integer-valued |x| <= 8: every partial sum is exact, result is bitwise A X."""
    rng = np.random.default_rng(7)
    ei = rand_graph(rng, 50, 40, 400)
    X = rng.integers(-8, 9, (50, 7)).astype(np.float32)
    out = oracle.propagate(X, ei, n_dst=40, reduce="sum")
    check_exact(out, (dense_adj(ei, 50, 40) @ X).astype(np.float32))


def test_sum_matches_torch_index_add():
    """Independent library routine: torch CPU index_add_ in float64."""
    rng = np.random.default_rng(11)
    ei = rand_graph(rng, 200, 150, 3000)
    X = synth.features(200, 9, 3, signed=True)
    w = rng.random(3000).astype(np.float32)
    msg = torch.from_numpy(X).double()[torch.from_numpy(ei[0])] * torch.from_numpy(w).double()[:, None]
    ref = torch.zeros(150, 9, dtype=torch.float64).index_add_(0, torch.from_numpy(ei[1]), msg)
    out, ab = oracle.propagate(X, ei, n_dst=150, reduce="sum", edge_weight=w, with_abs=True)
    check_close(out, ref.numpy(), abs_sum=ab, rtol=1e-7)


def test_gs_equals_torch_sparse_spmm():
    """GS = SpMM: CSR(row = target) . X via torch.sparse (library)."""
    rng = np.random.default_rng(5)
    for deg in (1, 4, 16, 64):
        N = 100
        ei = rand_graph(rng, N, N, N * deg)
        X = synth.features(N, 4, deg)
        A = torch.sparse_coo_tensor(torch.from_numpy(ei[::-1].copy()), torch.ones(ei.shape[1], dtype=torch.float64),
                                    (N, N)).coalesce().to_sparse_csr()
        ref = (A @ torch.from_numpy(X).double()).numpy()
        check_close(oracle.propagate(X, ei, reduce="sum"), ref, rtol=1e-6, atol=1e-7)


def test_mean_constant_rows_exact():
    """scatter-mean of constant-c rows = c on every non-empty segment, exactly."""
    rng = np.random.default_rng(3)
    idx = rng.integers(0, 30, 500)
    c = np.float32(0.3713)
    out = oracle.scatter(np.full((500, 4), c, np.float32), idx, 31, "mean")
    deg = np.bincount(idx, minlength=31)
    check_exact(out[deg > 0], np.full(((deg > 0).sum(), 4), c, np.float32))
    check_exact(out[deg == 0], np.zeros(((deg == 0).sum(), 4), np.float32))


def test_permutation_invariance_and_relabel_equivariance():
    """S:374 edge-permutation invariance; S:376 node-relabelling equivariance."""
    rng = np.random.default_rng(9)
    N, E = 60, 700
    ei = rand_graph(rng, N, N, E)
    X = synth.features(N, 5, 1, signed=True)
    p = rng.permutation(E)
    for red in ("sum", "mean"):
        a, ab = oracle.propagate(X, ei, reduce=red, with_abs=True)
        b = oracle.propagate(X, ei[:, p], reduce=red)
        check_close(b, a, abs_sum=ab, rtol=1e-7)
    m1, a1 = oracle.propagate(X, ei, reduce="max")
    m2, a2 = oracle.propagate(X, ei[:, p], reduce="max")
    check_exact(m2, m1)  # values bitwise
    pi = rng.permutation(N)
    ei_r = pi[ei]
    Xr = np.empty_like(X)
    Xr[pi] = X
    for red in ("sum", "mean"):
        a = oracle.propagate(X, ei, reduce=red)
        b = oracle.propagate(Xr, ei_r, reduce=red)
        check_exact(b[pi], a)  # same edges in the same order => identical accumulation
    mr, ar = oracle.propagate(Xr, ei_r, reduce="max")
    check_exact(mr[pi], m1)
    check_exact(ar[pi], a1)


# --------------------------------------------------------------------------- max / argmax

@pytest.mark.parametrize("seed", range(5))
def test_max_brute_force_and_invariants(seed):
    rng = np.random.default_rng(seed)
    n_src, n_dst, E, F = 40, 30, int(rng.integers(0, 250)), 4
    ei = rand_graph(rng, n_src, n_dst, E)
    # tie-heavy values including +-0 (reading Q4: IEEE equality, lowest edge id wins)
    X = rng.integers(-3, 4, (n_src, F)).astype(np.float32)
    X[rng.random((n_src, F)) < 0.2] = -0.0
    w = None
    if seed % 2:
        w = rng.choice(np.array([0.5, 1.0, 2.0], np.float32), E)
    M = X[ei[0]] * (w[:, None] if w is not None else np.float32(1))
    out, arg = oracle.propagate(X, ei, n_dst=n_dst, reduce="max", edge_weight=w)
    ro, ra = brute_max(M.astype(np.float32), ei[1], n_dst)
    check_exact(out, ro)
    check_exact(arg, ra)
    # invariants: dst[arg] = i; out = m_arg; no lower id with an equal value; out >= all members
    for i in range(n_dst):
        ks = np.nonzero(ei[1] == i)[0]
        for c in range(F):
            if ks.size == 0:
                assert arg[i, c] == E and out[i, c] == 0
                continue
            k = arg[i, c]
            assert ei[1][k] == i and M[k, c] == out[i, c]
            assert (M[ks, c] <= out[i, c]).all()
            assert not ((M[ks, c] == out[i, c]) & (ks < k)).any()


def test_scatter_max_concat_and_edge_attr_blocks():
    """Message [x_i || w x_j || e_ji]: each block reduced independently."""
    rng = np.random.default_rng(1)
    N, E, F, D = 20, 120, 3, 2
    ei = rand_graph(rng, N, N, E)
    X = synth.features(N, F, 4, signed=True)
    ea = synth.features(E, D, 5, signed=True)
    w = rng.random(E).astype(np.float32)
    M = np.concatenate([X[ei[1]], X[ei[0]] * w[:, None], ea], axis=1).astype(np.float32)
    for red in ("sum", "mean", "max"):
        res = oracle.propagate(X, ei, reduce=red, edge_weight=w, edge_attr=ea, concat_xi=True)
        ref = oracle.scatter(M, ei[1], N, red)
        if red == "max":
            check_exact(res[0], ref[0])
            check_exact(res[1], ref[1])
        else:
            check_close(res, ref, rtol=1e-6, atol=1e-7)


# --------------------------------------------------------------------------- backward

@pytest.mark.parametrize("red", ["sum", "mean"])
def test_scatter_backward_adjoint(red):
    """<scatter(u), v> = <u, scatter_backward(v)> for the linear reductions (closed form)."""
    rng = np.random.default_rng(2)
    E, n, F = 400, 35, 6
    idx = rng.integers(0, n, E)
    u = synth.features(E, F, 1, signed=True)
    v = synth.features(n, F, 2, signed=True)
    su = oracle.scatter(u, idx, n, red).astype(np.float64)
    gb = oracle.scatter_backward(v, idx, red).astype(np.float64)
    lhs = (su * v).sum()
    rhs = (u.astype(np.float64) * gb).sum()
    assert abs(lhs - rhs) <= 1e-5 * (np.abs(su * v).sum() + 1e-9)


def test_scatter_backward_max_finite_differences():
    """scatter-max backward pinned by the forward alone: L(src) = <g, scatter_max(src)> is
    piecewise linear, so away from ties the one-sided difference quotient of the FORWARD oracle in one
    coordinate, (L(src + h e_kc) - L(src)) / h, equals dL/dsrc[k][c] -- g[index[k]][c] where k is the
    argmax of its (segment, column), else 0.  Values are distinct multiples of 1/64 and h = 1/1024, so
    no perturbation changes an argmax and every difference is exact in fp32."""
    rng = np.random.default_rng(4)
    E, n, F = 120, 13, 3
    idx = rng.integers(0, n, E)
    src = (rng.permutation(E * F).reshape(E, F).astype(np.float32) - E * F / 2) / 64.0
    g = synth.features(n, F, 3, signed=True).astype(np.float64)
    _, arg = oracle.scatter(src, idx, n, "max")
    gs = oracle.scatter_backward(g.astype(np.float32), idx, "max", arg=arg)
    h = 1.0 / 1024

    def L(s):
        return float((oracle.scatter(s, idx, n, "max")[0].astype(np.float64) * g).sum())

    base = L(src)
    fd = np.zeros((E, F))
    for k in range(E):
        for c in range(F):
            s2 = src.copy()
            s2[k, c] += h
            fd[k, c] = (L(s2) - base) / h
    check_close(gs, fd, rtol=1e-6, atol=1e-6)
    assert (gs != 0).sum() == int((arg < E).sum())  # one routed entry per non-empty (segment, column)


@pytest.mark.parametrize("red", ["sum", "mean"])
def test_propagate_backward_adjoint(red):
    """propagate is linear in x_src, x_dst (concat block), edge_attr and w for sum/mean:
    <propagate(.), G> = <input, grad_input> for each input (closed form)."""
    rng = np.random.default_rng(6)
    n_src, n_dst, E, F, D = 30, 25, 200, 4, 3
    ei = rand_graph(rng, n_src, n_dst, E)
    X = synth.features(n_src, F, 1, signed=True)
    Xd = synth.features(n_dst, F, 2, signed=True)
    ea = synth.features(E, D, 3, signed=True)
    w = rng.random(E).astype(np.float32)
    G = synth.features(n_dst, 2 * F + D, 4, signed=True).astype(np.float64)
    gr = oracle.propagate_backward(X, ei, G.astype(np.float32), n_dst=n_dst, reduce=red, edge_weight=w, D=D,
                                   concat_xi=True, need_x_dst=True, need_edge_attr=True,
                                   need_edge_weight=True)
    z = np.zeros_like
    def f(Xs, Xdd, eaa, ww):
        return (oracle.propagate(Xs, ei, n_dst=n_dst, reduce=red, edge_weight=ww, edge_attr=eaa, x_dst=Xdd,
                                 concat_xi=True).astype(np.float64) * G).sum()
    base = f(z(X), z(Xd), z(ea), w)
    assert base == 0
    tol = lambda a: 1e-5 * a + 1e-9
    lhs = f(X, z(Xd), z(ea), w)
    assert abs(lhs - (X * gr["x_src"]).sum()) <= tol(np.abs(X).sum() * np.abs(G).max() * 10)
    lhs = f(z(X), Xd, z(ea), w)
    assert abs(lhs - (Xd * gr["x_dst"]).sum()) <= tol(np.abs(Xd).sum() * np.abs(G).max() * 10)
    lhs = f(z(X), z(Xd), ea, w)
    assert abs(lhs - (ea * gr["edge_attr"]).sum()) <= tol(np.abs(ea).sum() * np.abs(G).max() * 10)
    # linear in w with x_i/e blocks at zero
    lhs = f(X, z(Xd), z(ea), w)
    assert abs(lhs - (w * gr["edge_weight"]).sum()) <= tol(np.abs(X).sum() * np.abs(G).max() * 10)


def test_propagate_backward_max_routing_and_fd():
    rng = np.random.default_rng(8)
    n, E, F = 20, 60, 3
    ei = rand_graph(rng, n, n, E)
    X = synth.features(n, F, 1, signed=True)
    w = (0.5 + rng.random(E)).astype(np.float32)
    out, arg = oracle.propagate(X, ei, reduce="max", edge_weight=w)
    G = synth.features(n, F, 2, signed=True)
    gr = oracle.propagate_backward(X, ei, G, reduce="max", edge_weight=w, arg=arg, need_edge_weight=True)
    ref = np.zeros((n, F))
    refw = np.zeros(E)
    for i in range(n):
        for c in range(F):
            k = arg[i, c]
            if k < E:
                ref[ei[0][k], c] += w[k] * G[i, c]
                refw[k] += X[ei[0][k], c] * G[i, c]
    check_close(gr["x_src"], ref, rtol=1e-6, atol=1e-7)
    check_close(gr["edge_weight"], refw, rtol=1e-6, atol=1e-7)
    # central finite difference along a random direction (max is piecewise linear)
    d = synth.features(n, F, 3, signed=True).astype(np.float64)
    h = 1e-3
    def f(Xs):
        return (oracle.propagate(Xs.astype(np.float32), ei, reduce="max", edge_weight=w)[0].astype(np.float64) * G).sum()
    fd = (f(X + h * d) - f(X - h * d)) / (2 * h)
    assert abs(fd - (d * gr["x_src"]).sum()) < 1e-3 * (1 + abs(fd))


# --------------------------------------------------------------------------- structure

def test_degree_and_csr_match_numpy():
    rng = np.random.default_rng(12)
    for n, E in ((1, 0), (10, 100), (500, 5000)):
        dst = rng.integers(0, n, E)
        check_exact(oracle.degree(dst, n), np.bincount(dst, minlength=n))
        rowptr, perm = oracle.csr(dst, n)
        check_exact(rowptr, np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=n))]))
        check_exact(perm, np.argsort(dst, kind="stable"))


def test_collate_batching_equivalence_and_errors():
    """P:87 'no messages are exchanged between disconnected graphs'."""
    nn, eptr, local = synth.random_graph_list(7, seed=3)
    ei, batch, node_ptr = oracle.collate(nn, eptr, local)
    check_exact(node_ptr, np.concatenate([[0], np.cumsum(nn)]))
    check_exact(batch, np.repeat(np.arange(7), nn))
    N = int(nn.sum())
    X = synth.features(N, 3, 5, signed=True)
    full = {r: oracle.propagate(X, ei, reduce=r) for r in ("sum", "mean", "max")}
    for g in range(7):
        lo, hi = node_ptr[g], node_ptr[g + 1]
        le = local[:, eptr[g]:eptr[g + 1]]
        for r in ("sum", "mean", "max"):
            part = oracle.propagate(X[lo:hi], le, reduce=r)
            if r == "max":
                check_exact(full[r][0][lo:hi], part[0])
                a = part[1].copy()
                a[a == le.shape[1]] = ei.shape[1] - eptr[g]  # empty sentinel E differs
                check_exact(full[r][1][lo:hi], a + eptr[g])
            else:
                check_exact(full[r][lo:hi], part)
    with pytest.raises(oracle.OracleError):
        oracle.collate([], [0], np.zeros((2, 0)))
    bad = local.copy()
    bad[0, 0] = nn[0]
    with pytest.raises(oracle.OracleError) as e:
        oracle.collate(nn, eptr, bad)
    assert e.value.code == 3


def test_errors():
    x = np.ones((3, 2), np.float32)
    with pytest.raises(oracle.OracleError) as e:
        oracle.propagate(x, np.array([[0, 3], [0, 1]]), reduce="sum")
    assert e.value.code == 3
    with pytest.raises(oracle.OracleError) as e:
        oracle.scatter(x, [0, 1, 5], 3, "sum")
    assert e.value.code == 3
    with pytest.raises(oracle.OracleError) as e:
        oracle.scatter(x, [0, 1], 3, "sum")
    assert e.value.code == 2
