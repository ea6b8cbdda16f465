"""Pins of the NEXT-1 oracle functions (segment softmax, GAT attention aggregation and their
backward) against things other than themselves: SPEC's printed
examples (tests/golden/attention_examples.json), the mean-aggregation special case,
normalisation / shift-invariance properties, scipy's softmax per segment, and torch float64
autograd of an independently written edge-list formulation (the gradients are derived by the
library, not by the oracle's hand-written chain rule), plus central finite differences."""
import json
import os

import numpy as np
import pytest
import torch

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "attention_examples.json")))


def _graph(seed, n_src, n_dst, E):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, n_src, E), rng.integers(0, n_dst, E)]).astype(np.int64)


def test_softmax_printed_examples():
    g = GOLD["softmax_symmetry"]
    out = oracle.segment_softmax(np.array(g["values"], np.float32), np.array(g["index"]), g["n"])
    assert np.array_equal(out, np.array(g["out"], np.float32))
    g = GOLD["softmax_single"]
    out = oracle.segment_softmax(np.array(g["values"], np.float32), np.array(g["index"]), g["n"])
    k, v = g["out_at"]
    assert out[k, 0] == v
    assert abs(out[1, 0] + out[2, 0] - 1.0) < 1e-7


@pytest.mark.parametrize("H", [1, 3])
def test_softmax_vs_scipy_and_properties(H):
    from scipy.special import softmax

    rng = np.random.default_rng(H)
    E, n = 500, 40
    idx = rng.integers(0, n, E)
    v = (rng.standard_normal((E, H)) * 5).astype(np.float32)
    out = oracle.segment_softmax(v, idx, n)
    for i in range(n):
        m = idx == i
        if not m.any():
            continue
        ref = softmax(v[m].astype(np.float64), axis=0)
        assert np.allclose(out[m], ref, rtol=1e-6, atol=1e-12)
        assert np.allclose(out[m].astype(np.float64).sum(0), 1.0, atol=1e-6)
    # shift invariance per segment (max subtraction)
    shift = (rng.standard_normal(n) * 8).astype(np.float32)[idx][:, None]
    out2 = oracle.segment_softmax(v + shift, idx, n)
    assert np.allclose(out2, out, rtol=1e-5, atol=1e-9)


def test_softmax_backward_vs_autograd_and_fd():
    rng = np.random.default_rng(7)
    E, n, H = 300, 25, 2
    idx = rng.integers(0, n, E)
    v = rng.standard_normal((E, H)).astype(np.float32)
    g = rng.standard_normal((E, H)).astype(np.float32)
    out = oracle.segment_softmax(v, idx, n)
    gs, ab = oracle.segment_softmax_backward(out, g, idx, n, with_abs=True)
    # torch float64 autograd of a per-segment torch.softmax (library derivation)
    vt = torch.tensor(v, dtype=torch.float64, requires_grad=True)
    res = torch.zeros_like(vt)
    outs = []
    for i in range(n):
        m = torch.from_numpy(idx == i)
        if m.any():
            outs.append((m, torch.softmax(vt[m], dim=0)))
    for m, o in outs:
        res = res.index_put((torch.nonzero(m).flatten(),), o)
    (res * torch.tensor(g, dtype=torch.float64)).sum().backward()
    ref = vt.grad.numpy()
    assert (np.abs(gs - ref) <= 1e-6 * ab + 1e-7).all()
    # central finite differences of L = sum g * softmax(v) in double through scipy
    from scipy.special import softmax

    def L(vv):
        tot = 0.0
        for i in range(n):
            m = idx == i
            if m.any():
                tot += (g[m].astype(np.float64) * softmax(vv[m], axis=0)).sum()
        return tot

    vd = v.astype(np.float64)
    for k, h in [(0, 0), (17, 1), (123, 0), (299, 1)]:
        e = np.zeros_like(vd)
        e[k, h] = 1e-6
        fd = (L(vd + e) - L(vd - e)) / 2e-6
        assert abs(fd - gs[k, h]) < 1e-5 * (1 + abs(fd))


def test_gat_printed_single_node():
    g = GOLD["gat_single_node"]
    out, alpha = oracle.gat(np.array(g["z"], np.float32), np.array(g["s_src"]), np.array(g["s_dst"]),
                            np.array(g["edges"]).T, g["H"])
    assert np.array_equal(alpha, np.array(g["alpha"], np.float32))
    assert np.array_equal(out, np.array(g["out"], np.float32))


def test_gat_zero_attention_is_mean():
    """a = 0 (s_src = s_dst = 0) -> uniform attention -> mean aggregation of z."""
    ei = _graph(3, 60, 60, 400)
    z = np.random.default_rng(4).standard_normal((60, 12)).astype(np.float32)
    out, alpha = oracle.gat(z, np.zeros((60, 3)), np.zeros((60, 3)), ei, 3)
    ref = oracle.propagate(z, ei, reduce="mean")
    assert np.allclose(out, ref, rtol=1e-6, atol=1e-7)
    deg = np.bincount(ei[1], minlength=60)
    assert np.allclose(alpha, (1.0 / deg[ei[1]])[:, None].repeat(3, 1), rtol=1e-7)


def _torch_gat(z, ss, sd, ei, H, slope, n_dst):
    """Independent edge-list GAT in torch float64 (scatter_reduce amax / index_add)."""
    src, dst = torch.from_numpy(ei[0]), torch.from_numpy(ei[1])
    E = ei.shape[1]
    C = z.shape[1] // H
    pre = ss[src] + sd[dst]
    logit = torch.nn.functional.leaky_relu(pre, slope)
    m = torch.full((n_dst, H), -torch.inf, dtype=torch.float64).scatter_reduce(
        0, dst[:, None].expand(E, H), logit, "amax", include_self=True)
    ex = torch.exp(logit - m[dst])
    den = torch.zeros((n_dst, H), dtype=torch.float64).index_add(0, dst, ex)
    alpha = ex / den[dst]
    msg = (alpha[:, :, None] * z[src].view(E, H, C)).view(E, H * C)
    return torch.zeros((n_dst, H * C), dtype=torch.float64).index_add(0, dst, msg), alpha


@pytest.mark.parametrize("H,C,bip", [(1, 5, False), (4, 3, False), (2, 8, True)])
def test_gat_forward_backward_vs_torch_autograd(H, C, bip):
    rng = np.random.default_rng(H * 10 + C)
    n_src, n_dst, E = 50, (30 if bip else 50), 400
    ei = _graph(H + C, n_src, n_dst, E)
    z = rng.standard_normal((n_src, H * C)).astype(np.float32)
    ss = rng.standard_normal((n_src, H)).astype(np.float32) * 2
    sd = rng.standard_normal((n_dst, H)).astype(np.float32) * 2
    g = rng.standard_normal((n_dst, H * C)).astype(np.float32)
    out, alpha, ab = oracle.gat(z, ss, sd, ei, H, n_dst=n_dst, with_abs=True)
    zt = torch.tensor(z, dtype=torch.float64, requires_grad=True)
    st = torch.tensor(ss, dtype=torch.float64, requires_grad=True)
    dt = torch.tensor(sd, dtype=torch.float64, requires_grad=True)
    ref, ralpha = _torch_gat(zt, st, dt, ei, H, 0.2, n_dst)
    assert np.allclose(alpha, ralpha.detach().numpy(), rtol=1e-6, atol=1e-12)
    assert (np.abs(out - ref.detach().numpy()) <= 1e-6 * ab + 1e-7).all()
    (ref * torch.tensor(g, dtype=torch.float64)).sum().backward()
    gr = oracle.gat_backward(z, ss, sd, ei, H, g, n_dst=n_dst, with_abs=True)
    for key, t, a in (("z", zt, "abs_z"), ("s_src", st, "abs_s_src"), ("s_dst", dt, "abs_s_dst")):
        assert (np.abs(gr[key] - t.grad.numpy()) <= 1e-6 * gr[a] + 1e-7).all(), key


def test_gat_empty_segments_and_errors():
    ei = np.array([[0, 1], [2, 2]])
    out, alpha = oracle.gat(np.ones((3, 2), np.float32), np.zeros((3, 1)), np.zeros((3, 1)), ei, 1)
    assert np.array_equal(out[:2], np.zeros((2, 2), np.float32))
    assert np.array_equal(alpha, np.full((2, 1), 0.5, np.float32))
    with pytest.raises(oracle.OracleError):
        oracle.gat(np.ones((3, 2), np.float32), np.zeros((3, 1)), np.zeros((3, 1)), np.array([[0], [3]]), 1)


# ---- NEXT-2: APPNP / SGC --------------------------------------------------

def _gcn_graph(seed, n=40, E=160):
    rng = np.random.default_rng(seed)
    ei = np.stack([rng.integers(0, n, E), rng.integers(0, n, E)]).astype(np.int64)
    ei = ei[:, ei[0] != ei[1]]
    ei = np.concatenate([ei, ei[::-1]], axis=1)  # symmetric
    ei2, w = oracle.gcn_norm(ei, n)
    S = np.zeros((n, n))
    np.add.at(S, (ei2[1], ei2[0]), w.astype(np.float64))  # S[i][j] = sum of w over j -> i
    return ei2, w, S


def test_appnp_printed_special_cases():
    """S:445 alpha = 1 -> h for any K; S:446 K = 1, alpha = 0 -> one GCN propagation."""
    ei, w, _ = _gcn_graph(1)
    h = np.random.default_rng(2).random((40, 3)).astype(np.float32)
    assert np.array_equal(oracle.appnp(h, ei, K=7, alpha=1.0, edge_weight=w), h)
    one = oracle.appnp(h, ei, K=1, alpha=0.0, edge_weight=w)
    assert np.array_equal(one, oracle.propagate(h, ei, reduce="sum", edge_weight=w))
    assert np.array_equal(oracle.appnp(h, ei, K=0, alpha=0.3, edge_weight=w), h)
    with pytest.raises(oracle.OracleError):
        oracle.appnp(h, ei, K=2, alpha=1.5, edge_weight=w)


def test_appnp_dense_power_iteration_and_fixed_point():
    """S:447 dense power-iteration oracle; the K -> inf limit is the closed form
    alpha (I - (1 - alpha) S)^-1 h (APPNP's personalized-PageRank fixed point), reached to
    within (1 - alpha)^K; SGC (alpha = 0, K = 2) equals the dense S^2 h."""
    ei, w, S = _gcn_graph(3)
    h = np.random.default_rng(4).random((40, 5)).astype(np.float32)
    hd = h.astype(np.float64)
    z = hd.copy()
    for _ in range(10):
        z = 0.9 * (S @ z) + 0.1 * hd
    assert np.allclose(oracle.appnp(h, ei, K=10, alpha=0.1, edge_weight=w), z, rtol=1e-6, atol=1e-7)
    fixed = 0.1 * np.linalg.solve(np.eye(40) - 0.9 * S, hd)
    assert np.allclose(oracle.appnp(h, ei, K=300, alpha=0.1, edge_weight=w), fixed, rtol=1e-5, atol=1e-6)
    assert np.allclose(oracle.appnp(h, ei, K=2, alpha=0.0, edge_weight=w), S @ (S @ hd), rtol=1e-6, atol=1e-7)


def test_appnp_constant_fixed_point():
    """complete graph with self-loops, constant features -> unchanged (stochastic matrix)."""
    n = 6
    src, dst = np.meshgrid(np.arange(n), np.arange(n))
    ei = np.stack([src.ravel(), dst.ravel()]).astype(np.int64)
    ei2, w = oracle.gcn_norm(ei, n)
    h = np.full((n, 2), 0.75, np.float32)
    out = oracle.appnp(h, ei2, K=5, alpha=0.2, edge_weight=w)
    assert np.allclose(out, h, rtol=1e-7)


# ---- NEXT-2: dense transform --------------------------------------------------------

def test_dense_transform_vs_numpy_and_special_cases():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((37, 23)).astype(np.float32)
    w = rng.standard_normal((11, 23)).astype(np.float32)
    b = rng.standard_normal(11).astype(np.float32)
    rs = rng.random(37).astype(np.float32)
    y, ab = oracle.dense_transform(x, w, bias=b, row_scale=rs, with_abs=True)
    ref = rs[:, None].astype(np.float64) * (x.astype(np.float64) @ w.T.astype(np.float64)) + b
    assert np.allclose(y, ref, rtol=1e-6, atol=1e-6)
    assert (ab >= np.abs(ref - b) - 1e-9).all()
    # identity weight -> copy (exact); zero weight -> bias
    eye = np.eye(23, dtype=np.float32)
    assert np.array_equal(oracle.dense_transform(x, eye), x)
    assert np.array_equal(oracle.dense_transform(x, np.zeros((4, 23), np.float32), bias=b[:4]),
                          np.broadcast_to(b[:4], (37, 4)))
