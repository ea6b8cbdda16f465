"""GPU parity of the NEXT-1 attention kernels (segment softmax, GAT aggregation, backward;
P:52) against the C oracle on the same seeded inputs, through the
C ABI.  Tolerance (Q11): |got - ref| <= 1e-5 * S + 1e-6 with S the oracle's sum of
term magnitudes (alpha: S = |alpha|)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerance import check_close

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _with_loops(ei, n):
    loops = np.arange(n, dtype=np.int64)
    return np.concatenate([ei, np.stack([loops, loops])], axis=1)


def _case(name):
    rng = np.random.default_rng(abs(hash(name)) % 2**31)
    if name == "cora_h8c8":  # config-1 graph + self-loops, GAT's 8 heads x 8 channels
        ei, _ = synth.cora_like()
        n = 2708
        return _with_loops(ei, n), n, n, 8, 8
    if name == "ragged_h3c5":  # H*C = 15: scalar path, ragged tail
        n = 500
        return np.stack([rng.integers(0, n, 4000), rng.integers(0, n, 4000)]).astype(np.int64), n, n, 3, 5
    if name == "rmat_h4c16":  # power-law rows: hub rows > 2048 positions take the CTA / split paths
        n = 4096
        return synth.rmat_edges_np(scale=12, E=300000, N=n, seed=9), n, n, 4, 16
    if name == "bipartite_h2c36":  # n_src != n_dst, many empty targets, F = 72 (3 float4 chunks/lane)
        return np.stack([rng.integers(0, 700, 3000), rng.integers(0, 900, 3000)]).astype(np.int64), 700, 900, 2, 36
    if name == "h8c5":  # 8 heads of 5 channels: float4 chunks straddle heads -> two-pass kernels even with TMA forced
        n = 600
        return np.stack([rng.integers(0, n, 9000), rng.integers(0, n, 9000)]).astype(np.int64), n, n, 8, 5
    if name == "h4c6":  # F = 24, C % 4 = 2
        n = 500
        return np.stack([rng.integers(0, n, 6000), rng.integers(0, n, 6000)]).astype(np.int64), n, n, 4, 6
    if name == "wide_h8c64":  # H*C = 512
        n = 1200
        return np.stack([rng.integers(0, n, 20000), rng.integers(0, n, 20000)]).astype(np.int64), n, n, 8, 64
    raise KeyError(name)


CASES = ["cora_h8c8", "ragged_h3c5", "rmat_h4c16", "bipartite_h2c36", "wide_h8c64", "h8c5", "h4c6"]


def _inputs(name):
    ei, n_src, n_dst, H, C = _case(name)
    rng = np.random.default_rng(len(name))
    z = rng.standard_normal((n_src, H * C)).astype(np.float32)
    ss = (rng.standard_normal((n_src, H)) * 2).astype(np.float32)
    sd = (rng.standard_normal((n_dst, H)) * 2).astype(np.float32)
    g = rng.standard_normal((n_dst, H * C)).astype(np.float32)
    return ei, n_src, n_dst, H, C, z, ss, sd, g


@pytest.mark.parametrize("tma", ["auto", "1"])
@pytest.mark.parametrize("name", CASES)
def test_gat_forward(name, tma, monkeypatch):
    """tma = "1" forces the TMA gather4 kernel for the alpha-weighted sum wherever it applies
    (C % 4 == 0, F >= 64); "auto" lets the library choose (the LDG kernel at these sizes)."""
    import paper_1903_02428_b200 as pg

    if tma == "1":
        monkeypatch.setenv("PYG_SEG_TMA", "1")

    ei, n_src, n_dst, H, C, z, ss, sd, _ = _inputs(name)
    ref, ralpha, ab = oracle.gat(z, ss, sd, ei, H, n_dst=n_dst, with_abs=True)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n_dst, n_src)
    out, alpha = pg.pyg_gat_propagate(_t(z), _t(ss), _t(sd), H, plan)
    check_close(alpha.cpu().numpy(), ralpha, what="alpha")
    check_close(out.cpu().numpy(), ref, abs_sum=ab, what="out")
    # determinism: a second call is bitwise identical
    out2, alpha2 = pg.pyg_gat_propagate(_t(z), _t(ss), _t(sd), H, plan)
    assert torch.equal(out, out2) and torch.equal(alpha, alpha2)


@pytest.mark.parametrize("factored", [False, True])
@pytest.mark.parametrize("tma", ["auto", "1"])
@pytest.mark.parametrize("name", CASES)
def test_gat_forward_factored(name, tma, factored, monkeypatch):
    """row_sums given: alpha comes back in factored form, alpha / row_sums[dst] = the oracle's alpha;
    out is the same either way."""
    import paper_1903_02428_b200 as pg

    if tma == "1":
        monkeypatch.setenv("PYG_SEG_TMA", "1")
    ei, n_src, n_dst, H, C, z, ss, sd, _ = _inputs(name)
    ref, ralpha, ab = oracle.gat(z, ss, sd, ei, H, n_dst=n_dst, with_abs=True)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n_dst, n_src)
    rs = torch.full((n_dst, H), float("nan"), device=DEV) if factored else None
    out, alpha = pg.pyg_gat_propagate(_t(z), _t(ss), _t(sd), H, plan, row_sums=rs)
    a = alpha / rs[eit[1]] if factored else alpha
    check_close(a.cpu().numpy(), ralpha, what="alpha")
    check_close(out.cpu().numpy(), ref, abs_sum=ab, what="out")


@pytest.mark.parametrize("mode", ["plain", "out", "factored"])
@pytest.mark.parametrize("tma", ["auto", "1"])
@pytest.mark.parametrize("name", CASES)
def test_gat_backward(name, tma, mode, monkeypatch):
    """mode "out"/"factored": the forward output is passed, so (H in {4, 8}, tma = "1") the one-pass TMA
    backward runs (gat_tma.cu: t_i = g_i . out_i); "factored" also keeps alpha in factored form
    (row_sums) through forward and backward; "plain": the two-pass softmax backward."""
    import paper_1903_02428_b200 as pg

    if tma == "1":
        monkeypatch.setenv("PYG_SEG_TMA", "1")

    ei, n_src, n_dst, H, C, z, ss, sd, g = _inputs(name)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n_dst, n_src)
    planT = pg.pyg_plan_build(eit[0], eit[1], n_src, n_dst)
    zt, sst, sdt = _t(z), _t(ss), _t(sd)
    rs = torch.empty((n_dst, H), device=DEV) if mode == "factored" else None
    out, alpha = pg.pyg_gat_propagate(zt, sst, sdt, H, plan, row_sums=rs)
    got = pg.pyg_gat_backward(zt, sst, sdt, H, alpha, _t(g), plan, planT, out=out if mode != "plain" else None,
                              row_sums=rs)
    ref = oracle.gat_backward(z, ss, sd, ei, H, g, n_dst=n_dst, with_abs=True)
    check_close(got["z"].cpu().numpy(), ref["z"], abs_sum=ref["abs_z"], what="grad_z")
    check_close(got["s_src"].cpu().numpy(), ref["s_src"], abs_sum=ref["abs_s_src"], what="grad_s_src")
    check_close(got["s_dst"].cpu().numpy(), ref["s_dst"], abs_sum=ref["abs_s_dst"], what="grad_s_dst")


@pytest.mark.parametrize("blocked_T", [False, True])
@pytest.mark.parametrize("factored", [False, True])
def test_gat_blocked_forward_then_backward(factored, blocked_T, monkeypatch):
    """Training step with the forward on a source-blocked plan (z above L2 in the bench) and the one-pass
    backward on the unblocked plan + its transpose: alpha (by edge id) and row_sums mean the same
    thing on both plans, so the gradients equal the oracle's."""
    import paper_1903_02428_b200 as pg

    monkeypatch.setenv("PYG_SEG_TMA", "1")
    rng = np.random.default_rng(31)
    n, H, C, E = 1500, 8, 16, 24000
    ei = np.stack([rng.integers(0, n, E), rng.integers(0, n - 50, E)]).astype(np.int64)
    z = rng.standard_normal((n, H * C)).astype(np.float32)
    ss = rng.standard_normal((n, H)).astype(np.float32)
    sd = rng.standard_normal((n, H)).astype(np.float32)
    g = rng.standard_normal((n, H * C)).astype(np.float32)
    eit = _t(ei)
    plan_b = pg.pyg_plan_build(eit[1], eit[0], n, n, col_block=400)
    assert plan_b.view()["n_col_blocks"] == 4
    plan = pg.pyg_plan_build(eit[1], eit[0], n, n)
    # blocked_T: grad_z / grad_s_src as passes over blocks of grad_out rows (the transposed plan's sources)
    planT = pg.pyg_plan_build(eit[0], eit[1], n, n, col_block=350 if blocked_T else 0)
    if blocked_T:
        assert planT.view()["n_col_blocks"] == 5
    zt, sst, sdt = _t(z), _t(ss), _t(sd)
    rs = torch.empty((n, H), device=DEV) if factored else None
    out, alpha = pg.pyg_gat_propagate(zt, sst, sdt, H, plan_b, row_sums=rs)
    got = pg.pyg_gat_backward(zt, sst, sdt, H, alpha, _t(g), plan, planT, out=out, row_sums=rs)
    ref = oracle.gat_backward(z, ss, sd, ei, H, g, n_dst=n, with_abs=True)
    check_close(got["z"].cpu().numpy(), ref["z"], abs_sum=ref["abs_z"], what="grad_z")
    check_close(got["s_src"].cpu().numpy(), ref["s_src"], abs_sum=ref["abs_s_src"], what="grad_s_src")
    check_close(got["s_dst"].cpu().numpy(), ref["s_dst"], abs_sum=ref["abs_s_dst"], what="grad_s_dst")


@pytest.mark.parametrize("fused", ["0", "1"])
def test_gat_forward_far_logits_fall_back_exactly(fused, monkeypatch):
    """The one-pass forward shifts each row's logits by the bound leaky_relu(max_j s_src[j] + s_dst[i])
    instead of the row's own max (softmax is shift-invariant).  One outlier source (s_src = 400)
    pushes that bound ~400 above every other row's logits, so their exp() sums underflow: those rows
    must be detected and recomputed with their own max -- the result still equals the oracle (whose
    softmax subtracts the exact max).  fused = "0" runs the two-pass kernels for comparison."""
    import paper_1903_02428_b200 as pg

    monkeypatch.setenv("PYG_SEG_TMA", "1")
    monkeypatch.setenv("PYG_GAT_FUSED", fused)
    rng = np.random.default_rng(11)
    n, H, C = 3000, 4, 16
    ei = np.stack([rng.integers(1, n, 40000), rng.integers(0, n, 40000)]).astype(np.int64)
    ei[0, :50] = 0  # a few rows see the outlier source
    z = rng.standard_normal((n, H * C)).astype(np.float32)
    ss = rng.standard_normal((n, H)).astype(np.float32)
    ss[0] = 400.0
    sd = rng.standard_normal((n, H)).astype(np.float32)
    ref, ralpha, ab = oracle.gat(z, ss, sd, ei, H, n_dst=n, with_abs=True)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n, n)
    out, alpha = pg.pyg_gat_propagate(_t(z), _t(ss), _t(sd), H, plan)
    check_close(alpha.cpu().numpy(), ralpha, what="alpha")
    check_close(out.cpu().numpy(), ref, abs_sum=ab, what="out")


@pytest.mark.parametrize("factored", [False, True])
@pytest.mark.parametrize("outlier", [False, True])
def test_gat_forward_source_blocked(factored, outlier):
    """GAT forward on a source-blocked plan (one pass per block of z rows; the fixed per-row shift of
    reading A9 makes the passes additive) equals the oracle, alpha (normalised, or factored through
    row_sums) and out; rows without in-edges stay 0.  outlier: an s_src of 400 forces the exact
    fallback for most rows (their sums underflow against the global bound)."""
    import paper_1903_02428_b200 as pg

    rng = np.random.default_rng(23)
    n, H, C = 2000, 8, 16
    E = 30000
    ei = np.stack([rng.integers(1, n, E), rng.integers(0, n - 100, E)]).astype(np.int64)  # last 100 rows empty
    ei[0, :40] = 0
    z = rng.standard_normal((n, H * C)).astype(np.float32)
    ss = rng.standard_normal((n, H)).astype(np.float32)
    if outlier:
        ss[0] = 400.0
    sd = rng.standard_normal((n, H)).astype(np.float32)
    ref, ralpha, ab = oracle.gat(z, ss, sd, ei, H, n_dst=n, with_abs=True)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n, n, col_block=450)
    assert plan.view()["n_col_blocks"] == 5
    rs = torch.empty((n, H), device=DEV) if factored else None
    out, alpha = pg.pyg_gat_propagate(_t(z), _t(ss), _t(sd), H, plan, row_sums=rs)
    a = alpha / rs[eit[1]] if factored else alpha
    check_close(a.cpu().numpy(), ralpha, what="alpha")
    check_close(out.cpu().numpy(), ref, abs_sum=ab, what="out")
    assert torch.equal(out[n - 100:], torch.zeros_like(out[n - 100:]))


def test_gat_source_blocked_needs_whole_float4_heads():
    """The blocked GAT forward weighs each float4 chunk of z with one head's alpha: C % 4 != 0 (a chunk
    straddling two heads) is refused instead of computed wrong."""
    import paper_1903_02428_b200 as pg

    rng = np.random.default_rng(5)
    n, H, C, E = 600, 4, 6, 5000
    ei = _t(np.stack([rng.integers(0, n, E), rng.integers(0, n, E)]).astype(np.int64))
    plan = pg.pyg_plan_build(ei[1], ei[0], n, n, col_block=200)
    z = torch.randn((n, H * C), device=DEV)
    s = torch.randn((n, H), device=DEV)
    with pytest.raises(pg.PygError) as e:
        pg.pyg_gat_propagate(z, s, s, H, plan)
    assert e.value.status == "PYG_ERR_UNSUPPORTED"


def test_gat_zero_attention_equals_mean():
    """S:428 on the GPU: s = 0 -> uniform attention = the mean aggregation kernel's result."""
    import paper_1903_02428_b200 as pg

    ei, _ = synth.cora_like()
    n, H, C = 2708, 2, 16
    z = synth.features(n, H * C, 5)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n, n)
    zero = torch.zeros((n, H), device=DEV)
    out, alpha = pg.pyg_gat_propagate(_t(z), zero, zero, H, plan)
    mean = pg.pyg_propagate(_t(z), eit, reduce="mean", plan=plan)
    check_close(out.cpu().numpy(), mean.cpu().numpy(), what="gat(a=0) vs mean")


@pytest.mark.parametrize("H", [1, 3, 4, 8])
def test_segment_softmax(H):
    import paper_1903_02428_b200 as pg

    rng = np.random.default_rng(H)
    E, n = 30000, 2000
    idx = synth.rmat_edges_np(scale=11, E=E, N=n, seed=H)[1]
    v = (rng.standard_normal((E, H)) * 4).astype(np.float32)
    ref = oracle.segment_softmax(v, idx, n)
    plan = pg.pyg_plan_build(_t(idx), None, n)
    out = pg.pyg_segment_softmax(_t(v), plan, n)
    check_close(out.cpu().numpy(), ref, what="softmax")
    g = rng.standard_normal((E, H)).astype(np.float32)
    gs, ab = oracle.segment_softmax_backward(out.cpu().numpy(), g, idx, n, with_abs=True)
    got = pg.pyg_segment_softmax_backward(out, _t(g), plan, n)
    check_close(got.cpu().numpy(), gs, abs_sum=ab, what="softmax backward")


def test_softmax_printed_example():
    """values [0, 0] in one segment -> [0.5, 0.5]; S:168 single element -> 1."""
    import paper_1903_02428_b200 as pg

    idx = torch.tensor([0, 0, 2], device=DEV)
    plan = pg.pyg_plan_build(idx, None, 3)
    out = pg.pyg_segment_softmax(torch.tensor([[0.0], [0.0], [3.5]], device=DEV), plan, 3)
    assert out.flatten().tolist() == [0.5, 0.5, 1.0]


def test_attention_errors():
    import paper_1903_02428_b200 as pg

    ei = torch.randint(0, 50, (2, 300), device=DEV)
    plan = pg.pyg_plan_build(ei[1], ei[0], 50, 50)
    z = torch.zeros((50, 9 * 4), device=DEV)
    with pytest.raises(pg.PygError):  # 9 heads > 8
        pg.pyg_gat_propagate(z, torch.zeros((50, 9), device=DEV), torch.zeros((50, 9), device=DEV), 9, plan)
    with pytest.raises(pg.PygError):  # forward plan given where a scatter plan is required
        pg.pyg_segment_softmax(torch.zeros((300, 1), device=DEV), plan, 50)
    splan = pg.pyg_plan_build(ei[1], None, 50)
    with pytest.raises(pg.PygError):  # more than 8 columns
        pg.pyg_segment_softmax(torch.zeros((300, 9), device=DEV), splan, 50)


def test_gat_empty_graph_and_single_edge():
    """Degenerate cases: E = 0 (every segment empty -> out 0, all gradients 0) and one edge
    (alpha = 1, out = z_j, d alpha = 0 -> zero attention gradients)."""
    import paper_1903_02428_b200 as pg

    n, H, C = 10, 2, 4
    z = torch.randn((n, H * C), device=DEV)
    ss = torch.randn((n, H), device=DEV)
    sd = torch.randn((n, H), device=DEV)
    g = torch.randn((n, H * C), device=DEV)
    ei = torch.zeros((2, 0), dtype=torch.int64, device=DEV)
    plan = pg.pyg_plan_build(ei[1], ei[0], n, n)
    planT = pg.pyg_plan_build(ei[0], ei[1], n, n)
    out, alpha = pg.pyg_gat_propagate(z, ss, sd, H, plan)
    assert alpha.shape == (0, H) and torch.equal(out, torch.zeros_like(out))
    gr = pg.pyg_gat_backward(z, ss, sd, H, alpha, g, plan, planT)
    for k in ("z", "s_src", "s_dst"):
        assert torch.equal(gr[k], torch.zeros_like(gr[k])), k
    ei1 = torch.tensor([[3], [7]], device=DEV)
    plan1 = pg.pyg_plan_build(ei1[1], ei1[0], n, n)
    planT1 = pg.pyg_plan_build(ei1[0], ei1[1], n, n)
    out1, a1 = pg.pyg_gat_propagate(z, ss, sd, H, plan1)
    assert torch.equal(a1, torch.ones_like(a1))
    assert torch.equal(out1[7], z[3]) and torch.equal(out1[:7], torch.zeros_like(out1[:7]))
    gr1 = pg.pyg_gat_backward(z, ss, sd, H, a1, g, plan1, planT1)
    assert torch.equal(gr1["z"][3], g[7])
    assert gr1["s_src"].abs().max().item() == 0 and gr1["s_dst"].abs().max().item() == 0


@pytest.mark.parametrize("fused", ["0", "1"])
def test_gat_backward_one_pass_single_in_edge(fused, monkeypatch):
    """The one-pass backward takes t_i = g_i . out_i in the SDDMM's own product order and reduction
    tree.  Rows with one in-edge have alpha = 1, so the chain rule gives dlogit = 0 (softmax over one
    element is constant): with the two-pass forward (fused = "0": out_i = 1 * z_j bitwise) it is 0
    EXACTLY; with the one-pass forward out_i = (p z_j) / p can differ from z_j in the last bit, so
    dlogit is 0 only to within rounding (checked through grad_s_dst against the oracle's bound).
    Every row matches the oracle."""
    import paper_1903_02428_b200 as pg

    monkeypatch.setenv("PYG_SEG_TMA", "1")
    monkeypatch.setenv("PYG_GAT_FUSED", fused)
    rng = np.random.default_rng(5)
    n, H, C = 3000, 8, 16
    dst = np.concatenate([np.arange(1000), rng.integers(1000, n, 20000)])  # rows 0..999: one in-edge
    src = rng.integers(0, n, dst.size)
    ei = np.stack([src, dst]).astype(np.int64)
    z = rng.standard_normal((n, H * C)).astype(np.float32)
    ss = rng.standard_normal((n, H)).astype(np.float32)
    sd = rng.standard_normal((n, H)).astype(np.float32)
    g = rng.standard_normal((n, H * C)).astype(np.float32)
    eit = _t(ei)
    plan = pg.pyg_plan_build(eit[1], eit[0], n, n)
    planT = pg.pyg_plan_build(eit[0], eit[1], n, n)
    out, alpha = pg.pyg_gat_propagate(_t(z), _t(ss), _t(sd), H, plan)
    gr = pg.pyg_gat_backward(_t(z), _t(ss), _t(sd), H, alpha, _t(g), plan, planT, out=out)
    # positions of rows 0..999 are the first 1000 edges (edge id = position in dst order)
    if fused == "0":
        assert torch.equal(gr["logit"][:1000], torch.zeros_like(gr["logit"][:1000]))
        assert torch.equal(gr["s_dst"][:1000], torch.zeros_like(gr["s_dst"][:1000]))
    ref = oracle.gat_backward(z, ss, sd, ei, H, g, n_dst=n, with_abs=True)
    check_close(gr["s_dst"].cpu().numpy(), ref["s_dst"], abs_sum=ref["abs_s_dst"], what="grad_s_dst")
    check_close(gr["s_src"].cpu().numpy(), ref["s_src"], abs_sum=ref["abs_s_src"], what="grad_s_src")
