"""GPU parity of the tcgen05 TF32 dense transform (NEXT-2) against the fp64 oracle.
Tolerance from the arithmetic (A7): TF32 keeps 10 mantissa bits of each operand, so
|got - ref| <= 2.5e-3 * sum_k |x_k w_k| + 1e-6 (2^-9 = 1.95e-3 plus fp32 accumulation)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerance import check_close

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TF32_RTOL = 2.5e-3


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("M,K,N", [(19717, 500, 16), (300, 37, 3), (1000, 64, 64), (129, 128, 128),
                                   (4096, 602, 256), (5, 8, 100), (2708, 1433, 16),
                                   (1000, 64, 300), (300, 128, 600), (129, 37, 513)])  # N > 256: column tiles
@pytest.mark.parametrize("epi", ["plain", "bias_scale"])
def test_dense_transform(M, K, N, epi):
    import paper_1903_02428_b200 as pg

    rng = np.random.default_rng(M + K + N)
    x = rng.standard_normal((M, K)).astype(np.float32)
    w = (rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.standard_normal(N).astype(np.float32) if epi != "plain" else None
    rs = rng.random(M).astype(np.float32) if epi != "plain" else None
    ref, ab = oracle.dense_transform(x, w, bias=b, row_scale=rs, with_abs=True)
    ldk = (K + 3) // 4 * 4  # TMA needs 16-byte row strides: pad K
    xb = torch.zeros((M, ldk), device=DEV)
    xb[:, :K] = _t(x)
    wb = torch.zeros((N, ldk), device=DEV)
    wb[:, :K] = _t(w)
    got = pg.pyg_dense_transform(xb[:, :K], wb[:, :K], bias=None if b is None else _t(b),
                                 row_scale=None if rs is None else _t(rs))
    check_close(got.cpu().numpy(), ref, abs_sum=ab, rtol=TF32_RTOL, what=f"transform {M}x{K}x{N}")


def test_gcn_layer_transform_then_propagate():
    """A GCN layer S (X W^T) on the PubMed-shaped graph: transform on the tensor cores, then the
    GCN-weighted propagate; against the oracle's fp64 transform + propagate, with the TF32 bound
    carried through the (non-negative) propagation weights."""
    import paper_1903_02428_b200 as pg

    ei_np, x_np, _ = synth.pubmed_like()
    N = x_np.shape[0]
    rng = np.random.default_rng(9)
    w = (rng.standard_normal((16, 500)) / 20).astype(np.float32)
    ei, wg = pg.pyg_gcn_norm(_t(ei_np), N)
    plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
    xb = torch.zeros((N, 500), device=DEV)
    xb[:] = _t(x_np)
    h = pg.pyg_dense_transform(xb, _t(w))
    out = pg.pyg_propagate(h, None, reduce="sum", plan=plan, edge_weight=wg, E=ei.shape[1])
    href, hab = oracle.dense_transform(x_np, w, with_abs=True)
    rei, rw = ei.cpu().numpy(), wg.cpu().numpy()
    ref = oracle.propagate(href, rei, reduce="sum", edge_weight=rw)
    bound = oracle.propagate(hab.astype(np.float32), rei, reduce="sum", edge_weight=rw)
    s_abs = oracle.propagate(np.abs(href), rei, reduce="sum", edge_weight=rw)
    got = out.cpu().numpy()
    assert (np.abs(got - ref) <= TF32_RTOL * bound + 1e-5 * s_abs + 1e-6).all()


def test_dense_transform_errors():
    import paper_1903_02428_b200 as pg

    x = torch.zeros((10, 8), device=DEV)
    with pytest.raises(pg.PygError):  # GAT projections need the heads in one 256-column tile
        pg.pyg_gat_transform(x, torch.zeros((300, 8), device=DEV), torch.zeros(300, device=DEV),
                             torch.zeros(300, device=DEV), 5)
    with pytest.raises(pg.PygError):
        pg.pyg_dense_transform(torch.zeros((10, 9), device=DEV)[:, 1:], torch.zeros((4, 8), device=DEV))  # unaligned


@pytest.mark.parametrize("blocked", [False, True])
@pytest.mark.parametrize("cfg", ["cora", "pubmed", "rmat_hubs"])
def test_gcn_layer_fused_normalisation(cfg, blocked, monkeypatch):
    """pyg_gcn_layer (transform with D^-1/2 rows on the tensor cores, unweighted aggregation over A+I
    with a D^-1/2 row scale and the bias in the epilogue) against the oracle's gcn_norm-weighted
    propagate of its fp64 transform, plus bias.  blocked: a source-blocked plan (several
    L2-resident passes; D^-1/2 from the plan's total degree, epilogue in the last pass)."""
    import paper_1903_02428_b200 as pg

    if cfg == "cora":
        ei_np, x_np = synth.cora_like()
        x_np = np.concatenate([x_np, x_np[:, :4]], axis=1)  # K = 20
    elif cfg == "pubmed":
        ei_np, x_np, _ = synth.pubmed_like()
    else:  # hub rows > 2048 (split + fp64 combine with the epilogue), TMA path forced
        monkeypatch.setenv("PYG_SEG_TMA", "1")
        ei_np = synth.rmat_edges_np(scale=12, E=300000, N=4096, seed=31)
        x_np = synth.features(4096, 64, 32)
    N, K = x_np.shape
    F_out = 64 if cfg != "pubmed" else 16
    rng = np.random.default_rng(K)
    w = (rng.standard_normal((F_out, K)) / np.sqrt(K)).astype(np.float32)
    b = rng.standard_normal(F_out).astype(np.float32)
    ei2, _ = pg.pyg_gcn_norm(_t(ei_np), N)
    plan = pg.pyg_plan_build(ei2[1], ei2[0], N, N, col_block=(N // 5 + 1) if blocked else 0)
    if blocked:
        assert plan.view()["n_col_blocks"] >= 5
    ldk = (K + 3) // 4 * 4
    xb = torch.zeros((N, ldk), device=DEV)
    xb[:, :K] = _t(x_np)
    wb = torch.zeros((F_out, ldk), device=DEV)
    wb[:, :K] = _t(w)
    got = pg.pyg_gcn_layer(xb[:, :K], wb[:, :K], plan, bias=_t(b)).cpu().numpy()
    rei, rw = oracle.gcn_norm(ei_np, N)
    h, hab = oracle.dense_transform(x_np, w, with_abs=True)
    ref = oracle.propagate(h, rei, reduce="sum", edge_weight=rw) + b
    bound = oracle.propagate(hab.astype(np.float32), rei, reduce="sum", edge_weight=rw)
    s_abs = oracle.propagate(np.abs(h), rei, reduce="sum", edge_weight=rw) + np.abs(b)
    err = np.abs(got - ref) - (TF32_RTOL * bound + 1e-5 * s_abs + 1e-6)
    assert (err <= 0).all(), float(err.max())


def test_dense_transform_degenerate_shapes():
    """M = 1 (one row of a 128-row tile), K = 1 (one 32-wide K block, zero-filled), N = 1, and an
    exactly representable case (small integers: the TF32 products and sums are exact)."""
    import paper_1903_02428_b200 as pg

    x = torch.zeros((1, 4), device=DEV)
    x[0, 0] = 3.0
    w = torch.zeros((1, 4), device=DEV)
    w[0, 0] = -2.0
    y = pg.pyg_dense_transform(x[:, :1], w[:, :1], bias=torch.tensor([0.5], device=DEV))
    assert y.shape == (1, 1) and y.item() == -5.5
    xi = torch.randint(-4, 5, (300, 40), device=DEV).float()
    wi = torch.randint(-4, 5, (24, 40), device=DEV).float()
    assert torch.equal(pg.pyg_dense_transform(xi, wi), (xi.double() @ wi.double().T).float())


@pytest.mark.parametrize("M,K,H,C", [(2708, 1433, 8, 8), (1000, 64, 4, 16), (333, 100, 1, 64), (130, 36, 8, 32)])
def test_gat_transform_fused_projections(M, K, H, C):
    """pyg_gat_transform: z = x W^T (TF32 bound, A7) and the per-head attention projections
    s = z . a fused into the epilogue, against the fp64 oracle transform contracted with a."""
    import paper_1903_02428_b200 as pg

    rng = np.random.default_rng(M + H)
    x = rng.standard_normal((M, K)).astype(np.float32)
    w = (rng.standard_normal((H * C, K)) / np.sqrt(K)).astype(np.float32)
    a_s = rng.standard_normal(H * C).astype(np.float32)
    a_d = rng.standard_normal(H * C).astype(np.float32)
    ref, ab = oracle.dense_transform(x, w, with_abs=True)
    ldk = (K + 3) // 4 * 4
    xb = torch.zeros((M, ldk), device=DEV)
    xb[:, :K] = _t(x)
    wb = torch.zeros((H * C, ldk), device=DEV)
    wb[:, :K] = _t(w)
    z, ss, sd = pg.pyg_gat_transform(xb[:, :K], wb[:, :K], _t(a_s), _t(a_d), H)
    check_close(z.cpu().numpy(), ref, abs_sum=ab, rtol=TF32_RTOL, what="z")
    z64 = ref.astype(np.float64).reshape(M, H, C)
    for got, a in ((ss, a_s), (sd, a_d)):
        a64 = a.astype(np.float64).reshape(H, C)
        want = (z64 * a64).sum(-1)
        bound = TF32_RTOL * (ab.reshape(M, H, C) * np.abs(a64)).sum(-1) + 1e-5 * np.abs(z64 * a64).sum(-1) + 1e-6
        assert (np.abs(got.cpu().numpy() - want) <= bound).all()
