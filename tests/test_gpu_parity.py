"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on seeded inputs that span several tiles and ragged tails, plus the edge cases
(empty rows, E = 0, ties, split hub rows, bipartite, strided rows).

Tolerances (tests/tolerance.py): fp32 sum/mean |got-ref| <= 1e-5|ref| + 1e-6
(north_star) for non-negative data, the conditioned bound 1e-5*S + 1e-6 for signed data;
max values, argmax, degrees, plans, collate: exact.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from tests.tolerance import check_close, check_exact

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def pg():
    import paper_1903_02428_b200 as pg

    return pg


def T(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    return t if dtype is None else t.to(dtype)


def H(t):
    return t.detach().cpu().numpy()


def rand_graph(rng, n_src, n_dst, E):
    return np.stack([rng.integers(0, n_src, E), rng.integers(0, n_dst, E)]).astype(np.int64)


def strided(x, ld):
    """Device copy of x with row stride ld (zero padding)."""
    n, F = x.shape
    buf = torch.zeros((n, ld), dtype=torch.float32, device=DEV)
    buf[:, :F] = T(x)
    return buf[:, :F]


def compare(res, ref, red, abs_sum=None, what=""):
    if red == "max":
        check_exact(H(res[0]), ref[0], what + " max values")
        check_exact(H(res[1]), ref[1], what + " argmax")
    else:
        check_close(H(res), ref, abs_sum=abs_sum, what=what)


# ----------------------------------------------------------------------------- scatter

def test_scatter_printed_examples(pg):
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scatter_spec_examples.json")))
    for c in g["cases"]:
        src = T(np.array(c["src"], np.float32))
        idx = T(np.array(c["index"], np.int64))
        plan = pg.pyg_plan_build(idx, None, c["dim_size"])
        for p in (plan, None):
            res = pg.pyg_scatter(src, idx, c["dim_size"], c["reduce"], plan=p)
            out = res[0] if isinstance(res, tuple) else res
            check_exact(H(out), np.array(c["out"], np.float32))


@pytest.mark.parametrize("F", [1, 3, 4, 16, 37, 128, 300])
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
@pytest.mark.parametrize("strategy", ["segment", "atomic"])
def test_scatter_random(pg, F, red, strategy):
    rng = np.random.default_rng(F * 7 + len(red))
    E, n = 3000, 211
    idx = rng.integers(0, n, E)
    idx[idx == 5] = 6  # an empty segment
    src = synth.features(E, F, F, signed=(red == "max"))
    res_ref = oracle.scatter(src, idx, n, red, with_abs=True)
    ti = T(idx)
    plan = pg.pyg_plan_build(ti, None, n) if strategy == "segment" else None
    res = pg.pyg_scatter(T(src), ti, n, red, plan=plan)
    if red == "max":
        compare(res, res_ref[:2], red)
    else:
        compare(res, res_ref[0], red, abs_sum=res_ref[1])


def test_scatter_ties_and_signed_zero(pg):
    rng = np.random.default_rng(0)
    for trial in range(20):
        E, n, F = int(rng.integers(1, 400)), int(rng.integers(1, 40)), int(rng.integers(1, 9))
        idx = rng.integers(0, n, E)
        src = rng.integers(-2, 3, (E, F)).astype(np.float32)
        src[rng.random((E, F)) < 0.3] = -0.0
        ref = oracle.scatter(src, idx, n, "max")
        ti = T(idx)
        for p in (pg.pyg_plan_build(ti, None, n), None):
            res = pg.pyg_scatter(T(src), ti, n, "max", plan=p)
            compare(res, ref, "max", what=f"trial {trial}")


def test_scatter_backward(pg):
    rng = np.random.default_rng(3)
    E, n, F = 5000, 300, 20
    idx = rng.integers(0, n, E)
    src = synth.features(E, F, 1, signed=True)
    g = synth.features(n, F, 2, signed=True)
    out, arg = oracle.scatter(src, idx, n, "max")
    ti = T(idx)
    for red in ("sum", "mean", "max"):
        ref = oracle.scatter_backward(g, idx, red, arg=arg if red == "max" else None)
        got = pg.pyg_scatter_backward(T(g), ti, red, arg_out=T(arg) if red == "max" else None)
        check_exact(H(got), ref, red)  # pure gather / IEEE divide: bitwise


# ----------------------------------------------------------------------------- propagate

CASES = [
    # (n_src, n_dst, E, F, ld)
    (50, 40, 0, 8, None),
    (1, 1, 5, 1, None),
    (300, 257, 2000, 2, None),
    (300, 300, 4000, 5, None),
    (1000, 900, 20000, 16, None),
    (500, 400, 6000, 33, 36),
    (400, 400, 5000, 64, None),
    (200, 150, 3000, 130, 132),
    (150, 120, 2500, 602, 608),
    (150, 120, 2500, 602, None),
    (80, 60, 900, 2100, None),
    (500, 200, 20000, 16, None),   # few rows, degree 100: rows split above 32 positions (Fig. 3 regime)
    (700, 300, 30000, 130, 132),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
@pytest.mark.parametrize("strategy", ["segment", "atomic"])
def test_propagate_random(pg, case, red, strategy):
    n_src, n_dst, E, F, ld = case
    rng = np.random.default_rng(E + F)
    ei = rand_graph(rng, n_src, n_dst, E)
    x = synth.features(n_src, F, F, signed=(red == "max"))
    w = rng.random(E).astype(np.float32) if (E % 2 == 0) else None
    ref = oracle.propagate(x, ei, n_dst=n_dst, reduce=red, edge_weight=w, with_abs=True)
    tei = T(ei)
    xs = strided(x, ld) if ld else T(x)
    plan = pg.pyg_plan_build(tei[1], tei[0], n_dst, n_src) if strategy == "segment" else None
    res = pg.pyg_propagate(xs, tei, n_dst=n_dst, reduce=red, edge_weight=T(w) if w is not None else None, plan=plan)
    if red == "max":
        compare(res, ref[:2], red)
    else:
        compare(res, ref[0], red, abs_sum=ref[1])


@pytest.mark.parametrize("red", ["sum", "mean", "max"])
@pytest.mark.parametrize("strategy", ["segment", "atomic"])
def test_propagate_concat_and_edge_attr(pg, red, strategy):
    rng = np.random.default_rng(11)
    n_src, n_dst, E, F, D = 400, 300, 7000, 12, 5
    ei = rand_graph(rng, n_src, n_dst, E)
    x = synth.features(n_src, F, 1, signed=True)
    xd = synth.features(n_dst, F, 2, signed=True)
    ea = synth.features(E, D, 3, signed=True)
    w = rng.random(E).astype(np.float32)
    ref = oracle.propagate(x, ei, n_dst=n_dst, reduce=red, edge_weight=w, edge_attr=ea, x_dst=xd, concat_xi=True,
                           with_abs=True)
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], n_dst, n_src) if strategy == "segment" else None
    res = pg.pyg_propagate(T(x), tei, n_dst=n_dst, reduce=red, edge_weight=T(w), edge_attr=T(ea), x_dst=T(xd),
                           concat_xi=True, plan=plan)
    if red == "max":
        compare(res, ref[:2], red)
    else:
        compare(res, ref[0], red, abs_sum=ref[1])


def test_integer_sums_bitwise_across_strategies(pg):
    """|x| <= 8 integers: every partial sum is exact => atomic == segment == oracle bitwise."""
    rng = np.random.default_rng(5)
    ei = rand_graph(rng, 2000, 1500, 40000)
    x = rng.integers(-8, 9, (2000, 24)).astype(np.float32)
    ref = oracle.propagate(x, ei, n_dst=1500, reduce="sum")
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], 1500, 2000)
    for p in (plan, None):
        check_exact(H(pg.pyg_propagate(T(x), tei, n_dst=1500, reduce="sum", plan=p)), ref)


def test_split_hub_rows(pg):
    """Rows longer than the split threshold (power-law hubs) go through chunk partials + fp64 combine."""
    rng = np.random.default_rng(9)
    n, F = 3000, 20
    E_uni = 30000
    hubs = np.array([7, 100, 2999])
    hub_deg = np.array([2049, 9000, 25000])
    src = np.concatenate([rng.integers(0, n, E_uni)] + [rng.integers(0, n, d) for d in hub_deg])
    dst = np.concatenate([rng.integers(0, n, E_uni)] + [np.full(d, h) for h, d in zip(hubs, hub_deg)])
    p = rng.permutation(src.size)
    ei = np.stack([src[p], dst[p]]).astype(np.int64)
    x = synth.features(n, F, 4)
    xs = synth.features(n, F, 5, signed=True)
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], n, n)
    v = plan.view()
    deg = np.bincount(ei[1], minlength=n)
    heavy = deg[deg > v["heavy_threshold"]]
    assert v["n_heavy_rows"] == 3 and v["n_heavy_chunks"] == int((-(-heavy // v["chunk_size"])).sum())
    for red in ("sum", "mean"):
        ref, ab = oracle.propagate(x, ei, reduce=red, with_abs=True)
        compare(pg.pyg_propagate(T(x), tei, reduce=red, plan=plan), ref, red)
    ref = oracle.propagate(xs, ei, reduce="max")
    compare(pg.pyg_propagate(T(xs), tei, reduce="max", plan=plan), ref, "max")
    # slices that cut through the hub list
    for lo, hi in ((0, 50), (50, 2999), (2999, 3000), (0, 3000)):
        sl = plan.slice(lo, hi)
        res = pg.pyg_propagate(T(xs), tei, n_dst=hi - lo, reduce="max", plan=sl)
        check_exact(H(res[0]), ref[0][lo:hi])
        check_exact(H(res[1]), ref[1][lo:hi])


@pytest.mark.parametrize("col_block", [1, 37, 500, 2999])
def test_source_blocked_plan(pg, col_block):
    """Source-blocked plans (one pass per block of sources, accumulating in block order) give the
    oracle's result: sum/mean within tolerance, max/argmax exactly (cross-block ties -> lower id)."""
    rng = np.random.default_rng(col_block)
    n_src, n_dst, F = 3000, 700, 12
    E = 40000
    src = rng.integers(0, n_src, E + 6000)
    dst = np.concatenate([rng.integers(0, n_dst, E), np.full(6000, 5)])  # row 5: a hub split across blocks
    ei = np.stack([src, dst]).astype(np.int64)
    ei = ei[:, rng.permutation(ei.shape[1])]
    x = synth.features(n_src, F, 1)
    xt = rng.integers(-2, 3, (n_src, F)).astype(np.float32)  # tie-heavy for max
    w = rng.random(ei.shape[1]).astype(np.float32)
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], n_dst, n_src, col_block=col_block)
    v = plan.view()
    assert v["n_col_blocks"] == -(-n_src // col_block)
    for red, xx, ww in (("sum", x, w), ("mean", x, None), ("max", xt, None), ("max", xt, w)):
        ref = oracle.propagate(xx, ei, n_dst=n_dst, reduce=red, edge_weight=ww, with_abs=True)
        got = pg.pyg_propagate(T(xx), tei, n_dst=n_dst, reduce=red, edge_weight=T(ww) if ww is not None else None,
                               plan=plan)
        if red == "max":
            compare(got, ref[:2], red, what=f"blocked {col_block}")
        else:
            compare(got, ref[0], red, abs_sum=ref[1], what=f"blocked {col_block}")
        for lo, hi in ((0, 5), (5, 6), (6, 700), (100, 400)):
            sl = plan.slice(lo, hi)
            g2 = pg.pyg_propagate(T(xx), tei, n_dst=hi - lo, reduce=red,
                                  edge_weight=T(ww) if ww is not None else None, plan=sl)
            if red == "max":
                check_exact(H(g2[0]), ref[0][lo:hi]); check_exact(H(g2[1]), ref[1][lo:hi])
            else:
                check_close(H(g2), ref[0][lo:hi], abs_sum=ref[1][lo:hi])
    # concatenated x_i block with sum/mean uses the plan's total degree
    ref = oracle.propagate(x, ei, n_dst=n_dst, reduce="mean", concat_xi=True, x_dst=x[:n_dst])
    got = pg.pyg_propagate(T(x), tei, n_dst=n_dst, reduce="mean", concat_xi=True, x_dst=T(x[:n_dst]), plan=plan)
    check_close(H(got), ref)
    # transposed blocked plan for the backward
    g = synth.features(n_dst, F, 9, signed=True)
    planT = pg.pyg_plan_build(tei[0], tei[1], n_src, n_dst, col_block=max(1, col_block // 4))
    rr = oracle.propagate_backward(x, ei, g, n_dst=n_dst, reduce="mean", edge_weight=w, with_abs=True)
    gr = pg.pyg_propagate_backward(T(x), tei, T(g), reduce="mean", edge_weight=T(w), plan_T=planT)
    check_close(H(gr["x_src"]), rr["x_src"], abs_sum=rr["abs_x_src"])


@pytest.mark.parametrize("F,ld", [(256, 256), (300, 304), (602, 608), (1024, 1024), (257, 260)])
def test_bulk_pipeline_matches_ldg_bitwise_and_oracle(pg, F, ld, monkeypatch):
    """The row-staged bulk-copy kernel (segment_bulk.cu: rows streamed into shared memory with
    cp.async.bulk, mbarrier ring) on source-blocked passes: bitwise equal to the LDG kernel (same
    per-row order, same arithmetic) for sum / weighted sum / mean / max / weighted max, and equal to
    the oracle (max exact, ties across blocks to the lower edge id); includes empty rows, rows with
    one edge and a slice."""
    rng = np.random.default_rng(F)
    n_src, n_dst, E = 2500, 900, 30000
    src = rng.integers(0, n_src, E)
    dst = rng.integers(0, n_dst - 50, E)  # the last 50 rows are empty
    dst[:7] = n_dst - 60  # a few short rows
    ei = np.stack([src, dst]).astype(np.int64)
    buf = np.zeros((n_src, ld), np.float32)
    buf[:, :F] = rng.integers(-3, 4, (n_src, F)).astype(np.float32)  # ties for max
    xb = T(buf)
    x = xb[:, :F]
    xn = buf[:, :F]
    w = (rng.random(E) + 0.5).astype(np.float32)
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], n_dst, n_src, col_block=700)
    assert plan.view()["n_col_blocks"] == 4
    for red, ww in (("sum", None), ("sum", w), ("mean", None), ("max", None), ("max", w)):
        wt = T(ww) if ww is not None else None
        outs = {}
        for mode in ("0", "1"):
            monkeypatch.setenv("PYG_SEG_BULK", mode)
            outs[mode] = pg.pyg_propagate(x, tei, n_dst=n_dst, reduce=red, edge_weight=wt, plan=plan)
            sl = plan.slice(100, 850)
            outs[mode + "s"] = pg.pyg_propagate(x, tei, n_dst=750, reduce=red, edge_weight=wt, plan=sl)
        ref = oracle.propagate(xn, ei, n_dst=n_dst, reduce=red, edge_weight=ww, with_abs=True)
        for k in ("", "s"):
            a, b = outs["0" + k], outs["1" + k]
            if red == "max":
                check_exact(H(b[0]), H(a[0])); check_exact(H(b[1]), H(a[1]))
            else:
                check_exact(H(b), H(a))
        if red == "max":
            check_exact(H(outs["1"][0]), ref[0]); check_exact(H(outs["1"][1]), ref[1])
            check_exact(H(outs["1s"][1]), ref[1][100:850])
        else:
            check_close(H(outs["1"]), ref[0], abs_sum=ref[1])


@pytest.mark.parametrize("F", [64, 128, 200, 500, 602])
def test_tma_pipeline_matches_ldg_bitwise_and_oracle(pg, F, monkeypatch):
    """The TMA gather4 pipeline accumulates in the same order with the same arithmetic as the LDG
    kernel: outputs must be bitwise identical, and equal the oracle within tolerance (max exact).
    Graph: power-law (R-MAT) with hubs above the split threshold, many empty rows, weights.
    (PYG_SEG_TMA=1 forces the pipeline on this small graph; auto mode needs >= 1024 tasks.)"""
    monkeypatch.setenv("PYG_SEG_TMA", "1")
    N = 6000
    ei = synth.rmat_edges_np(scale=13, E=150000, N=N, seed=F)
    tei = T(ei)
    rng = np.random.default_rng(F)
    w = rng.random(ei.shape[1]).astype(np.float32)
    ld = (F + 7) // 8 * 8
    x = synth.features(N, F, F, signed=True)
    xs = strided(x, ld)
    plan = pg.pyg_plan_build(tei[1], tei[0], N, N)
    v = plan.view()
    assert v["n_heavy_rows"] > 0
    for red in ("sum", "mean", "max"):
        for ww in (None, w):
            tw = T(ww) if ww is not None else None
            a = pg.pyg_propagate(xs, tei, reduce=red, edge_weight=tw, plan=plan)
            b = pg.pyg_propagate(xs, tei, reduce=red, edge_weight=tw, plan=plan, flags=pg.NO_TMA)
            if red == "max":
                check_exact(H(a[0]).view(np.uint32), H(b[0]).view(np.uint32), "tma vs ldg max")
                check_exact(H(a[1]), H(b[1]), "tma vs ldg arg")
            else:
                check_exact(H(a).view(np.uint32), H(b).view(np.uint32), f"tma vs ldg {red}")
        ref = oracle.propagate(x, ei, reduce=red, edge_weight=w, with_abs=True)
        got = pg.pyg_propagate(xs, tei, reduce=red, edge_weight=T(w), plan=plan)
        if red == "max":
            compare(got, ref[:2], red)
        else:
            compare(got, ref[0], red, abs_sum=ref[1])
    # slices (multi-GPU partitions) through the TMA path
    ref = oracle.propagate(x, ei, reduce="sum", with_abs=True)
    for lo, hi in ((0, 1), (0, 2999), (2999, 6000), (1234, 4321)):
        got = pg.pyg_propagate(xs, tei, n_dst=hi - lo, reduce="sum", plan=plan.slice(lo, hi))
        check_close(H(got), ref[0][lo:hi], abs_sum=ref[1][lo:hi])


def test_segment_is_deterministic(pg):
    rng = np.random.default_rng(1)
    ei = rand_graph(rng, 5000, 5000, 200000)
    x = synth.features(5000, 48, 1, signed=True)
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], 5000, 5000)
    a = H(pg.pyg_propagate(T(x), tei, reduce="sum", plan=plan))
    b = H(pg.pyg_propagate(T(x), tei, reduce="sum", plan=plan))
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


# ----------------------------------------------------------------------------- backward

@pytest.mark.parametrize("red", ["sum", "mean", "max"])
@pytest.mark.parametrize("strategy", ["segment", "atomic"])
def test_propagate_backward(pg, red, strategy):
    rng = np.random.default_rng(21)
    n_src, n_dst, E, F, D = 700, 500, 12000, 24, 3
    ei = rand_graph(rng, n_src, n_dst, E)
    x = synth.features(n_src, F, 1, signed=True)
    ea = synth.features(E, D, 2, signed=True)
    w = rng.random(E).astype(np.float32)
    _, arg = oracle.propagate(x, ei, n_dst=n_dst, reduce="max", edge_weight=w, edge_attr=ea, concat_xi=True) \
        if red == "max" else (None, None)
    g = synth.features(n_dst, 2 * F + D, 3, signed=True)
    ref = oracle.propagate_backward(x, ei, g, n_dst=n_dst, reduce=red, edge_weight=w, D=D, concat_xi=True, arg=arg,
                                    need_x_dst=True, need_edge_attr=True, need_edge_weight=True, with_abs=True)
    tei = T(ei)
    planT = pg.pyg_plan_build(tei[0], tei[1], n_src, n_dst) if strategy == "segment" else None
    got = pg.pyg_propagate_backward(T(x), tei, T(g), reduce=red, edge_weight=T(w), D=D, concat_xi=True,
                                    arg_out=T(arg) if arg is not None else None, plan_T=planT, need_x_dst=True,
                                    need_edge_attr=True, need_edge_weight=True)
    check_close(H(got["x_src"]), ref["x_src"], abs_sum=ref["abs_x_src"], what="grad x_src")
    check_close(H(got["x_dst"]), ref["x_dst"], what="grad x_dst")
    check_close(H(got["edge_attr"]), ref["edge_attr"], what="grad edge_attr")
    # edge-weight grad: sum over F terms of signed products -> conditioned bound
    xg = np.abs(x[ei[0]]) @ np.ones(F) * np.abs(g[ei[1], F:2 * F]).max(1)
    check_close(H(got["edge_weight"]), ref["edge_weight"], abs_sum=xg * (1 if red != "mean" else 1), what="grad w")


def test_gcn_backward_symmetric_equals_forward(pg):
    """Config-2 invariant: symmetric graph => S^T = S => grad_X = S g."""
    ei, x, g = synth.pubmed_like()
    N = x.shape[0]
    tei = T(ei)
    ei2, w = pg.pyg_gcn_norm(tei, N)
    plan = pg.pyg_plan_build(ei2[1], ei2[0], N, N)
    planT = pg.pyg_plan_build(ei2[0], ei2[1], N, N)
    tg = T(g)
    fwd = H(pg.pyg_propagate(tg, ei2, reduce="sum", edge_weight=w, plan=plan))
    bwd = H(pg.pyg_propagate_backward(None, ei2, tg, n_src=N, F=g.shape[1], reduce="sum", edge_weight=w,
                                      plan_T=planT)["x_src"])
    rei, rw = oracle.gcn_norm(ei, N)
    ref, ab = oracle.propagate(g, rei, reduce="sum", edge_weight=rw, with_abs=True)
    check_close(fwd, ref, abs_sum=ab)
    check_close(bwd, ref, abs_sum=ab)


# ----------------------------------------------------------------------------- structure

def test_plan_matches_oracle_csr(pg):
    rng = np.random.default_rng(2)
    for n, E in ((1, 0), (7, 1), (1000, 30000), (70000, 300000)):
        ei = rand_graph(rng, n, n, E)
        tei = T(ei)
        plan = pg.pyg_plan_build(tei[1], tei[0], n, n)
        rowptr, col, perm = plan.export()
        rr, rp = oracle.csr(ei[1], n)
        check_exact(H(rowptr), rr, "rowptr")
        check_exact(H(perm), rp, "perm")
        if E > 0:
            check_exact(H(col), ei[0][rp], "col")
    # already sorted input => identity perm detected
    ei = np.stack([np.arange(100) % 7, np.repeat(np.arange(10), 10)]).astype(np.int64)
    plan = pg.pyg_plan_build(T(ei[1]), T(ei[0]), 10, 7)
    assert plan.view()["perm_is_identity"] == 1


def test_degree(pg):
    rng = np.random.default_rng(4)
    idx = rng.integers(0, 999, 50000)
    check_exact(H(pg.pyg_degree(T(idx), 1000)), oracle.degree(idx, 1000))


def test_gcn_norm_matches_oracle(pg):
    rng = np.random.default_rng(6)
    for N, E, weighted in ((1, 1, False), (2, 2, False), (300, 2000, False), (300, 2000, True)):
        ei = rand_graph(rng, N, N, E)
        if N > 10:
            ei[:, :4] = [[3, 3, 9, 9], [3, 3, 9, 9]]
        w = rng.random(E).astype(np.float32) + 0.5 if weighted else None
        rei, rw = oracle.gcn_norm(ei, N, edge_weight=w)
        ei2, w2 = pg.pyg_gcn_norm(T(ei), N, edge_weight=T(w) if w is not None else None)
        check_exact(H(ei2), rei, "gcn edges")
        check_close(H(w2), rw, rtol=1e-6, atol=0, what="gcn weights")


def test_collate_matches_oracle_and_errors(pg):
    for seed in range(3):
        nn, eptr, local = synth.random_graph_list(13, seed)
        ref = oracle.collate(nn, eptr, local)
        got = pg.pyg_collate(T(nn), T(eptr), T(local), flags=pg.VALIDATE)
        for a, b, nm in zip(got, ref, ("edge_index", "batch", "node_ptr")):
            check_exact(H(a), b, nm)
    nn, eptr, local = synth.random_graph_list(5, 7)
    bad = local.copy()
    bad[1, 0] = nn[0]
    with pytest.raises(pg.PygError) as e:
        pg.pyg_collate(T(nn), T(eptr), T(bad), flags=pg.VALIDATE)
    assert e.value.status == "PYG_ERR_INDEX_OUT_OF_BOUNDS"
    with pytest.raises(pg.PygError) as e:
        pg.pyg_collate(T(np.zeros(0, np.int64)), T(np.zeros(1, np.int64)), T(np.zeros((2, 0), np.int64)))
    assert e.value.status == "PYG_ERR_INVALID_ARGUMENT"


def test_validate_flag_reports_out_of_bounds(pg):
    x = T(np.ones((4, 2), np.float32))
    bad = T(np.array([[0, 4], [0, 1]], np.int64))
    with pytest.raises(pg.PygError) as e:
        pg.pyg_propagate(x, bad, reduce="sum", flags=pg.VALIDATE)
    assert e.value.status == "PYG_ERR_INDEX_OUT_OF_BOUNDS"
    with pytest.raises(pg.PygError) as e:
        pg.pyg_plan_build(bad[1], bad[0], 4, 4)
    assert e.value.status == "PYG_ERR_INDEX_OUT_OF_BOUNDS"
    # source-blocked plans check the same way (and never write outside their arrays: ADVICE r1)
    big = T(np.array([[0, 1, 2, 3], [0, 1, 2, 1 << 20]], np.int64))
    with pytest.raises(pg.PygError) as e:
        pg.pyg_plan_build(big[1], big[0], 4, 4, col_block=2)
    assert e.value.status == "PYG_ERR_INDEX_OUT_OF_BOUNDS"
    with pytest.raises(pg.PygError) as e:
        pg.pyg_plan_build(bad[1], bad[0], 4, 4, col_block=2)
    assert e.value.status == "PYG_ERR_INDEX_OUT_OF_BOUNDS"
    # after an error the library keeps working, and a validated call is not charged with an
    # earlier call's error
    ok = pg.pyg_propagate(x, T(np.array([[0, 3], [0, 1]], np.int64)), reduce="sum", flags=pg.VALIDATE)
    assert H(ok)[1].tolist() == [1.0, 1.0]
    p2 = pg.pyg_plan_build(T(np.array([1, 1], np.int64)), T(np.array([0, 3], np.int64)), 4, 4, col_block=2)
    assert p2.view()["n_col_blocks"] == 2


def test_global_pool(pg):
    nn, eptr, local = synth.random_graph_list(9, 3, n_range=(0, 50))
    N = int(nn.sum())
    x = synth.features(N, 19, 1, signed=True)
    node_ptr = np.concatenate([[0], np.cumsum(nn)])
    batch = np.repeat(np.arange(9), nn)
    for red in ("sum", "mean", "max"):
        ref = oracle.global_pool(x, batch, 9, red)
        got = pg.pyg_global_pool(T(x), T(node_ptr), red)
        if red == "max":
            check_exact(H(got[0]), ref[0])
            a = ref[1].copy()
            a[a == N] = N
            check_exact(H(got[1]), a)
        else:
            check_close(H(got), ref, abs_sum=oracle.global_pool(np.abs(x), batch, 9, red))


def test_batching_equivalence_on_gpu(pg):
    """batched propagate restricted to a block equals the per-graph propagate."""
    nn, eptr, local = synth.random_graph_list(6, 11)
    ei, batch, node_ptr = pg.pyg_collate(T(nn), T(eptr), T(local))
    N = int(nn.sum())
    x = synth.features(N, 10, 2, signed=True)
    plan = pg.pyg_plan_build(ei[1], ei[0], N, N)
    full_out, full_arg = pg.pyg_propagate(T(x), ei, reduce="max", plan=plan)
    full_out, full_arg = H(full_out), H(full_arg)
    npp = H(node_ptr)
    for g in range(6):
        lo, hi = npp[g], npp[g + 1]
        le = local[:, eptr[g]:eptr[g + 1]]
        o, a = oracle.propagate(x[lo:hi], le, reduce="max")
        check_exact(full_out[lo:hi], o)
        a = np.where(a == le.shape[1], ei.shape[1], a + eptr[g])
        check_exact(full_arg[lo:hi], a)


def test_suggest_col_block_decisions(pg):
    """pyg_plan_suggest_col_block (host logic + the device's L2 size): X that fits one 0.4 x L2
    block -> 0 (one pass); Reddit-shaped reuse (E / n = 492, |X| = 566 MB) -> blocks of about 0.4 x L2; R-MAT-shaped
    low reuse (average degree 20, |X| = 5.1 GB) -> 0, since the extra read+write of out per pass
    costs more than the DRAM it saves."""
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    assert pg.pyg_plan_suggest_col_block(1_000_000, 10_000, 10_000, 512) == 0  # 5 MB of X
    cb = pg.pyg_plan_suggest_col_block(114_615_892, 232_965, 232_965, 608 * 4)
    assert cb > 0
    assert 0.2 * l2 <= cb * 608 * 4 <= 0.45 * l2
    assert pg.pyg_plan_suggest_col_block(200_000_000, 10_000_000, 10_000_000, 128 * 4) == 0
    # a matrix just under L2 (Reddit's GCN-transformed H, 232,965 x 128) is still blocked: a random
    # gather keeps only about half of L2 as reuse capacity
    cb = pg.pyg_plan_suggest_col_block(114_615_892 + 232_965, 232_965, 232_965, 128 * 4)
    assert 0 < cb and cb * 128 * 4 <= 0.45 * l2


@pytest.mark.parametrize("sizes,F", [([1024] * 64, 64), ([0, 100_003, 7, 0, 2048], 19), ([3, 1, 0, 9], 300)])
def test_global_pool_long_segments(pg, sizes, F):
    """The readout with few long segments (the point-cloud batch: 64 x 1,024) and ragged / empty
    ones: one 8-CTA cluster per segment, partials combined through distributed shared memory in
    rank order.  max: exact value and lowest node id on ties (tie-heavy integer data)."""
    nn = np.array(sizes, np.int64)
    N = int(nn.sum())
    rng = np.random.default_rng(len(sizes) + F)
    x = synth.features(N, F, 5, signed=True)
    xt = rng.integers(-3, 4, (N, F)).astype(np.float32)
    node_ptr = np.concatenate([[0], np.cumsum(nn)])
    batch = np.repeat(np.arange(nn.size), nn)
    for red, xx in (("sum", x), ("mean", x), ("max", xt)):
        ref = oracle.global_pool(xx, batch, nn.size, red)
        got = pg.pyg_global_pool(T(xx), T(node_ptr), red)
        if red == "max":
            check_exact(H(got[0]), ref[0])
            check_exact(H(got[1]), ref[1])
        else:
            check_close(H(got), ref, abs_sum=oracle.global_pool(np.abs(xx), batch, nn.size, red))


@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_plan_pass_views_equal_whole_plan(pg, red):
    """pyg_plan_passes: running the source blocks of a blocked plan as consecutive views (in order,
    one stream; what the multi-GPU overlap does as each block's rows arrive) equals one call with the
    whole plan bitwise -- also for a slice of it."""
    rng = np.random.default_rng(3)
    n_src, n_dst, F, E = 4000, 900, 24, 50000
    ei = np.stack([rng.integers(0, n_src, E), rng.integers(0, n_dst, E)]).astype(np.int64)
    x = rng.integers(-3, 4, (n_src, F)).astype(np.float32) if red == "max" else synth.features(n_src, F, 2)
    tei = T(ei)
    plan = pg.pyg_plan_build(tei[1], tei[0], n_dst, n_src, col_block=700)
    nb = plan.view()["n_col_blocks"]
    assert nb == 6
    for p, n, lo in ((plan, n_dst, 0), (plan.slice(100, 700), 600, 100)):
        whole = pg.pyg_propagate(T(x), None, n_dst=n, reduce=red, plan=p, E=E)
        out = torch.empty((n, F), device="cuda")
        arg = torch.empty((n, F), dtype=torch.int64, device="cuda") if red == "max" else None
        for b0, b1 in ((0, 2), (2, 3), (3, 6)):
            pg.pyg_propagate(T(x), None, n_dst=n, reduce=red, plan=p.passes(b0, b1), E=E, out=out, arg_out=arg)
        if red == "max":
            check_exact(H(out), H(whole[0]))
            check_exact(H(arg), H(whole[1]))
        else:
            check_exact(H(out), H(whole))


@pytest.mark.parametrize("F", [16, 64, 37])
@pytest.mark.parametrize("red", ["sum", "mean", "max"])
def test_atomic_target_sorted_high_degree(pg, F, red):
    """Target-sorted ("coalesced") input with in-degree ~100 on the atomic strategy: most 32-edge
    batches of the tile kernel share one target (one RED per batch after a butterfly over the lane
    groups), some straddle two; plus an empty row and weights."""
    rng = np.random.default_rng(F + 3 * len(red))
    n = 400
    deg = rng.integers(60, 140, n)
    deg[7] = 0
    dst = np.repeat(np.arange(n), deg)
    src = rng.integers(0, n, dst.size)
    ei = np.stack([src, dst]).astype(np.int64)
    x = synth.features(n, F, F + 1, signed=(red == "max"))
    w = rng.random(dst.size).astype(np.float32)
    for ew in (None, w):
        ref = oracle.propagate(x, ei, reduce=red, edge_weight=ew, with_abs=True)
        got = pg.pyg_propagate(T(x), T(ei), reduce=red, edge_weight=None if ew is None else T(ew), plan=None)
        if red == "max":
            compare(got, ref[:2], red, what="sorted atomic")
        else:
            compare(got, ref[0], red, abs_sum=ref[1], what="sorted atomic")
