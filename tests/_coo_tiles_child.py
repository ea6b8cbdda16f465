"""Child of test_gpu_coo_tiles.py: runs with PYG_COO_L2_MB=1 so the atomic COO strategy splits the
columns into L2 tiles (coo.cu l2_tile_cols) at sizes the oracle checks in seconds.  Exits non-zero
(assertion) on any mismatch."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1903_02428_b200 as pg  # noqa: E402
import synth  # noqa: E402
from tests.tolerance import check_close, check_exact  # noqa: E402

assert os.environ.get("PYG_COO_L2_MB") == "1" and os.environ.get("PYG_COO_L2_MB_MAX") == "1"
DEV = "cuda:0"


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def H(t):
    return t.detach().cpu().numpy()


def graph(rng, n_src, n_dst, E, hub, hub_deg):
    """Random edges plus one hub row above the split threshold (2048): its edges go through the
    per-(slot, column tile) cursors."""
    ei = np.stack([rng.integers(0, n_src, E), rng.integers(0, n_dst, E)]).astype(np.int64)
    ei[1, rng.choice(E, hub_deg, replace=False)] = hub
    ei[1, ei[1] == 3] = 4  # an empty row
    return ei


# (n, F): F = 100 -> 16-column tiles (ragged 4-column tail, V = 4, 4 lanes per row);
# F = 37 -> V = 1 tiles of 16 columns; F = 300, n = 2000 -> 64-column tiles (16 lanes), 44-column tail
cases = [(5000, 100), (5000, 37), (2000, 300)]
for n, F in cases:
    rng = np.random.default_rng(n + F)
    E = 40000
    ei = graph(rng, n, n, E, hub=11, hub_deg=5000)
    x = synth.features(n, F, F, signed=True)
    w = rng.random(E).astype(np.float32)
    tei, tx, tw = T(ei), T(x), T(w)
    for red in ("sum", "mean", "max"):
        for ew in (None, w):
            ref = oracle.propagate(x, ei, reduce=red, edge_weight=ew, with_abs=True)
            got = pg.pyg_propagate(tx, tei, reduce=red, edge_weight=None if ew is None else tw, plan=None)
            what = f"atomic L2-tiled n={n} F={F} {red} w={ew is not None}"
            if red == "max":
                check_exact(H(got[0]), ref[0], what + " max")
                check_exact(H(got[1]), ref[1], what + " arg")
            else:
                check_close(H(got), ref[0], abs_sum=ref[1], what=what)
    # scatter of an edge-space src (no gather: only the output slice sizes the tiles)
    src = synth.features(E, F, 5, signed=True)
    for red in ("sum", "max"):
        ref = oracle.scatter(src, ei[1], n, red, with_abs=True)
        got = pg.pyg_scatter(T(src), tei[1].contiguous(), n, red, plan=None)
        if red == "max":
            check_exact(H(got[0]), ref[0], "scatter max")
            check_exact(H(got[1]), ref[1], "scatter arg")
        else:
            check_close(H(got), ref[0], abs_sum=ref[1], what="scatter sum")
    # backward w.r.t. x_src on the atomic path (plan_T NULL): a COO scatter into n_src rows
    g = synth.features(n, F, 9, signed=True)
    for red in ("sum", "mean"):
        ref = oracle.propagate_backward(x, ei, g, reduce=red, edge_weight=w, with_abs=True)
        got = pg.pyg_propagate_backward(tx, tei, T(g), reduce=red, edge_weight=tw, plan_T=None)
        check_close(H(got["x_src"]), ref["x_src"], abs_sum=ref["abs_x_src"], what=f"backward {red}")
    print(f"ok n={n} F={F}")
print("coo tiles ok")
