"""The seeded generators produce the shapes and structure DESIGN.md's input recipe states."""
import numpy as np

import synth


def test_cora_shape():
    ei, x = synth.cora_like()
    assert ei.shape == (2, 10556) and x.shape == (2708, 16)
    assert (ei[0] != ei[1]).all()
    assert x.min() >= 0 and x.max() < 1
    ei2, _ = synth.cora_like()
    assert np.array_equal(ei, ei2)  # deterministic


def test_pubmed_symmetric_no_loops_no_dups():
    ei, x, g = synth.pubmed_like()
    assert ei.shape == (2, 88648) and x.shape == (19717, 500)
    pairs = set(zip(ei[0].tolist(), ei[1].tolist()))
    assert len(pairs) == 88648
    assert all((b, a) in pairs for a, b in pairs)
    assert (ei[0] != ei[1]).all()
    assert g.min() < 0 < g.max()


def test_clouds_knn():
    nn, eptr, local = synth.knn_cloud_edges(G=2, P=64, k=16, seed=3)
    assert local.shape == (2, 2 * 64 * 16)
    for g in range(2):
        le = local[:, eptr[g]:eptr[g + 1]]
        assert (np.bincount(le[1], minlength=64) == 16).all()
        assert (le[0] != le[1]).all()
        assert (np.diff(le[1]) >= 0).all()  # ordered by target


def test_rmat_small():
    ei = synth.rmat_edges_np(scale=12, E=20000, N=3000, seed=5)
    assert ei.shape == (2, 20000)
    assert ei.min() >= 0 and ei.max() < 3000
    deg = np.bincount(ei[1], minlength=3000)
    assert deg.max() > 20 * deg.mean()  # skewed


def test_erdos_renyi_degree():
    ei = synth.erdos_renyi(10000, 8.0, seed=1)
    assert abs(ei.shape[1] / 10000 - 8.0) < 0.8
    assert (ei[0] != ei[1]).all()
