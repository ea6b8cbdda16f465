"""Atomic COO strategy with L2 column tiles (coo.cu l2_tile_cols) against the oracle.

The tiling switches on when one column's target + gathered rows times F exceed the L2 budget
(PYG_COO_L2_MB, default 72 MB: Reddit's 602 columns run as 19 tiles of 32).  The knob is read once per
process, so the check runs in a child process with a 1 MB budget (both for SUM / MEAN and MAX), where graphs of a few thousand
rows already split into 16- and 64-column tiles with ragged tails and a hub row above the split
threshold; sum / mean / max, weighted and not, scatter and the x_src backward."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("compact", ["2", "0"])
def test_atomic_l2_column_tiles_match_oracle(compact):
    """compact = 2: each tile packs its X columns into a compact scratch and accumulates into a compact
    target (what the default picks for large spans, forced here); 0: the tiles address X / out in place."""
    env = dict(os.environ, PYG_COO_L2_MB="1", PYG_COO_L2_MB_MAX="1", PYG_COO_COMPACT=compact)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_coo_tiles_child.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "coo tiles ok" in r.stdout
