"""The N > 1 path of bench.py (dst-range partition, all-gather or halo exchange, max-over-ranks
timing, the JSON contract) with two ranks on one GPU: --dist-backend gloo stages the exchange
through host memory (NCCL refuses two ranks on one device).  The production N > 1 runs use NCCL
over NVLink; this checks everything around the collective."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,exchange,reduce,extra", [
    ("cora", "allgather", "sum", []), ("cora", "halo", "max", []), ("pubmed", "auto", "mean", []),
    ("cora", "push", "sum", []),
    # source-blocked plan: shard-aligned blocks, per-owner broadcasts overlapped with the block passes
    ("cora", "auto", "max", ["--col-block", "500"]), ("pubmed", "allgather", "sum", ["--col-block", "3000"])])
def test_bench_two_ranks(cfg, exchange, reduce, extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--config", cfg, "--reduce", reduce, "--steps", "3", "--warmup", "3", "--dist-backend", "gloo",
           "--exchange", exchange] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dst-range x2"
    want = {"allgather": "allgather", "halo": "halo", "push": "push"}.get(exchange)
    if extra:
        want = "allgather-overlap"
    if want:
        assert d["config"]["exchange"] == want
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    for k in ("roofline", "clocks", "steps", "warmup", "metric", "unit"):
        assert k in d
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0  # the N > 1 end-to-end leg


@pytest.mark.parametrize("cfg,reduce,extra", [("cora", "sum", []), ("cora", "max", ["--col-block", "500"]),
                                              ("clouds", "max", [])])
def test_bench_dist_capi_world1(cfg, reduce, extra):
    """bench.py's multi-GPU product path (the library's pyg_dist_* layer, NCCL inside libpygs) at N = 1:
    the same JSON contract, and the oracle pre-check on the sampled rows passes."""
    cmd = [sys.executable, "bench.py", "--config", cfg, "--reduce", reduce, "--steps", "3", "--warmup", "3",
           "--dist-capi", "--cpu-seconds", "1", "--no-variants"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    d = json.loads(lines[-1])
    assert d["config"]["exchange"].startswith("capi-allgather"), d["config"]
    assert d["cpu_baseline"]["parity_on_sample"] is True
    assert d["value"] > 0 and d["gpu_launches"] > 0
