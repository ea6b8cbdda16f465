#!/usr/bin/env python
"""Benchmark of the gather / phi / scatter-reduce hot path (arXiv 1903.02428, Eq. 1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config reddit|rmat|pubmed|clouds|cora] [--reduce sum|mean|max]
                    [--strategy segment|atomic]

Default workload (BASELINE.json config 4, the metric's headline): Reddit-shaped synthetic
graph, N=232,965 nodes, E=114,615,892 iid uniform edges, F=602, mean aggregation
(x'_i = mean_{j in N(i)} x_j), CSR segment-reduce strategy, X rows padded to ldx=608.
A "step" is one pass of the hot path over the batch: gather + phi + reduce + epilogue
(and, for N > 1, the NCCL all-gather of the X shards of the dst-range partition).  The plan
(CSR, "performed as part of the pre-processing") is built once, outside the timed
region, and reported as plan_build_ms; the e2e leg includes it every step.

Metric (BASELINE.json): aggregation edges*F/s (value) and HBM GB/s as a fraction of the
measured peak (roofline).  Inputs (X: 566 MB, indices: 0.9 GB) are larger than the 126 MB
L2, so no flush is needed between steps.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CONFIGS = {
    "reddit": dict(name="reddit-shaped (config 4)", default_reduce="mean"),
    "rmat": dict(name="R-MAT power-law (config 5)", default_reduce="sum"),
    "pubmed": dict(name="PubMed-shaped GCN (config 2)", default_reduce="sum"),
    "clouds": dict(name="batched kNN point clouds (config 3)", default_reduce="max"),
    "cora": dict(name="Cora-shaped (config 1)", default_reduce="sum"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="reddit", choices=list(CONFIGS))
    ap.add_argument("--reduce", default=None, choices=["sum", "mean", "max"])
    ap.add_argument("--strategy", default="segment", choices=["segment", "atomic"])
    ap.add_argument("--op", default="propagate", choices=["propagate", "gat", "gatlayer", "appnp", "gcn"],
                    help="gat: GAT attention aggregation forward + backward (NEXT-1) on the config's graph; "
                         "appnp: K-step APPNP propagation (NEXT-2) with GCN weights")
    ap.add_argument("--K", type=int, default=10, help="appnp: propagation steps")
    ap.add_argument("--hidden", type=int, default=128, help="gcn: output width of the layer's transform")
    ap.add_argument("--alpha", type=float, default=0.1, help="appnp: teleport probability")
    ap.add_argument("--heads", type=int, default=0, help="GAT heads (0: 8)")
    ap.add_argument("--gat-c", type=int, default=0, help="GAT channels per head (0: 8 on citation graphs, F/8 else)")
    ap.add_argument("--ld", type=int, default=0, help="X row stride (0: padded to a multiple of 8 floats)")
    ap.add_argument("--col-block", default="auto",
                    help="source rows per L2-resident pass: auto (pyg_plan_suggest_col_block), 0 (off) or N")
    ap.add_argument("--exchange", default="auto", choices=["auto", "allgather", "halo", "push"],
                    help="N > 1 source exchange: NCCL all-gather of X shards, or halo exchange of only the "
                         "referenced remote rows (auto: halo when it moves < half the all-gather rows); push: "
                         "the halo rows stored into the peers' buffers over NVLink by one kernel (CUDA IPC)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as a CUDA graph (auto: on for the launch-bound L2-resident configs)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo stages the exchange through host memory: only for exercising the N > 1 path "
                         "with several ranks on one GPU (tests); nccl is the measured backend")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N > 1 with a source-blocked plan: one all-gather, then the propagate (no per-owner overlap)")
    ap.add_argument("--dist-capi", action="store_true",
                    help="run the propagate through the library's multi-GPU layer (pyg_dist_*: NCCL inside "
                         "libpygs) also at N = 1 (at N > 1 with NCCL it is the default)")
    ap.add_argument("--dist-python", action="store_true",
                    help="N > 1 with NCCL: the torch.distributed exchange in dist.py instead of pyg_dist_*")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle time for cpu_baseline")
    a = ap.parse_args()
    if a.reduce is None:
        a.reduce = CONFIGS[a.config]["default_reduce"]
    a.warmup = max(a.warmup, 3)
    return a


# --------------------------------------------------------------------------- distributed plumbing

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, local, backend="nccl"):
    if world <= 1:
        return None
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local % max(1, torch.cuda.device_count())))
    else:
        dist.init_process_group(backend)
    return dist


def partition_rows(n, world):
    """Contiguous destination ranges (dst-node partitioning, north_star (3)); padded equal shards."""
    from paper_1903_02428_b200.dist import partition_rows as pr

    return pr(n, world)


# --------------------------------------------------------------------------- workloads

def make_workload(cfg, dev, ld_arg):
    """Returns dict(ei [2,E] int64 cuda, x [N,F] float32 cuda (row stride ld), N, E, F, ld, extra)."""
    if cfg == "reddit":
        F = synth.REDDIT["F"]
        ld = ld_arg or ((F + 7) // 8 * 8)
        ei, x = synth.reddit_like_torch(dev, ld=ld)
        w = None
    elif cfg == "rmat":
        F = synth.RMAT["F"]
        ld = ld_arg or F
        ei = synth.rmat_torch(dev)
        g = torch.Generator(device=dev)
        g.manual_seed(105)
        buf = torch.zeros((synth.RMAT["N"], ld), dtype=torch.float32, device=dev)
        buf[:, :F] = torch.rand((synth.RMAT["N"], F), generator=g, device=dev)
        x = buf[:, :F]
        w = None
    elif cfg == "pubmed":
        ei_np, x_np, _ = synth.pubmed_like()
        F = x_np.shape[1]
        ld = ld_arg or ((F + 7) // 8 * 8)
        buf = torch.zeros((x_np.shape[0], ld), dtype=torch.float32, device=dev)
        buf[:, :F] = torch.from_numpy(x_np).to(dev)
        x = buf[:, :F]
        ei = torch.from_numpy(ei_np).to(dev)
        w = None
    elif cfg == "clouds":
        import paper_1903_02428_b200 as pg

        nn, eptr, local, x_np = synth.clouds_like()
        args = (torch.from_numpy(nn).to(dev), torch.from_numpy(eptr).to(dev), torch.from_numpy(local).to(dev))
        ei, _, _ = pg.pyg_collate(*args)
        # the mini-batch collate (a9) timed on its own: CUDA events, median of 20 calls
        ts = []
        for _ in range(23):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pg.pyg_collate(*args, N_total=int(nn.sum()))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        cms = float(np.median(ts[3:]))
        Et, Nt, G = local.shape[1], int(nn.sum()), nn.size
        cbytes = 2 * (2 * Et * 8) + Nt * 8 + (G + 1) * 8 * 2 + G * 8  # edges in/out, batch, ptrs
        extra = {"collate_ms": cms, "collate_GBps": cbytes / (cms * 1e-3) / 1e9, "collate_alg_bytes": cbytes,
                 "collate_note": "pyg_collate of 64 graphs (1,048,576 edges, 65,536 nodes), incl. binding overhead"}
        x = torch.from_numpy(x_np).to(dev)
        # global max pooling readout over the batch (NEXT-3): 65,536 x 64 -> 64 x 64 (+ arg)
        _, _, node_ptr = pg.pyg_collate(*args)
        ts = []
        for _ in range(23):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pg.pyg_global_pool(x, node_ptr, reduce="max")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        pms = float(np.median(ts[3:]))
        pbytes = x.numel() * 4 + G * x.shape[1] * 12 + (G + 1) * 8
        extra.update({"global_pool_max_ms": pms, "global_pool_GBps": pbytes / (pms * 1e-3) / 1e9,
                      "global_pool_note": "pyg_global_pool max over 64 graphs x 1,024 nodes x 64 features, incl. "
                                          "binding overhead"})
        F = x_np.shape[1]
        ld = F
        w = None
        return dict(ei=ei, x=x, N=x.shape[0], E=ei.shape[1], F=F, ld=ld, w=w, extra=extra)
    else:
        ei_np, x_np = synth.cora_like()
        ei = torch.from_numpy(ei_np).to(dev)
        x = torch.from_numpy(x_np).to(dev)
        F = x_np.shape[1]
        ld = F
        w = None
    return dict(ei=ei, x=x, N=x.shape[0], E=ei.shape[1], F=F, ld=ld, w=w)


def alg_bytes(E, n_dst, F, reduce, strategy, weighted=False):
    """Algorithmic bytes per pass (actual index widths, reading Q13):
    gathered x_j rows + index arrays + output (+ arg for max, + weights)."""
    b = E * F * 4
    if strategy == "segment":
        b += E * 4 + 8 * (n_dst + 1)  # col (int32) + rowptr (int64)
        if reduce == "max" or weighted:
            b += E * 4  # perm (int32) for edge ids
    else:
        b += 16 * E  # COO src + dst (int64)
    if weighted:
        b += 4 * E
    b += n_dst * F * 4
    if reduce == "max":
        b += n_dst * F * 8
    return b


def gat_step_bytes(E, N, F, H):
    """Algorithmic bytes of one GAT aggregation forward + backward (NEXT-1), every array counted once
    per kernel that must read or write it (index widths as stored: int32 col / edge id / row):
      per edge: softmax (two passes: col + edge id + s_src row 4H each, alpha write 4H) 16 + 12H;
                alpha-weighted sum (col, edge id, z row 4F, alpha 4H) 8 + 4F + 4H;
                one-pass backward (col, edge id, row, z row 4F, alpha, s_src, dlogit write) 12 + 4F + 12H;
                grad_z over the transposed plan (col, edge id, grad_out row 4F, alpha) 8 + 4F + 4H;
                grad_s_src (edge id, dlogit row) 4 + 4H;
      per node: out write 4F; t_i = g_i . out_i (g, out, t) 8F + 4H; backward row state (g, t, s_dst,
                grad_s_dst) 4F + 12H; grad_z write 4F; grad_s_src write 4H; s_dst in the softmax 4H;
                rowptrs 2 x 8."""
    per_edge = 48 + 12 * F + 32 * H
    per_node = 20 * F + 24 * H + 16
    return E * per_edge + N * per_node


# --------------------------------------------------------------------------- clocks

class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [s.strip() for s in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def l2_gather_peak():
    """Measured L2 -> SM row-gather bandwidth (scripts/l2peak.cu, committed as profiles/l2_peak.json):
    the roof of a kernel whose gathered matrix (or source block) is L2-resident."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_peak.json")) as f:
            d = json.load(f)
        return float(d["l2_row_gather_gbs"]), "measured (profiles/l2_peak.json l2_row_gather_gbs, scripts/l2peak.cu)"
    except Exception:
        return None, None


def gat_fwd_blocked_ok(C, F):
    """The blocked GAT forward weighs float4 chunks with one head's alpha (C % 4 == 0); rows up to
    PYG_BENCH_GAT_BLOCKED_MAX_F floats (default: the kernel's 1024).  Reddit training step at 8 x 64 with
    the blocked transposed plan: 113.1 ms with the blocked forward, 126.1 ms with the unblocked one-pass
    forward (gpurun_out/r3ao); at 8 x 72 the blocked forward first measured slower (275 vs 257 ms,
    gpurun_out/r3ac) until wide rows kept fewer z rows in flight (251.6 vs 255.5 ms, gpurun_out/r3ad)."""
    return C % 4 == 0 and F <= int(os.environ.get("PYG_BENCH_GAT_BLOCKED_MAX_F", "1024"))


def l2_red_peak():
    """Measured gather + red.global.add.v4 throughput into L2-resident rows (scripts/l2red.cu,
    profiles/l2_red.json): the roof of the atomic strategy once its column tiles fit L2."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_red.json")) as f:
            d = json.load(f)
        return float(d["gather_red_w32_gbs"]), "measured (profiles/l2_red.json gather_red_w32_gbs, scripts/l2red.cu)"
    except Exception:
        return None, None


def _profile_lookup(fname, workload_key):
    """Entry of profiles/<fname> for this workload; the col_block part of the key may differ between
    boxes (it follows the L2 size), so fall back to the same config / reduce / strategy / N."""
    try:
        with open(os.path.join(ROOT, "profiles", fname)) as f:
            d = json.load(f)
    except Exception:
        return None
    if workload_key in d:
        return d[workload_key]
    head, tail = workload_key.split("-cb")[0], workload_key.split("-cb", 1)[-1].split("-", 1)[-1]
    for k, v in d.items():
        if k.startswith(head + "-cb") and k.split("-cb", 1)[-1].split("-", 1)[-1] == tail:
            return v
    return None


def traffic_for(workload_key):
    return _profile_lookup("traffic.json", workload_key)


# --------------------------------------------------------------------------- CPU oracle leg

# The CPU baseline's sample: the in-edges of the first R target rows, R a FIXED fraction of the rows
# per config (the same rows for bench's cpu_baseline and for the --impl reference arm, so both time
# the same work); ~10-15 s of single-threaded oracle work on the large graphs, the whole graph on
# the small ones.  (A full Reddit pass, ~150 s, is timed once by scripts/cpu_full_pass.py and
# reported from profiles/cpu_full_pass.json.)
CPU_SAMPLE_FRAC = {"reddit": 0.05, "rmat": 0.08, "pubmed": 1.0, "clouds": 1.0, "cora": 1.0}


def cpu_sample_rows(cfg, n_rows):
    return max(1, min(n_rows, int(round(n_rows * CPU_SAMPLE_FRAC.get(cfg, 1.0)))))


def host_info():
    """The host cores the oracle ran on (nproc, affinity, CPU model)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"nproc": os.cpu_count(), "affinity": aff, "cpu_model": model}


def full_pass_record(cfg, reduce):
    """The committed full-pass oracle timing for this workload (scripts/cpu_full_pass.py), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "cpu_full_pass.json")) as f:
            return json.load(f).get(f"{cfg}-{reduce}")
    except Exception:
        return None


def oracle_rows(ei_cpu, x_cpu, R, reduce, F, w=None):
    """Time the oracle (as it stands, single-threaded C) on the in-edges of the first R target rows.
    Returns (edges*F/s, seconds, E_s, R, out)."""
    import oracle

    m = ei_cpu[1] < R
    sub = ei_cpu[:, m]
    ws = w[m] if w is not None else None
    t0 = time.perf_counter()
    out = oracle.propagate(x_cpu, sub, n_dst=R, reduce=reduce, edge_weight=ws)
    dt = time.perf_counter() - t0
    return sub.shape[1] * F / dt, dt, sub.shape[1], R, out


def oracle_sample(ei_cpu, x_cpu, n_rows, reduce, target_s, F, w=None):
    """Time the oracle (as it stands) on the edges of the first R target rows, R sized for
    ~target_s seconds from a short calibration run.  Returns (edges*F/s, seconds, E_s, R, out)."""
    import oracle

    dst = ei_cpu[1]

    def run(R):
        m = dst < R
        sub = ei_cpu[:, m]
        ws = w[m] if w is not None else None
        t0 = time.perf_counter()
        out = oracle.propagate(x_cpu, sub, n_dst=R, reduce=reduce, edge_weight=ws)
        dt = time.perf_counter() - t0
        return sub.shape[1], dt, out

    R = max(1, min(n_rows, 256))
    Es, dt, _ = run(R)
    rate = max(Es * F / max(dt, 1e-6), 1.0)
    avg = max(ei_cpu.shape[1] / n_rows, 1e-9)
    R = int(min(n_rows, max(1, target_s * rate / (F * avg))))
    Es, dt, out = run(R)
    return Es * F / dt, dt, Es, R, out


def oracle_gat_sample(ei_cpu, z_cpu, ss, sd, H, n_rows, target_s, F):
    """The GAT oracle (forward) on the in-edges of the first R target rows, R sized for ~target_s."""
    import oracle

    dst = ei_cpu[1]

    def run(R):
        m = dst < R
        sub = ei_cpu[:, m]
        t0 = time.perf_counter()
        res = oracle.gat(z_cpu, ss, sd[:R], sub, H, n_dst=R, with_abs=True)
        return sub.shape[1], time.perf_counter() - t0, res

    R = max(1, min(n_rows, 256))
    Es, dt, _ = run(R)
    rate = max(Es * F / max(dt, 1e-6), 1.0)
    avg = max(ei_cpu.shape[1] / n_rows, 1e-9)
    R = int(min(n_rows, max(1, target_s * rate / (F * avg))))
    Es, dt, res = run(R)
    return Es * F / dt, dt, Es, R, res


def oracle_appnp_run(ei_cpu, x_cpu, w_cpu, K, alpha, target_s, F):
    """The APPNP oracle is a whole-graph recurrence: timed on the full graph when one step of it
    (estimated from one propagate pass over a sample) fits target_s, else on the sample pass only."""
    import oracle

    E = ei_cpu.shape[1]
    n = x_cpu.shape[0]
    rate, dt, Es, R, _ = oracle_sample(ei_cpu, x_cpu, n, "sum", min(2.0, target_s / 4), F, w=w_cpu)
    if E * F * K / rate <= 2 * target_s:
        t0 = time.perf_counter()
        ref = oracle.appnp(x_cpu, ei_cpu, K=K, alpha=alpha, edge_weight=w_cpu)
        dt = time.perf_counter() - t0
        return E * F * K / dt, dt, E * K, n, ref
    return rate, dt, Es, 0, None


def oracle_gcn_sample(ei_cpu, x_cpu, W, b, n_rows, target_s):
    """The oracle GCN layer (fp64 transform of the needed source rows, gcn_norm-weighted propagate, bias)
    on the in-edges of the first R target rows; edges*F counted at the hidden width."""
    import oracle

    ei2, w2 = oracle.gcn_norm(ei_cpu, n_rows)
    dst = ei2[1]
    Fh = W.shape[0]

    def run(R):
        m = dst < R
        sub = ei2[:, m]
        t0 = time.perf_counter()
        srcs = np.unique(sub[0])
        h, hab = oracle.dense_transform(x_cpu[srcs], W, with_abs=True)
        remap = np.zeros(n_rows, np.int64)
        remap[srcs] = np.arange(srcs.size)
        loc = np.stack([remap[sub[0]], sub[1]])
        out = oracle.propagate(h, loc, n_dst=R, reduce="sum", edge_weight=w2[m]) + b
        bound = oracle.propagate(hab.astype(np.float32), loc, n_dst=R, reduce="sum", edge_weight=w2[m])
        s_abs = oracle.propagate(np.abs(h), loc, n_dst=R, reduce="sum", edge_weight=w2[m]) + np.abs(b)
        return sub.shape[1], time.perf_counter() - t0, (out, bound, s_abs)

    R = max(1, min(n_rows, 64))
    Es, dt, _ = run(R)
    rate = max(Es * Fh / max(dt, 1e-6), 1.0)
    avg = max(ei2.shape[1] / n_rows, 1e-9)
    R = int(min(n_rows, max(1, target_s * rate / (Fh * avg))))
    Es, dt, res = run(R)
    return Es * Fh / dt, dt, Es, R, res


def run_reference(a):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    import oracle

    oracle.build()
    cfg = a.config
    # the same workload: the big generators draw on the GPU when there is one (torch's CUDA generator,
    # so the edges are identical to our arm's) and the arrays are copied to the host; smaller ones
    # use numpy.  Nothing of our library runs on this path.
    dev = torch.device("cuda" if (torch.cuda.is_available() and cfg in ("reddit", "rmat")) else "cpu")
    w = make_workload(cfg, dev, a.ld)
    w["ei"], w["x"] = w["ei"].cpu(), w["x"].cpu()
    ei = w["ei"].numpy()
    x = np.ascontiguousarray(w["x"].numpy())
    F, N, E = w["F"], w["N"], w["E"]
    per_step = max(1.0, 150.0 / max(1, a.steps + a.warmup))
    rates = []
    info = None
    # the oracle of the same op as our arm (units: edges x the op's aggregation width)
    rng = np.random.default_rng(110)
    if a.op in ("gat", "gatlayer"):
        H = a.heads or 8
        C = a.gat_c or (8 if cfg in ("cora", "pubmed", "clouds") else max(4, 1 << ((F // H).bit_length() - 1)))
        zc = rng.standard_normal((N, H * C)).astype(np.float32)
        ss = rng.standard_normal((N, H)).astype(np.float32)
        sd = rng.standard_normal((N, H)).astype(np.float32)

        def one():
            return oracle_gat_sample(ei, zc, ss, sd, H, N, per_step, H * C)
        what = f"oracle.gat forward ({H} heads x {C})"
    elif a.op == "gcn":
        W = (rng.standard_normal((a.hidden, F)) / np.sqrt(F)).astype(np.float32)
        b = rng.standard_normal(a.hidden).astype(np.float32)

        def one():
            return oracle_gcn_sample(ei, x, W, b, N, per_step)
        what = f"oracle GCN layer (dense_transform + gcn_norm-weighted propagate), hidden {a.hidden}"
    else:
        R_fix = cpu_sample_rows(cfg, N)
        # the same rows as bench's cpu_baseline; if K + W steps of it would overrun ~150 s, every step
        # takes a proportionally shorter prefix (calibrated once)
        rate0, dt0, _, _, _ = oracle_rows(ei, x, R_fix, a.reduce, F)
        if dt0 * (a.steps + a.warmup) > 150.0:
            R_fix = max(1, int(R_fix * per_step / dt0))

        def one():
            return oracle_rows(ei, x, R_fix, a.reduce, F)
        what = f"oracle.propagate {a.reduce}" + (" (one pass of the K-step APPNP recurrence)" if a.op == "appnp" else "")
    for i in range(a.warmup + a.steps):
        rate, dt, Es, R, _ = one()
        if i >= a.warmup:
            rates.append(rate)
            info = (Es, R, dt)
    v = float(np.mean(rates))
    Es, R, dt = info
    sample = f"{what}: {Es} edges of the first {R} target rows of {N} ({Es / E:.3%} of E), one pass per step"
    Fu = a.hidden if a.op == "gcn" else F
    line = {
        "impl": "reference", "metric": "aggregation edges*F/s", "value": v, "unit": "edges*F/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        # one whole pass of the workload at the sampled rate (the sample itself took sample_ms)
        "ms_per_step": E * Fu / v * 1e3, "sample_ms": dt * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64-accumulate/f32-io",
        "data": "synthetic", "config": {"workload": CONFIGS[cfg]["name"], "N": N, "E": E, "F": F,
                                        "reduce": a.reduce, "op": a.op},
        "cpu_baseline": {"value": v, "unit": "edges*F/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host": host_info(), "full_pass": full_pass_record(cfg, a.reduce)},
        "e2e": {"value": v, "unit": "edges*F/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm

def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    world, rank, local = dist_env()
    if world > 1 and a.gpus != world:
        a.gpus = world
    # several ranks may share one GPU in the gloo test mode (--dist-backend gloo)
    gpu = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist = init_dist(world, local, backend=a.dist_backend)

    import paper_1903_02428_b200 as pg
    from paper_1903_02428_b200.dist import gather_x, halo_exchange

    t0 = time.perf_counter()
    w = make_workload(a.config, dev, a.ld)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    ei, x, N, E, F, ld = w["ei"], w["x"], w["N"], w["E"], w["F"], w["ld"]
    red = a.reduce

    # dst-range partition (N > 1): rank owns targets [lo, hi) and their in-edges; X is sharded by
    # the same ranges and all-gathered every step (NCCL over NVLink).
    ranges, per = partition_rows(N, world)
    # the library's multi-GPU layer (pyg_dist_plan_build / pyg_dist_propagate, NCCL inside libpygs):
    # the product path at N > 1; --dist-capi runs it at N = 1 too
    use_capi = (a.strategy == "segment" and a.op == "propagate" and a.exchange != "push" and
                ((world > 1 and a.dist_backend == "nccl" and not a.dist_python) or a.dist_capi))
    dplan = None

    t0 = time.perf_counter()
    plan_full = None
    col_block = 0
    overlap = False
    if use_capi:
        col_block = pg.pyg_plan_suggest_col_block(E, N, N, ld * 4) if a.col_block == "auto" else int(a.col_block)
        ids = [pg.pyg_dist_unique_id() if rank == 0 else None]
        if dist:
            dist.broadcast_object_list(ids, src=0)
        comm = pg.pyg_dist_init(ids[0], rank, world)
        dplan = pg.pyg_dist_plan_build(comm, ei, N, F, ld, col_block, a.exchange)
        torch.cuda.synchronize()
        col_block = dplan.col_block
        per = dplan.per
        ranges = [(min(q * per, N), min((q + 1) * per, N)) for q in range(world)]
        if world == 1:  # the single-GPU extras below (e2e leg, variants, collate) use a plain plan
            plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=col_block)
    elif a.strategy == "segment":
        if a.col_block == "auto":
            col_block = pg.pyg_plan_suggest_col_block(E, N, N, ld * 4)
        else:
            col_block = int(a.col_block)
        if world > 1 and col_block > 0 and not a.no_overlap and a.exchange in ("auto", "allgather"):
            # source blocks aligned with the shards: block b's rows come from one owner, so its pass can
            # run as soon as that owner's broadcast has landed (dist.OverlappedGather)
            from paper_1903_02428_b200.dist import aligned_partition

            ranges, per, col_block = aligned_partition(N, world, col_block)
            overlap = True
        plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=col_block)
        torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t0) * 1e3
    lo, hi = ranges[rank]
    n_loc = hi - lo
    plan = plan_full.slice(lo, hi) if (plan_full is not None and world > 1) else plan_full
    if a.strategy == "atomic" and world > 1:
        m = (ei[1] >= lo) & (ei[1] < hi)
        ei_loc = ei[:, m].clone()
        ei_loc[1] -= lo
    else:
        ei_loc = ei
    # edges owned by this rank (byte accounting only; source-blocked plans have no single CSR to export)
    E_loc = int(((ei[1] >= lo) & (ei[1] < hi)).sum().item()) if world > 1 else ei_loc.shape[1]

    exchange = "none"
    halo = None
    if world > 1 and plan is not None and col_block == 0 and a.exchange not in ("allgather", "push"):
        from paper_1903_02428_b200.dist import halo_setup

        hplan, hids = pg.pyg_halo_build(plan, N, lo, hi, per)
        nh = torch.tensor([hids.numel()], dtype=torch.int64, device=dev if a.dist_backend == "nccl" else "cpu")
        dist.all_reduce(nh, op=dist.ReduceOp.MAX)
        if a.exchange == "halo" or int(nh.item()) < 0.5 * (world - 1) * per:
            send_rows, sc, rc = halo_setup(hids, lo, per, world)
            halo = dict(plan=hplan, n=hids.numel(), send_rows=send_rows, sc=sc, rc=rc,
                        sendbuf=torch.empty((send_rows.numel(), ld), dtype=torch.float32, device=dev))
    hpush = None
    if world > 1 and a.exchange == "push":
        assert plan is not None and col_block == 0, "--exchange push: segment strategy, unblocked plan"
        from paper_1903_02428_b200.dist import HaloPush

        hpush = HaloPush(plan, N, lo, hi, per, ld, world, rank)
        halo = None
    if hpush is not None:
        exchange = "push"
        hpush.shard[:n_loc] = x.as_strided((N, ld), (x.stride(0), 1))[lo:hi]
        x_full = hpush.xloc[:, :F]
        plan = hpush.plans[0]
        halo = dict(n=hpush.n_halo)
    elif world > 1 and halo is not None:
        exchange = "halo"
        xbuf = torch.zeros((per + halo["n"], ld), dtype=torch.float32, device=dev)
        shard = xbuf[:per]
        shard[:n_loc] = x.as_strided((N, ld), (x.stride(0), 1))[lo:hi]
        x_full = xbuf[:, :F]
        plan = halo["plan"]
    elif use_capi:
        exchange = "capi-" + dplan.exchange + ("-overlap" if (dplan.col_block and world > 1) else "")
        halo = dict(n=dplan.n_halo) if dplan.exchange == "halo" else None
        x_full = dplan.x_shard()  # this rank's rows inside the library's exchange buffer
        x_full.copy_(x.as_strided((N, ld), (x.stride(0), 1))[lo:hi, :F])
    elif world > 1 and overlap:
        from paper_1903_02428_b200.dist import OverlappedGather

        exchange = "allgather-overlap"
        xbuf = torch.zeros((per * world, ld), dtype=torch.float32, device=dev)
        ovg = OverlappedGather(plan, xbuf, per, col_block, world, rank)
        shard = ovg.shard(rank)
        shard[:n_loc] = x.as_strided((N, ld), (x.stride(0), 1))[lo:hi]
        x_full = xbuf[:N, :F]
    elif world > 1:
        exchange = "allgather"
        xbuf = torch.zeros((per * world, ld), dtype=torch.float32, device=dev)
        shard = torch.zeros((per, ld), dtype=torch.float32, device=dev)
        shard[:n_loc] = x.as_strided((N, ld), (x.stride(0), 1))[lo:hi]
        x_full = xbuf[:N, :F]
    else:
        x_full = x
    e2e_host = None
    if world > 1 and not a.no_e2e and a.op == "propagate" and a.strategy == "segment":
        # N > 1 end-to-end leg (below): this rank's X rows and the edge list in pinned host memory
        from paper_1903_02428_b200.dist import partition_rows as _pr

        lo_e, hi_e = _pr(N, world)[0][rank]
        xs_all = x.as_strided((N, ld), (x.stride(0), 1))
        e2e_host = dict(lo=lo_e, hi=hi_e,
                        hx=torch.empty((hi_e - lo_e, ld), dtype=torch.float32, pin_memory=True),
                        hei=torch.empty(ei.shape, dtype=torch.int64, pin_memory=True))
        e2e_host["hx"].copy_(xs_all[lo_e:hi_e])
        e2e_host["hei"].copy_(ei)
        del xs_all
    if world > 1:
        del x  # every rank keeps only its shard (+ the exchange buffer)
        w.pop("x")
        torch.cuda.empty_cache()
    out = torch.empty((n_loc, ((F + 7) // 8 * 8) if a.config == "reddit" else F), dtype=torch.float32,
                      device=dev)[:, :F]
    arg = torch.empty((n_loc, out.stride(0)), dtype=torch.int64, device=dev)[:, :F] if red == "max" else None
    ws = None if use_capi else torch.empty(max(1, pg.pyg_workspace_size(plan, n_loc, F, red, E=ei_loc.shape[1])),
                                           dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    passes, weighted, prep_ms = 1, False, 0.0

    cur = {"plan": plan}

    def one(p):
        pg.pyg_propagate(x_full, None if p is not None else ei_loc, n_dst=n_loc, reduce=red, plan=p, out=out,
                         arg_out=arg, E=E if p is not None else None, workspace=ws)

    def compute():
        if use_capi:  # exchange (all-gather / per-owner broadcasts / halo) + propagate, all in the library
            pg.pyg_dist_propagate(dplan, x_full, red, out=out, arg_out=arg)
        elif exchange == "allgather-overlap":  # the broadcasts and the per-owner passes interleave
            ovg.step(one)
        else:
            one(cur["plan"])

    if a.config == "pubmed" and world == 1:
        # config 2: GCN sym-normalised sum aggregation, forward + backward.  The normalisation
        # (self-loops + D^-1/2 (A+I) D^-1/2 weights) and both plans are per-graph
        # preprocessing, as in a cached GCN layer; the step is the forward propagate plus the
        # backward w.r.t. X (transposed plan).
        t1 = time.perf_counter()
        ei, wgt = pg.pyg_gcn_norm(ei, N)
        E = ei.shape[1]
        plan = plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N) if a.strategy == "segment" else None
        planT = pg.pyg_plan_build(ei[0], ei[1], N, N) if a.strategy == "segment" else None
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - t1) * 1e3
        g = torch.from_numpy(synth.pubmed_like()[2]).to(dev)
        gx = torch.empty((N, F), dtype=torch.float32, device=dev)
        ws = torch.empty(max(1, pg.pyg_workspace_size(plan, N, F, red, E=ei.shape[1])), dtype=torch.uint8, device=dev)
        passes, weighted, red = 2, True, "sum"

        def compute():
            pg.pyg_propagate(x_full, ei, reduce="sum", edge_weight=wgt, plan=plan, out=out, workspace=ws)
            pg.pyg_propagate_backward(None, ei, g, n_src=N, F=F, reduce="sum", edge_weight=wgt, plan_T=planT,
                                      grad_x_src=gx)

    gat = None
    if a.op == "gat":
        # NEXT-1: GAT layer aggregation, forward (segment softmax of leaky_relu(s_src[j] + s_dst[i]),
        # alpha-weighted sum per head) + backward (SDDMM + softmax backward, grad_z over the
        # transposed plan, grad_s_src).  z = the config's X (the transformed features x W); the
        # attention projections s_src / s_dst are seeded inputs (dense per-node ops, outside the path).
        assert world == 1 and a.strategy == "segment", "--op gat: one GPU, segment strategy"
        # z = x W: the GAT paper's 8 heads x 8 channels on the citation graphs, 8 x F/8 on
        # the large graphs; z is a seeded input (the transform is the tcgen05 path, --op gcn)
        H = a.heads or 8
        # (channels per head: the largest power of two <= F / H -- the one-pass TMA forward needs C % 4 == 0
        # and the one-pass backward a power of two; Reddit's 602 columns -> 8 x 64, R-MAT's 128 -> 8 x 16.
        # With 8 x 72 the backward took the two-pass softmax kernel: 167 of a 243 ms step, gpurun_out/r3an)
        C = a.gat_c or (8 if a.config in ("cora", "pubmed", "clouds") else max(4, 1 << ((F // H).bit_length() - 1)))
        t1 = time.perf_counter()
        if plan_full.view()["n_col_blocks"] > 1:
            plan = plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N)
            col_block = 0
        # the transposed plan gathers grad_out rows (n x H*C): source-blocked when they exceed L2
        cb_t = pg.pyg_plan_suggest_col_block(E, N, N, H * C * 4) if a.col_block == "auto" else 0
        planT = pg.pyg_plan_build(ei[0], ei[1], N, N, col_block=cb_t)
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - t1) * 1e3
        gg = torch.Generator(device=dev)
        gg.manual_seed(107)
        s_src = torch.randn((N, H), generator=gg, device=dev) * 2
        s_dst = torch.randn((N, H), generator=gg, device=dev) * 2
        F = H * C
        zc = torch.randn((N, F), generator=gg, device=dev)
        gout = torch.randn((N, F), generator=gg, device=dev)
        gat = dict(H=H, alpha=torch.empty((E, H), device=dev), out=torch.empty((N, F), device=dev))
        # the training step keeps the attention in factored form (alpha = p / row_sums[dst]): the forward's
        # consumer is the backward, which divides where it reads alpha (no E x H normalisation pass)
        # (large graphs only: the small ones take the two-pass kernels, where alpha comes out normalised and
        # the factored form would only add the row-sum fill and the grad_out scaling)
        gat["row_sums"] = torch.empty((N, H), device=dev) if E >= (1 << 22) else None
        gws = torch.empty(max(pg.pyg_gat_backward_workspace_size(plan, planT, H, C, gat["row_sums"] is not None), 1),
                          dtype=torch.uint8, device=dev)
        # the forward gathers z rows: when z exceeds L2 (Reddit 8 x 72: 537 MB) it runs on a source-blocked
        # plan, one L2-resident pass per block; alpha (by edge id) and row_sums carry over to the backward,
        # which runs on the unblocked plan and its transpose
        cb_f = pg.pyg_plan_suggest_col_block(E, N, N, F * 4) if a.col_block == "auto" else 0
        plan_f = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=cb_f) if cb_f > 0 and gat_fwd_blocked_ok(C, F) else plan
        gat["fwd_col_blocks"] = plan_f.view()["n_col_blocks"]
        gat["T_col_blocks"] = planT.view()["n_col_blocks"]
        gfw = torch.empty(max(pg.pyg_gat_propagate_workspace_size(plan_f, H, C), 1), dtype=torch.uint8, device=dev)
        passes, red = 2, "gat"

        def compute():
            o, al = pg.pyg_gat_propagate(zc, s_src, s_dst, H, plan_f, out=gat["out"], alpha=gat["alpha"], workspace=gfw,
                                         row_sums=gat["row_sums"])
            gat["grads"] = pg.pyg_gat_backward(zc, s_src, s_dst, H, al, gout, plan, planT, out=o, workspace=gws,
                                               row_sums=gat["row_sums"])

    gatl = None
    if a.op == "gatlayer":
        # a whole GAT layer forward in this library: z = x W^T with the per-head attention
        # projections fused into the tcgen05 epilogue (pyg_gat_transform), then the segment softmax and
        # the alpha-weighted aggregation (pyg_gat_propagate); 8 heads x 8 (citation graphs) or x F/8
        assert world == 1 and a.strategy == "segment", "--op gatlayer: one GPU, segment strategy"
        H = a.heads or 8
        C = a.gat_c or (8 if a.config in ("cora", "pubmed", "clouds") else max(1, min(F, 256) // H))
        # the gathered matrix is z [N x H*C]: source blocks sized for ITS rows (an L2-resident pass per
        # block when z exceeds L2, e.g. Reddit 232,965 x 256 floats = 238 MB)
        # (sized for twice the z row: blocks of ~0.2 x L2 -- the per-edge alpha stores and s_src reads
        # share L2 with the block; Reddit 8 x 32: 8 passes 11.3-11.6 ms against 5 passes 12.1-12.3 ms,
        # gpurun_out/r3s)
        cb_z = pg.pyg_plan_suggest_col_block(E, N, N, 2 * H * C * 4) if a.col_block == "auto" else int(a.col_block)
        if plan_full.view()["col_block"] != cb_z:
            plan = plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=cb_z)
            col_block = cb_z
        gg = torch.Generator(device=dev)
        gg.manual_seed(109)
        Wg = torch.zeros((H * C, ld), device=dev)
        Wg[:, :F] = torch.randn((H * C, F), generator=gg, device=dev) / (F ** 0.5)
        a_s = torch.randn(H * C, generator=gg, device=dev)
        a_d = torch.randn(H * C, generator=gg, device=dev)
        go = torch.empty((N, H * C), device=dev)
        gal = torch.empty((E, H), device=dev)
        gatl = dict(H=H, C=C, out=go)
        glw = torch.empty(max(pg.pyg_gat_propagate_workspace_size(plan, H, C), 1), dtype=torch.uint8, device=dev)
        # attention in factored form (alpha = p / row_sums[dst]) on the large graphs (see --op gat)
        grs = torch.empty((N, H), device=dev) if E >= (1 << 22) else None
        passes, red = 1, "gatlayer"

        def compute():
            z, ss, sd = pg.pyg_gat_transform(x_full, Wg[:, :F], a_s, a_d, H)
            pg.pyg_gat_propagate(z, ss, sd, H, plan, out=go, alpha=gal, workspace=glw, row_sums=grs)

    appnp = None
    if a.op == "appnp":
        # NEXT-2: APPNP propagation z_{k+1} = (1 - alpha) S z_k + alpha h, S = D^-1/2 (A+I) D^-1/2,
        # K steps on one plan, the teleport term fused into the segment-reduce epilogue.  h = the config's X.
        assert world == 1 and a.strategy == "segment", "--op appnp: one GPU, segment strategy"
        t1 = time.perf_counter()
        if a.config != "pubmed":
            ei, wgt = pg.pyg_gcn_norm(ei, N)
            E = ei.shape[1]
            cb = pg.pyg_plan_suggest_col_block(E, N, N, ld * 4) if a.col_block == "auto" else int(a.col_block)
            plan = plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=cb)
            col_block = cb
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - t1) * 1e3
        zbuf = torch.empty((N, ld), dtype=torch.float32, device=dev)[:, :F]
        obuf = torch.empty((N, ld), dtype=torch.float32, device=dev)[:, :F]
        # + E floats: the weights gathered into plan order once per call (streamed by every step)
        ws_a = torch.empty(max(1, pg.pyg_workspace_size(plan, N, F, "sum") + E * 4 + 256), dtype=torch.uint8, device=dev)
        appnp = dict(out=obuf)
        passes, weighted, red = a.K, True, "sum"

        def compute():
            pg.pyg_appnp(x_full, plan, K=a.K, alpha=a.alpha, edge_weight=wgt, out=obuf, scratch=zbuf, workspace=ws_a)

    gcn = None
    if a.op == "gcn":
        # NEXT-2: one GCN layer D^-1/2 (A+I) D^-1/2 X W^T + b: the transform on the tcgen05
        # tensor cores (TF32, D^-1/2 row scale fused), then the unweighted aggregation over A+I at the
        # hidden width with the D^-1/2 row scale and the bias fused into its epilogue.
        assert world == 1 and a.strategy == "segment", "--op gcn: one GPU, segment strategy"
        t1 = time.perf_counter()
        if a.config != "pubmed":
            ei, _ = pg.pyg_gcn_norm(ei, N)
            E = ei.shape[1]
        # the aggregation gathers the transformed rows (hidden wide): block the plan for THAT row size
        ldh = (a.hidden + 7) // 8 * 8
        col_block = (pg.pyg_plan_suggest_col_block(E, N, N, ldh * 4) if a.col_block == "auto"
                     else int(a.col_block))
        plan = plan_full = pg.pyg_plan_build(ei[1], ei[0], N, N, col_block=col_block)
        torch.cuda.synchronize()
        prep_ms = (time.perf_counter() - t1) * 1e3
        gg = torch.Generator(device=dev)
        gg.manual_seed(108)
        Wt = torch.randn((a.hidden, ld), generator=gg, device=dev) / (F ** 0.5)
        bias = torch.randn(a.hidden, generator=gg, device=dev)
        gout = torch.empty((N, a.hidden), dtype=torch.float32, device=dev)
        nbw = pg.lib.pyg_gcn_layer_workspace_size  # size query through the binding
        ws_g = None
        gcn = dict(out=gout, W=Wt[:, :F], b=bias)
        passes, red = 1, "sum"
        pg.pyg_gcn_layer(x_full, gcn["W"], plan, bias=bias, out=gout)  # allocates the workspace once

        import ctypes as _ct
        _nb = _ct.c_size_t()
        pg._abi.check(nbw(plan.handle, N, a.hidden, _ct.byref(_nb)), "pyg_gcn_layer_workspace_size")
        ws_g = torch.empty(max(1, _nb.value), dtype=torch.uint8, device=dev)

        def compute():
            pg.pyg_gcn_layer(x_full, gcn["W"], plan, bias=gcn["b"], out=gcn["out"], workspace=ws_g)

    def exchange_step():
        if exchange == "push":  # one kernel stores the requested rows into the peers' X_loc (dist.py)
            cur["plan"] = hpush.exchange()
        elif exchange == "halo":  # pack the requested rows + one NCCL all-to-all (dist.py)
            halo_exchange(shard, halo["send_rows"], halo["sc"], halo["rc"], xbuf[per:],
                          pack=lambda xs, rows, o: pg.pyg_gather_rows(xs, rows, out=o), send_buf=halo["sendbuf"])
        elif exchange == "allgather":
            gather_x(shard, world, out=xbuf)  # NCCL all-gather of the X shards (dist.py)

    def step():
        exchange_step()
        compute()

    # numeric pre-check against the oracle before timing: sampled rows, rank 0 / N=1 below
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()

    # CUDA graph of the step (single GPU): the small configs (Cora, PubMed, point clouds) take tens of
    # microseconds per call, so host launch overhead would otherwise dominate the device timeline
    # (all K timed steps are captured into ONE graph and replayed once, so the device runs them back
    # to back; per-step time = total / K)
    use_graph = ((a.graph == "on" or (a.graph == "auto" and a.config in ("cora", "pubmed", "clouds"))) and world == 1
                 and not use_capi)
    launches_per_replay = 0
    if use_graph:
        l0 = pg.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(a.steps):
                compute()
        torch.cuda.synchronize()
        launches_per_replay = pg.launch_count() - l0
        graph.replay()  # untimed: uploads the graph
        torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clocks = Clocks(gpu)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    launches0 = pg.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    if use_graph:
        graph.replay()
    else:
        for i in range(a.steps):
            ev[i][0].record(stream)
            exchange_step()
            kev[i][0].record(stream)
            compute()
            kev[i][1].record(stream)
            ev[i][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = pg.launch_count() - launches0 + launches_per_replay
    clk = clocks.stop()
    if dist:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    if use_graph:
        kern_ms = step_ms = total_ms / a.steps
    else:
        kern_ms = float(np.mean([s.elapsed_time(e) for s, e in kev]))
        step_ms = float(np.mean([s.elapsed_time(e) for s, e in ev]))
    # per-step distribution (median and min beside the mean); one value under a CUDA graph
    per_step = [s.elapsed_time(e) for s, e in ev] if not use_graph else [total_ms / a.steps]
    if dist:
        tt = torch.tensor([total_ms, kern_ms, step_ms - kern_ms], device=dev if a.dist_backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, kern_ms, xchg_ms = tt.tolist()
    else:
        xchg_ms = 0.0
    ms_step = total_ms / a.steps
    units = passes * E * (a.hidden if a.op == "gcn" else (gatl["H"] * gatl["C"] if gatl else F))  # edges*F, all ranks
    value = units / (ms_step * 1e-3)

    peak, peak_src = measured_peak()
    if gat is not None:
        B = gat_step_bytes(E, N, F, gat["H"])
    elif gcn is not None:  # transform (X once, W, H write) + unweighted aggregation at the hidden width
        Fh = a.hidden
        B = N * F * 4 + Fh * F * 4 + N * Fh * 4 + (E * Fh * 4 + E * 4 + 8 * (N + 1) + N * Fh * 4 + 2 * N * 4)
        result_flops = 2.0 * N * F * Fh
    elif gatl is not None:  # transform (X once, W, z + projections written) + softmax + alpha-weighted sum
        Fz = gatl["H"] * gatl["C"]
        Hh = gatl["H"]
        B = (N * F * 4 + Fz * F * 4 + N * Fz * 4 + 2 * N * Hh * 4) + \
            (E * (8 + 2 * 4 * Hh + 4 * Hh) + N * Hh * 4) + (E * (8 + 4 * Hh + 4 * Fz) + N * Fz * 4 + 8 * (N + 1))
        result_flops = 2.0 * N * F * Fz
    elif appnp is not None:  # K weighted propagations + the teleport read of h per step
        B = a.K * (alg_bytes(E, N, F, "sum", a.strategy, weighted=True) + (N * F * 4 if a.alpha else 0))
    else:
        B = passes * alg_bytes(E_loc if world > 1 else E, n_loc, F, red, a.strategy, weighted=weighted)
    achieved = B / (kern_ms * 1e-3) / 1e9
    lpc = max(1, int(round(launches / a.steps)))  # launches of the propagate call per step
    wk = f"{a.config}-{red}-{a.strategy}-cb{col_block}-n{world}" + ("" if a.op == "propagate" else f"-{a.op}")
    tr = traffic_for(wk)
    # The dominant kernel is the segment-reduce (or COO) kernel family of one propagate call (one
    # launch per source-blocked pass, plus the split-hub chunk/combine launches).  achieved =
    # algorithmic bytes of the call / device time of the call (CUDA events on the call's stream).
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": (tr / lpc) if tr else None, "peak_source": peak_src,
            "alg_bytes_per_launch": B / lpc, "launches_per_call": lpc, "kernel_ms_per_launch": kern_ms / lpc,
            "alg_bytes_per_call": B, "call_ms": kern_ms, "traffic_per_call": tr,
            "note": "achieved = algorithmic bytes (north_star byte model: every gathered x_j row, indices, out) / "
                    "device time of the call",
            "ncu": _profile_lookup("ncu_summary.json", wk)}
    # Which roof binds: when the matrix one pass gathers from fits in L2 (a source block of a blocked plan,
    # or the whole X / transformed H) the x_j rows come from L2, so the physical roof is the L2 -> SM
    # gather bandwidth, measured by scripts/l2peak.cu (profiles/l2_peak.json); the HBM-model number stays
    # as modeled_frac.  The atomic strategy is bound by the DRAM read-modify-write of `out` (HBM) unless
    # its column tiles fit L2 (below).
    l2pk, l2src = l2_gather_peak()
    l2_size = torch.cuda.get_device_properties(dev).L2_cache_size
    Fg = a.hidden if gcn is not None else (gatl["H"] * gatl["C"] if gatl else F)
    x_pass = (col_block if col_block else N) * (Fg if (gcn is not None or gatl) else ld) * 4
    if (l2pk and a.strategy == "segment" and gat is None and x_pass <= l2_size):
        l2_bytes = units * 4 + 4 * passes * (E_loc if world > 1 else E)  # x_j rows + col indices, from L2
        l2_ach = l2_bytes / (kern_ms * 1e-3) / 1e9
        roof = dict(roof, bound="l2", achieved=l2_ach, peak=l2pk, frac=l2_ach / l2pk, peak_source=l2src,
                    l2_bytes_per_call=l2_bytes, gathered_matrix_bytes_per_pass=x_pass, l2_size=l2_size,
                    modeled_achieved=achieved, modeled_peak=peak, modeled_frac=achieved / peak,
                    note="x_j rows (+ col indices) are served from L2 (the gathered matrix of a pass <= L2): "
                         "achieved = those bytes / call time against the measured L2 row-gather peak; "
                         "modeled_* = the north_star HBM byte model against the HBM copy peak")

    # The atomic strategy in L2 column tiles (pyg_atomic_tile_cols > 0): the out slice and the gathered
    # slice of a tile are L2-resident, so each edge costs one row gather + one red.global per tile from /
    # into L2: the roof is the measured gather + RED rate (scripts/l2red.cu)
    if a.strategy == "atomic" and a.op == "propagate" and world == 1:
        tcols = pg.pyg_atomic_tile_cols(N, N, F, red)
        rpk, rsrc = l2_red_peak()
        if tcols > 0 and rpk:
            red_bytes = units * 4  # gathered x_j payload = RED payload (E * F * 4)
            r_ach = red_bytes / (kern_ms * 1e-3) / 1e9
            roof = dict(roof, bound="l2_red", achieved=r_ach, peak=rpk, frac=r_ach / rpk, peak_source=rsrc,
                        l2_red_bytes_per_call=red_bytes, tile_cols=tcols, tiles=-(-F // tcols),
                        modeled_achieved=achieved, modeled_peak=peak, modeled_frac=achieved / peak,
                        note="atomic strategy in L2 column tiles: every x_j row slice is gathered from and every "
                             "message RED-added into L2-resident slices; achieved = E*F*4 / call time against "
                             "the measured gather + RED rate; modeled_* = the north_star HBM byte model")

    result = {
        "metric": "aggregation edges*F/s", "value": value, "unit": "edges*F/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": CONFIGS[a.config]["name"], "N": N, "E": E, "F": F, "ldx": ld, "reduce": red,
                   "strategy": a.strategy, "col_block": col_block,
                   "col_blocks": plan_full.view()["n_col_blocks"] if plan_full is not None else (
                       (-(-N // col_block) if col_block else 1) if dplan is not None else 0),
                   "parallelism": f"dst-range x{world}" if world > 1 else "single",
                   "exchange": exchange,
                   "cuda_graph": bool(use_graph),
                   "halo_rows": halo["n"] if halo else None,
                   "l2": "inputs larger than L2 (no flush)" if a.config in ("reddit", "rmat")
                   else "L2-resident inputs (warm, back-to-back as in Fig. 3's 1000 runs)"},
        "roofline": roof, "gpu_launches": int(launches), "clocks": clk, "plan_build_ms": plan_ms,
        "exchange_ms": xchg_ms, "compute_ms": kern_ms,
        "ms_per_step_median": float(np.median(per_step)), "ms_per_step_min": float(np.min(per_step)),
        "ms_per_step_max": float(np.max(per_step)),
        "gen_s": gen_s,
    }
    if w.get("extra"):
        result.update(w["extra"])
    if gatl is not None:
        result["config"]["op"] = "gatlayer"
        result["config"]["heads"] = gatl["H"]
        result["config"]["channels"] = gatl["C"]
        result["config"]["step"] = ("GAT layer forward: tcgen05 TF32 transform with fused attention projections + "
                                    "segment softmax + alpha-weighted aggregation")
        result["transform_tflops_per_step"] = result_flops / 1e12
        result["units_note"] = "edges*F counts E x heads*channels per step"
    if gcn is not None:
        result["config"]["op"] = "gcn"
        result["config"]["hidden"] = a.hidden
        result["config"]["E_with_self_loops"] = E
        result["config"]["step"] = ("GCN layer: tcgen05 TF32 transform X W^T (D^-1/2 rows fused) + unweighted "
                                    "aggregation over A+I at the hidden width (D^-1/2 and bias fused)")
        result["gcn_norm_and_plans_ms"] = prep_ms
        result["transform_tflops_per_step"] = result_flops / 1e12
        result["units_note"] = "edges*F counts E x hidden (the aggregation width) per step"
    if appnp is not None:
        result["config"]["op"] = "appnp"
        result["config"]["K"] = a.K
        result["config"]["alpha"] = a.alpha
        result["config"]["step"] = "APPNP K-step propagation with GCN weights (K segment-reduce passes, fused teleport)"
        result["config"]["E_with_self_loops"] = E
        result["gcn_norm_and_plans_ms"] = prep_ms
    if gat is not None:
        result["config"]["op"] = "gat"
        result["config"]["heads"] = gat["H"]
        result["config"]["channels"] = F // gat["H"]
        result["config"]["forward_col_blocks"] = gat["fwd_col_blocks"]
        result["config"]["transposed_col_blocks"] = gat["T_col_blocks"]
        result["config"]["step"] = ("GAT aggregation forward (segment softmax + alpha-weighted sum) + backward "
                                    "(grad z, s_src, s_dst)")
        result["plans_ms"] = prep_ms
        result["roofline"]["note"] = ("achieved = algorithmic bytes of the whole step (5 kernels, gat_step_bytes) / step time; "
                                      "with source-blocked forward / transposed plans those passes gather from L2, so "
                                      "the HBM-modeled frac can exceed 1")
    elif passes == 2:
        result["config"]["step"] = "GCN forward (w = D^-1/2 (A+I) D^-1/2) + backward w.r.t. X"
        result["config"]["E_with_self_loops"] = E
        result["gcn_norm_and_plans_ms"] = prep_ms

    # ---- numeric pre-check + cpu_baseline (rank 0, N = 1) ----
    if rank == 0 and world == 1 and not a.no_cpu:
        import oracle

        oracle.build()
        ei_cpu = ei.cpu().numpy()
        x_cpu = np.ascontiguousarray(x.cpu().numpy())
        w_cpu = wgt.cpu().numpy() if weighted else None
        if gatl is not None:
            rate, dt, Es, R, ref = oracle_sample(ei_cpu, x_cpu, N, "sum", a.cpu_seconds, F)
            got = None
        elif gcn is not None:
            rate, dt, Es, R, ref = oracle_gcn_sample(ei_cpu, x_cpu, gcn["W"].cpu().numpy(), gcn["b"].cpu().numpy(), N,
                                                     a.cpu_seconds)
            got = gcn["out"][:R].cpu().numpy()
        elif appnp is not None:
            rate, dt, Es, R, ref = oracle_appnp_run(ei_cpu, x_cpu, w_cpu, a.K, a.alpha, a.cpu_seconds, F)
            got = appnp["out"].cpu().numpy() if R else None
        elif gat is not None:
            rate, dt, Es, R, ref = oracle_gat_sample(ei_cpu, zc.cpu().numpy(), s_src.cpu().numpy(), s_dst.cpu().numpy(),
                                                     gat["H"], N, a.cpu_seconds, F)
            got = gat["out"][:R].cpu().numpy()
        elif passes == 1:
            rate, dt, Es, R, ref = oracle_rows(ei_cpu, x_cpu, cpu_sample_rows(a.config, N), red, F, w=w_cpu)
            got = out[:R].cpu().numpy()
        else:
            rate, dt, Es, R, ref = oracle_sample(ei_cpu, x_cpu, N, red, a.cpu_seconds, F, w=w_cpu)
            got = out[:R].cpu().numpy()
        if gatl is not None:
            ok = None  # parity of the layer's parts: tests/test_gpu_transform.py + tests/test_gpu_attention.py
        elif gcn is not None:
            ok = bool((np.abs(got - ref[0]) <= 2.5e-3 * ref[1] + 1e-5 * ref[2] + 1e-6).all())
        elif appnp is not None:
            ok = bool((np.abs(got - ref) <= 1e-5 * np.abs(ref) + 1e-6).all()) if R else None
        elif gat is not None:
            ok = bool((np.abs(got - ref[0]) <= 1e-5 * ref[2] + 1e-6).all())
        elif red == "max":
            # the oracle ran on the masked edge list: its argmax counts positions in that subset (and uses
            # the subset's size for empty rows) -- map them back to the original edge ids first
            idx = np.flatnonzero(ei_cpu[1] < R)
            ra = np.asarray(ref[1])
            ra = np.where(ra < idx.size, idx[np.minimum(ra, max(idx.size - 1, 0))], E) if idx.size else np.full_like(ra, E)
            ok = np.array_equal(got, ref[0]) and np.array_equal(arg[:R].cpu().numpy(), ra)
        else:
            ok = bool((np.abs(got - ref) <= 1e-5 * np.abs(ref) + 1e-6).all())
        if appnp is not None and R:
            sample = f"the whole graph, K = {a.K} steps ({Es} edge visits), {dt:.1f} s single-threaded C, fp64 state"
        elif appnp is not None:
            sample = (f"one sum propagate pass over the {Es} in-edges of the first target rows ({Es / E:.2%} of E), "
                      f"{dt:.1f} s single-threaded C (the full K-step recurrence would take hours)")
        else:
            sample = (f"{Es} edges of the first {R} target rows ({Es / E:.2%} of E), {dt:.1f} s single-threaded C, "
                      f"fp64 accumulate")
        result["cpu_baseline"] = {"value": rate, "unit": "edges*F/s", "cores": 1, "kind": "oracle",
                                  "sample": sample, "parity_on_sample": ok, "host": host_info(),
                                  "full_pass": full_pass_record(a.config, red) if a.op == "propagate" else None}
        if ok is False:  # None: no element-wise check for this op (see parity_on_sample)
            result["parity_error"] = "GPU output disagrees with the oracle on the sampled rows"

    # ---- e2e at N > 1: every step the edge list and this rank's X rows come from pinned host memory,
    # the global plan is built and sliced, X is all-gathered (NCCL), the rank's rows are propagated and
    # copied back (dist.DistAggregation: the user-facing multi-GPU call); max over ranks ----
    if e2e_host is not None:
        from paper_1903_02428_b200.dist import DistAggregation

        dei = torch.empty(e2e_host["hei"].shape, dtype=torch.int64, device=dev)
        dxs = torch.empty(e2e_host["hx"].shape, dtype=torch.float32, device=dev)
        cb_e = pg.pyg_plan_suggest_col_block(E, N, N, ld * 4) if a.col_block == "auto" else int(a.col_block)
        hout_e = torch.empty((e2e_host["hi"] - e2e_host["lo"], F), dtype=torch.float32, pin_memory=True)

        def e2e_dist_step():
            dei.copy_(e2e_host["hei"], non_blocking=True)
            dxs.copy_(e2e_host["hx"], non_blocking=True)
            da = DistAggregation(dei, N, world, rank, col_block=cb_e, F=F, ld=ld,
                                 comm=comm if dplan is not None else None,
                                 exchange=a.exchange if dplan is not None else "allgather")
            shard_e = torch.zeros((da.per, ld), dtype=torch.float32, device=dev)
            shard_e[: da.hi - da.lo] = dxs
            r = da.forward(shard_e[:, :F], reduce=red)
            o = r[0] if isinstance(r, tuple) else r
            hout_e.copy_(o, non_blocking=True)

        e2e_dist_step()
        torch.cuda.synchronize()
        dist.barrier()
        k2 = max(2, min(a.steps, 3))
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(k2):
            e2e_dist_step()
        s1.record()
        torch.cuda.synchronize()
        tt = torch.tensor([s0.elapsed_time(s1) / k2], device=dev if a.dist_backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_ms = float(tt.item())
        result["e2e"] = {"value": units / (e_ms * 1e-3), "unit": "edges*F/s",
                         "h2d_bytes_per_step": int(e2e_host["hx"].numel() * 4 + e2e_host["hei"].numel() * 8),
                         "d2h_bytes_per_step": int(hout_e.numel() * 4), "ms_per_step": e_ms, "steps": k2,
                         "includes": "per rank: H2D(edge list, own X rows) + the dist plan build (global plan, "
                                     "slice, halo / transposed local plan) + NCCL exchange of X + propagate + "
                                     "D2H(own out rows); max over ranks"}

    # ---- e2e through the C ABI with host buffers (N = 1) ----
    if world == 1 and not a.no_e2e and passes == 1 and gat is None and appnp is None and gcn is None and gatl is None:
        xs = x.as_strided((N, ld), (x.stride(0), 1)) if x.stride(0) == ld else x.contiguous()
        hx = torch.empty(xs.shape, dtype=torch.float32, pin_memory=True)
        hx.copy_(xs)
        hei = torch.empty(ei.shape, dtype=torch.int64, pin_memory=True)
        hei.copy_(ei)
        hout = torch.empty(out.shape, dtype=torch.float32, pin_memory=True)
        # double-buffered device inputs: step k+1's H2D (copy stream) runs while step k builds its plan and
        # propagates, so in steady state a step costs its host-link time (the link is the bound: 2.4 GB in)
        dxs = [torch.empty_like(xs, device=dev) for _ in range(2)]
        deis = [torch.empty_like(ei) for _ in range(2)]
        done = [None, None]
        k2 = max(2, min(a.steps, 5))

        cp = torch.cuda.Stream()
        d2h = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        it = [0]

        def e2e_step():
            b = it[0] & 1
            it[0] += 1
            with torch.cuda.stream(cp):
                if done[b] is not None:  # the propagate that last read buffer b (two steps back)
                    cp.wait_event(done[b])
                deis[b].copy_(hei, non_blocking=True)
                ev_e = torch.cuda.Event()
                ev_e.record(cp)
                # X after the edge list: both share the host link, the plan build needs only the edges
                dxs[b].copy_(hx, non_blocking=True)
                ev_x = torch.cuda.Event()
                ev_x.record(cp)
            main.wait_event(ev_e)
            p = pg.pyg_plan_build(deis[b][1], deis[b][0], N, N, col_block=col_block) if a.strategy == "segment" else None
            main.wait_event(ev_x)
            r = pg.pyg_propagate(dxs[b][:, :F], deis[b] if p is None else None, n_dst=N, reduce=red, plan=p, E=E)
            done[b] = torch.cuda.Event()
            done[b].record(main)
            o = r[0] if isinstance(r, tuple) else r
            # the result goes back on its own stream: this step's D2H overlaps the next step's H2D (the
            # host link is full duplex); the next D2H into hout queues behind it on the same stream
            d2h.wait_stream(main)
            with torch.cuda.stream(d2h):
                hout.copy_(o, non_blocking=True)
            o.record_stream(d2h)

        e2e_step()
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        cp.wait_stream(main)  # no copy of the timed steps starts before s0
        for _ in range(k2):
            e2e_step()
        main.wait_stream(d2h)  # the last result is on the host before the clock stops
        s1.record()
        torch.cuda.synchronize()
        e_ms = s0.elapsed_time(s1) / k2
        result["e2e"] = {"value": units / (e_ms * 1e-3), "unit": "edges*F/s",
                         "h2d_bytes_per_step": int(hx.numel() * 4 + hei.numel() * 8),
                         "d2h_bytes_per_step": int(hout.numel() * 4), "ms_per_step": e_ms, "steps": k2,
                         "includes": "H2D(X, edge_index) + plan build + propagate + D2H(out), every step; "
                                     "double-buffered inputs: step k+1's H2D (copy stream) overlaps step "
                                     "k's plan build and propagate, its D2H (third stream) the next H2D"}
        # the pipelined path computes what the device-timed path computed (bitwise on the deterministic
        # segment path; the atomic sum order varies between runs)
        dev_out = out.detach().cpu()
        result["e2e"]["matches_device_output"] = bool(
            torch.equal(hout, dev_out) if a.strategy == "segment" else torch.allclose(hout, dev_out, rtol=1e-5, atol=1e-6))

    # ---- L2-resident configs: cold-cache device time (an untimed write of 2 x L2 before
    # each call), beside the warm back-to-back number above ----
    if world == 1 and a.config in ("cora", "pubmed", "clouds"):
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        scratch = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)
        cold = []
        for _ in range(12):
            scratch.fill_(1.0)
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            compute()
            c1.record()
            torch.cuda.synchronize()
            cold.append(c0.elapsed_time(c1))
        result["cold_ms_per_step"] = float(np.median(cold[2:]))
        result["cold_note"] = "median device time of one step after flushing L2 (2 x L2 scratch write), eager launch"
        del scratch
        if a.config == "clouds" and a.op == "propagate":
            # EdgeConv / PointNet-style message [x_i || x_j] (phi = concat, F_out = 128), max + arg
            o2 = torch.empty((N, 2 * F), dtype=torch.float32, device=dev)
            a2 = torch.empty((N, 2 * F), dtype=torch.int64, device=dev)

            def cat_call():
                pg.pyg_propagate(x, None if plan else ei, reduce="max", concat_xi=True, plan=plan, out=o2, arg_out=a2, E=E)

            for _ in range(3):
                cat_call()
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            for _ in range(20):
                cat_call()
            c1.record()
            torch.cuda.synchronize()
            result["concat_xi_max_ms"] = c0.elapsed_time(c1) / 20
            result["concat_xi_note"] = "phi = [x_i || x_j], F_out = 128, max + arg (eager, back to back)"

    # ---- other reductions on the same resident graph (informational) ----
    if world == 1 and not a.no_variants and passes == 1 and gat is None and appnp is None and gcn is None \
            and gatl is None:
        var = {}
        for r2 in ("sum", "mean", "max"):
            if r2 == red:
                continue
            a2 = torch.empty((N, out.stride(0)), dtype=torch.int64, device=dev)[:, :F] if r2 == "max" else None
            ws2 = torch.empty(max(1, pg.pyg_workspace_size(plan, N, F, r2, E=E)), dtype=torch.uint8, device=dev)
            for _ in range(3):
                pg.pyg_propagate(x, None if plan else ei, reduce=r2, plan=plan, out=out, arg_out=a2, E=E,
                                 workspace=ws2)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(5):
                pg.pyg_propagate(x, None if plan else ei, reduce=r2, plan=plan, out=out, arg_out=a2, E=E,
                                 workspace=ws2)
            s1.record()
            torch.cuda.synchronize()
            ms = s0.elapsed_time(s1) / 5
            b2 = alg_bytes(E, N, F, r2, a.strategy)
            var[r2] = {"ms": ms, "edges*F/s": units / (ms * 1e-3), "GB/s": b2 / (ms * 1e-3) / 1e9,
                       "frac": b2 / (ms * 1e-3) / 1e9 / peak}
        result["variants"] = var

    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
