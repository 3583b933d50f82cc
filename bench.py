#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 far-field path (arXiv 1409.2802, kernid).

Metric (BASELINE.json): kernel entries/s (targets x sources) of the FP64 fused
eval + reconstruction-error pass, and its fraction of the FP64 roofline.

Workload (N=1): BASELINE.json configs[1] at its largest dimension -- d=3, 1e6 N(0,I_3)
points (seed 1, trial 0), RandomPoint center, m=100 nearest sources, D_WS=2, Silverman h,
EuclideanNorm sampling of 2% of the rows, ID to eps=1e-2 (r=17) -> one fused pass over all
N_T ~ 1e6 targets x 100 sources = ~1e8 entries. Synthetic data (no dataset exists).

  value   device-resident pass (kid_recon_error_dev on the timed stream), CUDA events,
          L2 flushed (256 MB write) between timed steps, max over ranks;
  e2e     the same metric through the C-ABI with HOST buffers every step: points H2D
          from pinned memory, kid_split, target indices D2H, kid_recon_error (skeleton /
          P H2D, Grams D2H);
  roofline  the dominant kernel (k_gram in residual mode) timed by the library's own
          CUDA events on the launching stream (kid_profile), algorithmic FP64 flops per
          entry / its average duration vs the measured FP64 peak;
  cpu_baseline  the oracle restatement of the reference pipeline (threaded K assembly,
          exact QR+SVD norms) on a bounded slice of the same targets, rank 0, N=1.

Multi-GPU (torchrun): weak scaling, each rank holds its own 1e6-point shard; the split
exchanges the local top-m candidates (all_gather) and the pass all-reduces its Grams.
`--impl reference` times the reference's CPU path (oracle port; the reference itself
cannot be built here: no Eigen) on the same config / metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "kernel entries/s (targets x sources, FP64 fused eval+error)"
UNIT = "entries/s"
F_EXP = 32  # flops charged per exp (SURVEY.md 8d convention: CUDA 12.9 exp(double) = 14 DFMA + 2 DADD + 2 DMUL)

WORKLOADS = {
    # configs[1] (quoted config of the metric): d in {1,2,3}, 1e6 targets, m=100, D_WS=2
    "c2-d3": dict(d=3, N=1_000_000, m=100, xi=2.0, h_value=1.0, s=0.02, eps=1e-2),
    "c2-d2": dict(d=2, N=1_000_000, m=100, xi=2.0, h_value=1.0, s=0.02, eps=1e-8),
    "c2-d3-e4": dict(d=3, N=1_000_000, m=100, xi=2.0, h_value=1.0, s=0.02, eps=1e-4),
    "c2-d3-e6": dict(d=3, N=1_000_000, m=100, xi=2.0, h_value=1.0, s=0.02, eps=1e-6),
    "c2-d3-e8": dict(d=3, N=1_000_000, m=100, xi=2.0, h_value=1.0, s=0.02, eps=1e-8),
    "c1": dict(d=2, N=100_000, m=100, xi=2.0, h_value=1.0, s=0.02, eps=1e-8),
    "c3-d5": dict(d=5, N=1_000_000, m=100, xi=3.0, h_value=1.0, s=0.02, eps=1e-8),
    "c4-d16": dict(d=16, N=12_000_000, m=256, xi=2.0, h_value=1.0, s=0.002, eps=1e-2),
    "c5-d8-shard": dict(d=8, N=12_515_000, m=512, xi=2.0, h_value=1.0, s=0.002, eps=1e-2),
    # configs[4] at N=1 GPU: the largest single-GPU configuration (1.0012e8 points, 6.4 GB)
    "c5": dict(d=8, N=100_120_000, m=512, xi=2.0, h_value=1.0, s=4e-5, eps=1e-2),
}


def flops_per_entry(d: int, m: int, r: int) -> float:
    """SURVEY.md 8(d) per-entry flop figure of the fused pass (K5 mode S, spectral error with the
    D^T D Gram): eval 3d + 1 + F_EXP, skel.P 2r, SYRK m + 1 -> 3d + 2r + m + 34. This is the
    figure the roofline contract prescribes (`roofline.achieved`)."""
    return 3 * d + 2 * r + m + 34


def flops_per_entry_strict(d: int, m: int, r: int) -> float:
    """Stricter count of the work the kernel actually needs: eval 3d + 1 + F_EXP,
    sum K^2 (2), skel.P and the SYRK only over the m - r non-skeleton columns (the skeleton
    columns of D are exactly zero): 2 r (m - r) / m + (m - r)(m - r + 1) / m."""
    me = m - r
    return 3 * d + 1 + F_EXP + 2 + 2.0 * r * me / m + me * (me + 1) / m


def load_peaks():
    p = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {"fp64_tflops": 37.0, "source": "fallback: tools/fp64_peaks.cu DMMA m8n8k4 loop, round-1 measurement"}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [ln.split(",") for ln in self.f.read().strip().splitlines() if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                clk, cmax = float(r[0]), float(r[1])
            except (ValueError, IndexError):
                continue
            mx = max(mx, cmax)
            if clk > 0.5 * cmax:  # under load
                sm.append(clk)
                for n, v in zip(names, r[4:8]):
                    if v.strip().lower().startswith("active"):
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- dist helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------- workload setup (product path)
class Problem:
    """One rank's shard: points, the split, and the skeleton / P from the product host path."""

    def __init__(self, wl, dev, torch, ws, rank, seed=1):
        from paper_1409_2802_b200 import kernid as H
        self.wl, self.dev, self.torch, self.ws, self.rank = wl, dev, torch, ws, rank
        d, N, m, xi = wl["d"], wl["N"], wl["m"], wl["xi"]
        data_seed = H.derive_seed(seed, 0, 0)  # trial 0, scheme 0 (harness.hpp:160-161)
        pseed = H.derive_seed(data_seed, 0xDA7A) if rank == 0 else H.derive_seed(data_seed, 0xDA7A, rank)
        self.points = H.gen_normal(d, N, pseed)  # (N, d), rank 0 == the reference trial's data
        self.pts_cm = np.ascontiguousarray(self.points.T).ravel()
        self.offset = rank * N
        dev.set_points(self.points, self.offset)
        from paper_1409_2802_b200 import _lib
        # RandomPoint center (harness.hpp:95-100) from rank 0's shard
        ci = H.center_index(N, data_seed)
        center = self.points[ci].copy()
        self.center = self._bcast(center)
        self.h = wl["h_value"] * self._silverman(d, N * ws)
        self.data_seed = data_seed
        self.H, self._lib = H, _lib

    @staticmethod
    def _silverman(d, N):
        e = 1.0 / (d + 4.0)
        return (4.0 / (2.0 * d + 1.0)) ** e * float(N) ** (-e)

    def _bcast(self, arr):
        if self.ws == 1:
            return arr
        t = self.torch.tensor(arr, dtype=self.torch.float64, device="cuda")
        self.torch.distributed.broadcast(t, 0)
        return t.cpu().numpy()

    def split(self):
        """kid_split (N=1) or the sharded split: local top-m -> all_gather -> global top-m."""
        dev, m, xi = self.dev, self.wl["m"], self.wl["xi"]
        if self.ws == 1:
            src, rho, nt = dev.split(self.center, m, xi)
            self.src, self.rho, self.nt = src, rho, nt
            return
        from paper_1409_2802_b200 import dist as D
        src, rho, src_pts, nt = D.sharded_split(dev, self.points, self.offset, self.center, m, xi, device="cuda")
        self.src, self.rho, self.nt, self._src_pts = src, rho, nt, src_pts

    def skeleton(self):
        """EuclideanNorm sampling + host ID on rank 0 (product host path), broadcast."""
        H, dev, wl = self.H, self.dev, self.wl
        m = wl["m"]
        if self.rank == 0:
            w = dev.row_norms(self.h)
            tgt_local = dev.targets() - self.offset
            sample = H.draw(H.EUCLIDEAN_NORM, w.size, wl["s"], H.derive_seed(self.data_seed, 0, 1), w)
            src_local = self.src - self.offset if self.ws == 1 else None
            if self.ws == 1:
                Ks = H.kernel_rows(self.pts_cm, self.points.shape[0], wl["d"], tgt_local, sample, src_local, self.h)
            else:
                Ks = self._rows_global(tgt_local, sample)
            sv = H.singular_values(Ks)
            r = H.epsilon_rank(sv, wl["eps"])
            skel, P = H.interpolative_decomposition(Ks, r)
            self.sample_rows = sample.size
        else:
            r = 0
        if self.ws > 1:
            t = self.torch.tensor([r], dtype=self.torch.int64, device="cuda")
            self.torch.distributed.broadcast(t, 0)
            r = int(t.item())
            if self.rank != 0:
                skel, P = np.zeros(r, np.int64), np.zeros((r, m))
            ts = self.torch.tensor(skel, dtype=self.torch.int64, device="cuda")
            tp = self.torch.tensor(P, dtype=self.torch.float64, device="cuda")
            self.torch.distributed.broadcast(ts, 0)
            self.torch.distributed.broadcast(tp, 0)
            skel, P = ts.cpu().numpy(), tp.cpu().numpy()
        self.skel, self.P, self.r = skel, P, r

    def _rows_global(self, tgt_local, sample):
        # sources may live on other ranks: evaluate with the gathered source coordinates
        from paper_1409_2802_b200 import kernid as H
        d = self.wl["d"]
        src_pts = self._src_points_global()
        pts = np.concatenate([self.points, src_pts])
        pts_cm = np.ascontiguousarray(pts.T).ravel()
        src_idx = np.arange(self.points.shape[0], pts.shape[0], dtype=np.int64)
        return H.kernel_rows(pts_cm, pts.shape[0], d, tgt_local, sample, src_idx, self.h)

    def _src_points_global(self):
        return self._src_pts  # gathered with the split's candidates (dist.sharded_split)

    def entries(self):
        return self.nt * self.wl["m"]


def setup(wl, ws, rank, local, torch):
    from paper_1409_2802_b200._lib import Device
    dev = Device(local)
    prob = Problem(wl, dev, torch, ws, rank)
    prob.split()
    prob.skeleton()
    dev.recon_prepare(prob.skel, prob.P)
    return dev, prob


# ----------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = WORKLOADS[args.config]
    # a dedicated (non-default) stream: the library launches on it, the CUDA events time it
    torch.cuda.set_stream(torch.cuda.Stream())
    dev, prob = setup(wl, ws, rank, local, torch)
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    m, r = wl["m"], prob.r
    meff = m - r
    out = torch.empty(2 + max(meff, 1) ** 2, dtype=torch.float64, device="cuda")
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 256 MB > 126 MB L2

    def step():
        dev.recon_error_dev(prob.h, out.data_ptr())
        if ws > 1:
            torch.distributed.all_reduce(out)

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(local)
    dev.profile(True)
    l0 = dev.launches
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches = dev.launches - l0
    kern_ms = dev.profile_read()
    dev.profile(False)
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    ent = torch.tensor([float(prob.entries())], dtype=torch.float64, device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(ent)
    ms_max = float(t.item())
    total_entries = float(ent.item())
    value = total_entries * args.steps / (ms_max / 1e3)

    # roofline of the dominant kernel (k_gram, residual mode)
    peaks = load_peaks()
    kavg = float(np.mean(kern_ms)) if len(kern_ms) else float("nan")
    fpe = flops_per_entry(wl["d"], m, r)
    kernel_name = "k_gram (residual mode)"
    if r >= m:  # full-rank skeleton: D == 0, the pass is ||K||_F^2 alone (k_sumsq): eval + square-sum
        fpe, kernel_name = 3 * wl["d"] + 1 + F_EXP + 2, "k_sumsq (full-rank skeleton: D == 0)"
    achieved = prob.entries() * fpe / (kavg / 1e3) / 1e12
    fpe_strict = flops_per_entry_strict(wl["d"], m, r)
    achieved_strict = prob.entries() * fpe_strict / (kavg / 1e3) / 1e12
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(args.config)

    # e2e through the C-ABI with host buffers
    e2e = run_e2e(args, dev, prob, torch, ws, rank)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic: seeded N(0,I_d) points (harness seed streams), no dataset",
        "config": {"workload": f"BASELINE configs[1] {args.config}: d={wl['d']}, N={wl['N']} points/rank, "
                               f"N_T={prob.nt}/rank, m={m}, D_WS={wl['xi']}, h=silverman({prob.h:.6g}), "
                               f"euclidean_norm s={wl['s']}, eps={wl['eps']}, rank r={r}",
                   "global_targets": int(total_entries // m), "sources": m, "skeleton_rank": r,
                   "parallelism": f"target shards x{ws}, NCCL all_reduce of D^T D" if ws > 1 else "1 GPU",
                   "l2": "flushed (256 MB write) between timed steps"},
        "roofline": {"bound": "tensor", "pipe": "FP64 (DMMA + DFMA)", "achieved": achieved,
                     "peak": peaks["fp64_tflops"], "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"],
                     "traffic": traffic, "kernel": kernel_name, "kernel_ms": kavg,
                     "flops_per_entry": fpe, "flops_convention": "SURVEY.md 8(d) K5 mode S: 3d + 2r + m + 34",
                     "frac_strict": achieved_strict / peaks["fp64_tflops"], "flops_per_entry_strict": fpe_strict,
                     "peak_source": peaks["source"]},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(prob, budget_s=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_split(args):
    """--pass split: pass 1 (split_sources_targets) on the config's points, HBM roofline of its
    kernels (algorithmic bytes 8 d N read + 8 N_T written)."""
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    torch.cuda.set_stream(torch.cuda.Stream())
    wl = WORKLOADS[args.config]
    from paper_1409_2802_b200._lib import Device
    dev = Device(local)
    prob = Problem(wl, dev, torch, 1, 0)
    dev.set_stream(torch.cuda.current_stream().cuda_stream)
    N, d, m = wl["N"], wl["d"], wl["m"]
    for _ in range(args.warmup):
        prob.split()
    torch.cuda.synchronize()
    dev.profile(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record()
        prob.split()
        ev[i][1].record()
    torch.cuda.synchronize()
    kms = dev.profile_read()  # per split: [k_dist_cand, k_compact]
    dev.profile(False)
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    kd = float(np.mean(kms[0::2])) if len(kms) >= 2 else float("nan")
    kc = float(np.mean(kms[1::2])) if len(kms) >= 2 else float("nan")
    peak = 6552.6
    b_alg = 8.0 * d * N + 8.0 * prob.nt
    b_dist = 8.0 * d * N + 8.0 * N  # read points, write dist
    b_comp = 8.0 * N + 8.0 * prob.nt  # read dist, write indices
    line = {"metric": "split_sources_targets points/s (pass 1)", "value": N / (ms / 1e3), "unit": "points/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "dtype": "f64", "config": {"workload": f"{args.config}: N={N}, d={d}, m={m}, N_T={prob.nt}"},
            "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peak,
                         "achieved": b_alg / (ms / 1e3) / 1e9, "frac": b_alg / (ms / 1e3) / 1e9 / peak,
                         "algorithmic_bytes": b_alg,
                         "k_dist_cand": {"ms": kd, "gbs": b_dist / (kd / 1e3) / 1e9},
                         "k_compact": {"ms": kc, "gbs": b_comp / (kc / 1e3) / 1e9}}}
    print(json.dumps(line), flush=True)


def run_apply(args):
    """--pass apply: the skeleton matvec u = K(T, S_skel) (P q) over all targets (compress.hpp:
    309-325) for the config's ID; FP64 roofline with 3d + 33 + 2 flops per
    (target, skeleton point) entry (eval + exp by the 8(d) convention, multiply-add)."""
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    torch.cuda.set_stream(torch.cuda.Stream())
    wl = WORKLOADS[args.config]
    dev, prob = setup(wl, 1, 0, local, torch)
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    d, m, r = wl["d"], wl["m"], prob.r
    q = np.random.default_rng(0).standard_normal(m)
    q_skel = prob.P @ q
    u = torch.empty(max(prob.nt, 1), dtype=torch.float64, device="cuda")
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        dev.apply_skeleton_dev(prob.h, prob.skel, q_skel, u.data_ptr())
    torch.cuda.synchronize()
    dev.profile(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        dev.apply_skeleton_dev(prob.h, prob.skel, q_skel, u.data_ptr())
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    kms = dev.profile_read()
    dev.profile(False)
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    kavg = float(np.mean(kms)) if len(kms) else float("nan")
    entries = float(prob.nt) * r
    fpe = 3 * d + 33 + 2
    peaks = load_peaks()
    ach = entries * fpe / (kavg / 1e3) / 1e12
    line = {"metric": "apply_skeleton entries/s (targets x skeleton points, FP64)", "value": entries / (ms / 1e3),
            "unit": "entries/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "dtype": "f64",
            "config": {"workload": f"{args.config}: N_T={prob.nt}, m={m}, skeleton rank r={r}, d={d}",
                       "l2": "flushed (256 MB write) between timed steps"},
            "roofline": {"bound": "fp64", "unit": "TFLOP/s", "peak": peaks["fp64_tflops"], "achieved": ach,
                         "frac": ach / peaks["fp64_tflops"], "kernel": "k_apply_skel", "kernel_ms": kavg,
                         "flops_per_entry": fpe}}
    print(json.dumps(line), flush=True)


def run_next_pass(args):
    """--pass svd: the compress_svd error pass (kid_proj_gram, compress.hpp:243-262, SURVEY.md 8f
    item 1) with C = V_perp of the config's sample (rank r by its eps): per (target, source) entry
    eval 3d + 33, ||K||^2 2, D = K V_perp 2n, D^T D n(n+1)/m (n = m - r).
    --pass tsqr: the TSQR factor of the full K (kid_tsqr_r): eval 3d + 33 and
    the Householder fold ~2m per entry.
    --pass rownorms: the EuclideanNorm weights ||K_i|| (kid_row_norms, sampling.hpp:189-196, K2):
    3d + 35 per entry.
    --pass gram: K^T K of the full block (kid_gram, the right factor / leverage Gram, K3):
    3d + 33 + (m + 1) per entry.
    --pass leverage: l_i = ||K_i W||^2 (kid_leverage, lowrank.hpp:304-305, K4) with an m x r
    orthonormal W, r = the config's ID rank: 3d + 33 + 2r per entry."""
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    torch.cuda.set_stream(torch.cuda.Stream())
    wl = WORKLOADS[args.config]
    dev, prob = setup(wl, 1, 0, local, torch)
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)
    d, m = wl["d"], wl["m"]
    H = prob.H
    if args.pass_ == "svd":
        w = dev.row_norms(prob.h)
        sample = H.draw(H.EUCLIDEAN_NORM, w.size, wl["s"], H.derive_seed(prob.data_seed, 0, 1), w)
        Ks = H.kernel_rows(prob.pts_cm, prob.points.shape[0], d, dev.targets() - prob.offset, sample,
                           prob.src - prob.offset, prob.h)
        _, sv, Vt = np.linalg.svd(Ks, full_matrices=True)
        r = H.epsilon_rank(sv, wl["eps"])
        n = m - r
        out = torch.empty(2 + n * n, dtype=torch.float64, device="cuda")
        if args.svd_proj:  # the generic projected Gram over V_perp
            Vp = Vt.T[:, r:]
            Cm = torch.tensor(np.ascontiguousarray(Vp.T).ravel(), dtype=torch.float64, device="cuda")
            fn = lambda: dev.proj_gram_dev(prob.h, Cm.data_ptr(), n, out.data_ptr())
            fpe = 3 * d + 33 + 2 + 2 * n + n * (n + 1) / m
            kern = "k_proj_gram"
        else:  # the product route (kernid_b200::compress_svd): the fused residual pass on the ID of V_r^T
            a, Pa = H.interpolative_decomposition(np.ascontiguousarray(Vt[:r]), r)
            dev.recon_prepare(a, Pa)
            fn = lambda: dev.recon_error_dev(prob.h, out.data_ptr())
            fpe = flops_per_entry_strict(d, m, r)
            kern = "k_gram (residual mode on the ID of V_r^T)"
        metric = "compress_svd error-pass entries/s (targets x sources, FP64)"
        extra = {"rank": r, "n_perp": n}
    elif args.pass_ == "gram":
        G = torch.empty(2 + m * m, dtype=torch.float64, device="cuda")
        fn = lambda: dev.gram_dev(prob.h, G.data_ptr())
        fpe = 3 * d + 33 + (m + 1)
        kern, metric = "k_gram (mode K) / large-m batched Gram", "Gram K^T K entries/s (targets x sources, FP64)"
        extra = {}
    elif args.pass_ == "leverage":
        rl = max(1, prob.r)
        Wm = np.linalg.qr(np.random.default_rng(0).standard_normal((m, rl)))[0]
        Wd = torch.tensor(np.ascontiguousarray(Wm.T).ravel(), dtype=torch.float64, device="cuda")  # m x r col-major
        lv = torch.empty(max(prob.nt, 1), dtype=torch.float64, device="cuda")
        fn = lambda: dev.leverage_dev(prob.h, Wd.data_ptr(), rl, lv.data_ptr())
        fpe = 3 * d + 33 + 2 * rl
        kern, metric = "k_proj_gram (leverage mode) / batched", "leverage-score entries/s (targets x sources, FP64)"
        extra = {"rank": rl}
    elif args.pass_ == "rownorms":
        wv = torch.empty(max(prob.nt, 1), dtype=torch.float64, device="cuda")
        fn = lambda: dev.row_norms_dev(prob.h, wv.data_ptr())
        fpe = 3 * d + 35
        kern, metric = "k_row_norms", "EuclideanNorm row-norm entries/s (targets x sources, FP64)"
        extra = {}
    else:
        R = torch.empty(m * m, dtype=torch.float64, device="cuda")
        fn = lambda: dev.tsqr_r_dev(prob.h, R.data_ptr())
        fpe = 3 * d + 33 + 2 * m
        kern, metric = "k_tsqr", "TSQR entries/s (targets x sources, FP64)"
        extra = {}
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    dev.profile(True)
    l0 = dev.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        fn()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    launches = dev.launches - l0
    kms = dev.profile_read()
    dev.profile(False)
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    kavg = float(np.mean(kms)) if len(kms) else float("nan")
    entries = float(prob.nt) * m
    peaks = load_peaks()
    ach = entries * fpe / (kavg / 1e3) / 1e12
    line = {"metric": metric, "value": entries / (ms / 1e3), "unit": "entries/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "dtype": "f64",
            "gpu_launches": launches,
            "config": dict({"workload": f"{args.config}: N_T={prob.nt}, m={m}, d={d}",
                            "l2": "flushed (256 MB write) between timed steps"}, **extra),
            "roofline": {"bound": "fp64", "unit": "TFLOP/s", "peak": peaks["fp64_tflops"], "achieved": ach,
                         "frac": ach / peaks["fp64_tflops"], "kernel": kern, "kernel_ms": kavg,
                         "flops_per_entry": fpe}}
    print(json.dumps(line), flush=True)


def run_e2e(args, dev, prob, torch, ws, rank):
    """Same metric through the C-ABI with host buffers (pinned points H2D every step)."""
    wl = prob.wl
    N, d, m = wl["N"], wl["d"], wl["m"]
    host = torch.from_numpy(prob.pts_cm).pin_memory()
    stream = torch.cuda.current_stream()
    steps = max(3, min(args.steps, 20))
    times = []
    for i in range(steps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ws > 1:
            torch.distributed.barrier()
        e0.record(stream)
        dev.set_points_colmajor_ptr(host.data_ptr(), N, d, prob.offset)
        prob.split()  # kid_split: the target list stays on the device
        sd, sk, DtD, _ = dev.recon_error(prob.h, prob.skel, prob.P)
        if ws > 1:
            g = torch.tensor(DtD, device="cuda")
            torch.distributed.all_reduce(g)
            DtD = g.cpu().numpy()
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))  # host-side jitter (page-locked copies, syncs) -> median of the steps
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    r = prob.r
    h2d = N * d * 8 + d * 8 + r * 8 + r * m * 8 + m * d * 8
    d2h = m * 8 + 8 + 8 + (2 + m * m) * 8 + m * d * 8
    return {"value": prob.entries() * ws / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "ms_mean": float(np.mean(times)),
            "path": "kid_set_points(pinned) -> kid_split (targets stay on the device) -> kid_recon_error"}


# ----------------------------------------------------------------- CPU baseline (oracle port)
def reference_pipeline_sample(prob, rows: int, threads: int):
    """The reference's compress_id error path (compress.hpp:168-215) on the first `rows`
    targets: dense K assembly (threaded, kernel.hpp:134-172), C P - K and its exact spectral
    norm (QR + SVD, compress.hpp:141-147), ||K||_2 (compress.hpp:156-159)."""
    from oracle import oracle as O
    tg = prob.targets_sample[:rows]
    K = O.kernel_matrix(tg, prob.sources, prob.h, threads=threads)
    num = O.reconstruction_error_norm(K, prob.skel, prob.P)
    den = O.matrix_norm(K)
    return K.shape[0] * K.shape[1], num / den if den > 0 else 0.0


def _prep_cpu(prob):
    tgt = prob.dev.targets() - prob.offset
    prob.targets_sample = np.ascontiguousarray(prob.points[tgt])
    prob.sources = np.ascontiguousarray(prob.points[prob.src - prob.offset])


def cpu_baseline(prob, budget_s=15.0):
    threads = os.cpu_count() or 1
    _prep_cpu(prob)
    rows = 20000
    t0 = time.perf_counter()
    reference_pipeline_sample(prob, rows, threads)
    dt = time.perf_counter() - t0
    rows = int(min(prob.targets_sample.shape[0], max(rows, rows * budget_s / max(dt, 1e-3))))
    t0 = time.perf_counter()
    ent, _ = reference_pipeline_sample(prob, rows, threads)
    dt = time.perf_counter() - t0
    return {"value": ent / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {rows} of {prob.nt} targets x {prob.wl['m']} sources through the oracle's compress_id "
                      f"error path (K assembly on {threads} threads; QR+SVD exact norms single-threaded as the "
                      f"reference's Eigen build), {dt:.1f} s"}


class OracleProblem:
    """The same trial as our arm (harness seed streams), set up on the host by the oracle alone:
    points, RandomPoint center, split, EuclideanNorm sample, host ID -- no device code."""

    def __init__(self, wl, threads, seed=1):
        from oracle import oracle as O
        d, N, m, xi = wl["d"], wl["N"], wl["m"], wl["xi"]
        data_seed = O.derive_seed(seed, 0, 0)
        t = O.prepare_trial(d, N, m, xi, data_seed, h_value=wl["h_value"])
        self.wl, self.h, self.nt = wl, t.h, t.targets.shape[0]
        self.targets_sample, self.sources = t.targets, t.sources
        w = np.concatenate([O.row_norms(O.kernel_matrix(t.targets[i:i + 100_000], t.sources, t.h, threads=threads))
                            for i in range(0, self.nt, 100_000)])
        rows = O.sample_rows(O.SCHEME_EUCLIDEAN, self.nt, wl["s"], O.derive_seed(data_seed, 0, 1), w)
        Ks = O.kernel_matrix(t.targets[rows], t.sources, t.h, threads=threads)
        r = O.epsilon_rank(O.singular_values(Ks), wl["eps"])
        self.skel, self.P = O.interpolative_decomposition(Ks, r)


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path (the oracle port: the
    reference itself needs Eigen, absent here) on this arm's config and trial, rank 0 only, all
    host threads. Setup and timed region are host-only (no device code)."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    wl = WORKLOADS[args.config]
    threads = os.cpu_count() or 1
    prob = OracleProblem(wl, threads)
    rows = args.ref_rows
    for _ in range(args.warmup):
        reference_pipeline_sample(prob, rows, threads)
    times, ent = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        ent, _ = reference_pipeline_sample(prob, rows, threads)
        times.append(time.perf_counter() - t0)
    v = ent / float(np.mean(times))
    sample = (f"{rows} of {prob.nt} targets x {wl['m']} sources per step through the oracle port of compress_id's "
              f"error path (K assembly on {threads} threads, exact QR+SVD norms single-threaded)")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"BASELINE configs[1] {args.config}", "skeleton_rank": int(len(prob.skel))},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2-d3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-rows", type=int, default=50000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--svd-proj", action="store_true", help="--pass svd through kid_proj_gram (C = V_perp) instead of the ID route")
    ap.add_argument("--pass", dest="pass_", default="recon", choices=["recon", "split", "apply", "svd", "tsqr", "rownorms", "gram", "leverage"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.pass_ == "split":
        run_split(args)
    elif args.pass_ in ("svd", "tsqr", "rownorms", "gram", "leverage"):
        run_next_pass(args)
    elif args.pass_ == "apply":
        run_apply(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
