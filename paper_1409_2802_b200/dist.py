"""Multi-GPU host layer: targets sharded across ranks (one process per GPU).

The reference is single-process; here the N points are split into contiguous
index ranges, one per rank, and the only exchanges are

  * split (geometry.hpp:29-65): every rank's n smallest (dist, global idx) candidates plus
    their coordinates -> all_gather -> every rank selects the identical global top-n by
    (dist, idx), rho = its max, then compacts its local targets (kid_split_finish);
  * fused error pass (compress.hpp:141-159): per-rank [sumsq_D, sumsq_K, D^T D] partials ->
    all_reduce (NCCL over NVLink on GPUs, gloo in the CPU tests), or an ordered gather-sum
    when bitwise independence from the rank count is required.

Everything here is plain torch.distributed plumbing; the device work stays in the C-ABI.
"""
from __future__ import annotations

import numpy as np


def pack_candidates(cand_dist, cand_idx, coords, n: int) -> np.ndarray:
    """(n, 2 + d) float64 rows [dist, global idx, coords...]; padded rows carry dist = +inf."""
    d = coords.shape[1] if coords.ndim == 2 else 0
    k = len(cand_dist)
    out = np.zeros((n, 2 + d))
    out[:, 0] = np.inf
    out[:k, 0] = cand_dist
    out[:k, 1] = np.asarray(cand_idx, dtype=np.float64)  # exact for idx < 2^53
    if k:
        out[:k, 2:] = coords
    return out


def merge_candidates(packed: np.ndarray, n: int):
    """Global top-n by (dist, idx) (the nth_element comparator, geometry.hpp:39-45) from the
    concatenated per-rank candidate packs. Returns (src_idx ascending, rho, src_points in the
    same order)."""
    order = np.lexsort((packed[:, 1], packed[:, 0]))[:n]
    sel = packed[order]
    if not np.all(np.isfinite(sel[:, 0])):
        raise ValueError("merge_candidates: fewer than n points across all shards")
    rho = float(sel[:, 0].max())  # geometry.hpp:52-53
    idx = sel[:, 1].astype(np.int64)
    srt = np.argsort(idx, kind="stable")  # geometry.hpp:50-51
    return idx[srt], rho, np.ascontiguousarray(sel[srt, 2:])


def all_gather_np(arr: np.ndarray, group=None, device=None) -> np.ndarray:
    """all_gather of equally-shaped float64 arrays (NCCL needs device tensors, gloo host)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(arr))
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    return torch.cat(parts).cpu().numpy()


def sharded_split(dev, points_local: np.ndarray, offset: int, center, n: int, xi: float, group=None,
                  device=None):
    """split_sources_targets over the union of all ranks' shards. `dev` is a Device (or any
    object with split_candidates / split_finish); returns (src_idx, rho, src_points, nt_local)."""
    cd, ci = dev.split_candidates(center, n)
    coords = points_local[np.asarray(ci, dtype=np.int64) - offset] if len(ci) else np.zeros((0, len(center)))
    packed = all_gather_np(pack_candidates(cd, ci, coords, n), group, device)
    src, rho, src_pts = merge_candidates(packed, n)
    nt = dev.split_finish(src, rho, xi, src_points=src_pts)
    return src, rho, src_pts, nt


def ordered_sum(partial: np.ndarray, group=None, device=None) -> np.ndarray:
    """Sum of per-rank partials in rank order (bitwise independent of NCCL's reduction tree)."""
    allp = all_gather_np(partial.reshape(1, -1), group, device)
    out = np.zeros(allp.shape[1])
    for row in allp:
        out += row
    return out.reshape(partial.shape)


def sharded_tsqr(dev, h: float, group=None, device=None) -> np.ndarray:
    """TSQR factor of the sharded block: each rank's m x m factor of its
    targets (kid_tsqr_r), all_gather, then every rank folds the stack in rank order
    (kid_tsqr_combine) -> the identical R with R^T R = K^T K of the whole block."""
    R = np.asarray(dev.tsqr_r(h), dtype=np.float64)
    m = R.shape[0]
    allR = all_gather_np(R.reshape(1, -1), group, device)
    return dev.tsqr_combine([row.reshape(m, m) for row in allR])
