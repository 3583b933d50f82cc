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


def all_gather_ragged(arr: np.ndarray, group=None, device=None) -> np.ndarray:
    """all_gather of 1-D float64 arrays of different lengths, concatenated in rank order."""
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    n = np.array([float(arr.size)])
    sizes = all_gather_np(n, group, device).astype(np.int64)
    width = int(max(1, sizes.max()))
    pad = np.zeros(width)
    pad[: arr.size] = arr
    allp = all_gather_np(pad.reshape(1, -1), group, device)
    return np.concatenate([allp[g, : sizes[g]] for g in range(ws)])


def sharded_sample_rows(dev, points_local: np.ndarray, offset: int, src_pts: np.ndarray, h: float, s: float,
                        seed: int, scheme: int, group=None, device=None, weights_fn=None):
    """sample_rows (sampling.hpp:156-243) over the targets of ALL shards, then the sampled kernel rows.

    Each rank computes the weights of its own targets (EuclideanNorm: kid_row_norms, sampling.hpp:189-196;
    or weights_fn() -- e.g. leverage scores, sampling.hpp:212-221); the weight vectors are gathered in
    rank order -- the global target order, shards being contiguous index ranges -- and every rank draws
    the identical sample with the reference seed stream (the host draw, sampling.hpp:78-149). The
    sampled rows K(T[sample], S) are evaluated with the reference arithmetic by the rank that holds the
    target and gathered, so every rank then runs the identical host ID.
    Returns (sample positions in the global target list, K_s (count x m), global target count)."""
    from . import kernid as H
    d = points_local.shape[1]
    if scheme == H.UNIFORM:
        w_local = np.zeros(0)
        nt_local = dev.nt
        counts = all_gather_np(np.array([float(nt_local)]), group, device).astype(np.int64)
        NT = int(counts.sum())
        sample = H.draw(H.UNIFORM, NT, s, seed)
    else:
        w_local = weights_fn() if weights_fn is not None else dev.row_norms(h)
        counts = all_gather_np(np.array([float(w_local.size)]), group, device).astype(np.int64)
        w = all_gather_ragged(np.asarray(w_local, dtype=np.float64), group, device)
        NT = w.size
        sample = H.draw(scheme, NT, s, seed, w)
    import torch.distributed as dist
    rank = dist.get_rank(group)
    lo = int(counts[:rank].sum())
    hi = lo + int(counts[rank])
    mine = np.nonzero((sample >= lo) & (sample < hi))[0]  # positions in the sample held by this rank
    m = src_pts.shape[0]
    rows = np.zeros((sample.size, m))
    if mine.size:
        tgt_local = dev.targets() - offset
        pts = np.concatenate([points_local, src_pts])  # sources may live on other shards
        pcm = np.ascontiguousarray(pts.T).ravel()
        src_idx = np.arange(points_local.shape[0], pts.shape[0], dtype=np.int64)
        rows[mine] = H.kernel_rows(pcm, pts.shape[0], d, tgt_local, sample[mine] - lo, src_idx, h)
    # each sampled row is held by exactly one rank: the ordered sum over ranks assembles K_s exactly
    Ks = ordered_sum(rows, group, device)
    return sample, Ks, NT


def sharded_compress_id(dev, points_local: np.ndarray, offset: int, src_pts: np.ndarray, skel_rule_eps: float,
                        h: float, s: float, seed: int, scheme: int, group=None, device=None):
    """compress_id (compress.hpp:168-215) on the sharded block: the sample and K_s over all shards
    (sharded_sample_rows), the host ID (identical on every rank), the fused error pass on each shard,
    [||D||^2, ||K||^2, D^T D, K^T K] summed in rank order, rel_error = sqrt(lmax(D^T D) / lmax(K^T K)).
    Returns (skeleton, P, rel_error, rel_error_fro, sample)."""
    from . import kernid as H
    sample, Ks, _ = sharded_sample_rows(dev, points_local, offset, src_pts, h, s, seed, scheme, group, device)
    r = H.epsilon_rank(H.singular_values(Ks), skel_rule_eps)
    m = Ks.shape[1]
    if r == 0:
        return np.zeros(0, np.int64), np.zeros((0, m)), 1.0, 1.0, sample
    skel, P = H.interpolative_decomposition(Ks, r)
    sd, sk, DtD, KtK = dev.recon_error(h, skel, P, flags=3)
    red = ordered_sum(np.concatenate([[sd, sk], DtD.ravel(), KtK.ravel()]), group, device)
    nz = np.setdiff1d(np.arange(m), skel)
    D2 = red[2:2 + m * m].reshape(m, m)[np.ix_(nz, nz)]
    num = H.lambda_max(D2) if nz.size else 0.0
    den = H.lambda_max(red[2 + m * m:].reshape(m, m))
    rel = float(np.sqrt(num / den)) if den > 0 else 0.0
    fro = float(np.sqrt(red[0] / red[1])) if red[1] > 0 else 0.0
    return skel, P, rel, fro, sample
