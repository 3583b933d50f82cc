"""World-size-2 gloo tests of the multi-GPU host layer (paper_1409_2802_b200/dist.py) on CPU.

The device is replaced by a CPU stand-in with the reference's arithmetic (sequential squared
differences, no FMA, correctly rounded sqrt) so the exchange logic -- candidate packing,
all_gather, global (dist, idx) selection, per-shard compaction, ordered Gram reduction -- is
checked against the single-process oracle without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


class CpuShard:
    """Test double for Device.split_candidates / split_finish on one shard."""

    def __init__(self, pts, offset):
        self.pts, self.offset = pts, offset
        self.dist = None
        self.tgt = None

    def split_candidates(self, center, n):
        p = self.pts
        acc = (p[:, 0] - center[0]) * (p[:, 0] - center[0])
        for k in range(1, p.shape[1]):
            acc = acc + (p[:, k] - center[k]) * (p[:, k] - center[k])
        self.dist = np.sqrt(acc)
        idx = np.arange(p.shape[0]) + self.offset
        order = np.lexsort((idx, self.dist))[: min(n, p.shape[0])]
        return self.dist[order], idx[order]

    def tsqr_r(self, h):  # stand-in for kid_tsqr_r on this shard's block
        from oracle import oracle as O
        return np.linalg.qr(O.kernel_matrix(self.pts[self.tgt - self.offset], self.src_pts, h), mode="r")

    def tsqr_combine(self, Rs):  # stand-in for kid_tsqr_combine
        return np.linalg.qr(np.concatenate(Rs), mode="r")

    def targets(self):
        return self.tgt

    def split_finish(self, src_idx, rho, xi, src_points=None):
        self.src_pts = src_points
        local = np.arange(self.pts.shape[0]) + self.offset
        keep = (self.dist >= xi * rho) & ~np.isin(local, src_idx)
        self.tgt = local[keep]
        self.nt = int(keep.sum())
        return self.nt

    # the device passes on this shard's block, with the oracle's arithmetic
    def _K(self, h):
        from oracle import oracle as O
        return O.kernel_matrix(self.pts[self.tgt - self.offset], self.src_pts, h)

    def row_norms(self, h):
        from oracle import oracle as O
        return O.row_norms(self._K(h))

    def recon_error(self, h, skel, P, flags=1):
        from oracle import oracle as O
        return O.residual_stats(self._K(h), skel, P)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, d, N, n, xi, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle as O
    from paper_1409_2802_b200 import dist as D
    allpts = O.gen_normal(d, N, 12345)
    lo, hi = N * rank // ws, N * (rank + 1) // ws
    shard = CpuShard(allpts[lo:hi], lo)
    center = allpts[77]
    src, rho, src_pts, nt = D.sharded_split(shard, allpts[lo:hi], lo, center, n, xi)
    # per-shard fused-pass partials (oracle arithmetic), reduced in rank order
    t = O.split_sources_targets(allpts, center, n, xi)
    K_local = O.kernel_matrix(allpts[shard.tgt], src_pts, 0.3)
    skel = np.array([0, 5, 9])
    P = np.random.default_rng(0).standard_normal((3, n))
    P[:, skel] = np.eye(3)
    sd, sk, DtD, KtK = O.residual_stats(K_local, skel, P)
    red = D.ordered_sum(np.concatenate([[sd, sk], DtD.ravel()]))
    R = D.sharded_tsqr(shard, 0.3)
    q.put((rank, src, rho, shard.tgt, red, R))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,N,n,xi", [(2, 4001, 50, 2.0), (3, 3000, 100, 1.0)])
def test_sharded_split_and_reduction_match_single_process(oracle, d, N, n, xi):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, d, N, n, xi, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allpts = oracle.gen_normal(d, N, 12345)
    ref = oracle.split_sources_targets(allpts, allpts[77], n, xi)
    for _, src, rho, _, _, _ in res:
        assert np.array_equal(src, ref.source_indices)
        assert rho == ref.rho
    tg = np.concatenate([r[3] for r in res])
    assert np.array_equal(tg, ref.target_indices)
    # reduced partial Grams == the full-data Grams
    K = oracle.kernel_matrix(allpts[ref.target_indices], allpts[ref.source_indices], 0.3)
    skel = np.array([0, 5, 9])
    P = np.random.default_rng(0).standard_normal((3, n))
    P[:, skel] = np.eye(3)
    sd, sk, DtD, _ = oracle.residual_stats(K, skel, P)
    red = res[0][4]
    assert np.array_equal(red, res[1][4])  # every rank holds the identical reduction
    assert red[0] == pytest.approx(sd, rel=1e-12) and red[1] == pytest.approx(sk, rel=1e-12)
    assert np.allclose(red[2:].reshape(n, n), DtD, rtol=1e-11, atol=1e-14 * np.abs(DtD).max())
    # sharded TSQR: identical factor on every rank, R^T R == K^T K of the whole block
    R = res[0][5]
    assert np.array_equal(R, res[1][5])
    assert np.allclose(R.T @ R, K.T @ K, rtol=0, atol=1e-12 * np.abs(K.T @ K).max())


def _compress_worker(rank, ws, port, d, N, n, xi, h, s, eps, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import oracle as O
    from paper_1409_2802_b200 import dist as D
    from paper_1409_2802_b200 import kernid as H
    allpts = O.gen_normal(d, N, 4242)
    lo, hi = N * rank // ws, N * (rank + 1) // ws
    shard = CpuShard(allpts[lo:hi], lo)
    src, rho, src_pts, nt = D.sharded_split(shard, allpts[lo:hi], lo, allpts[11], n, xi)
    skel, P, rel, fro, sample = D.sharded_compress_id(shard, allpts[lo:hi], lo, src_pts, eps, h, s, 99,
                                                      H.EUCLIDEAN_NORM)
    q.put((rank, skel, P, rel, fro, sample))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ws", [2, 3])
def test_sharded_compress_id_matches_single_process(oracle, ws):
    """compress_id on a block sharded over ws ranks (gloo): the EuclideanNorm weights gathered in rank
    order give the single-process sample, the host ID the same skeleton and P (bitwise), and the rank-
    ordered sum of the per-shard residual Grams the single-process rel_error (sampling.hpp:189-196,
    compress.hpp:168-215)."""
    d, N, n, xi, h, s, eps = 3, 6000, 60, 2.0, 0.35, 0.05, 1e-6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_compress_worker, args=(r, ws, port, d, N, n, xi, h, s, eps, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    allpts = oracle.gen_normal(d, N, 4242)
    t = oracle.split_sources_targets(allpts, allpts[11], n, xi)
    K = oracle.kernel_matrix(allpts[t.target_indices], allpts[t.source_indices], h)
    w = oracle.row_norms(K)
    sample = oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, K.shape[0], s, 99, w)
    ref = oracle.compress_id(K, sample, eps=eps)
    for _, skel, P, rel, fro, smp in res:
        assert np.array_equal(smp, sample)
        assert np.array_equal(skel, ref.skeleton)
        assert np.array_equal(P, ref.P)
        assert rel == pytest.approx(ref.rel_error, rel=1e-9)
    assert all(r[3] == res[0][3] for r in res)  # identical on every rank


def test_merge_candidates_tie_break():
    from paper_1409_2802_b200 import dist as D
    a = D.pack_candidates([1.0, 2.0], [5, 7], np.array([[0.5], [0.7]]), 3)
    b = D.pack_candidates([1.0, 1.5], [3, 9], np.array([[0.3], [0.9]]), 3)
    src, rho, pts = D.merge_candidates(np.concatenate([a, b]), 3)
    assert list(src) == [3, 5, 9] and rho == 1.5 and np.allclose(pts[:, 0], [0.3, 0.5, 0.9])
