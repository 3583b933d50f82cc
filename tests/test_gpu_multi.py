"""The C++ multi-GPU mirror (kernid_multi.cpp: DeviceGroup, sharded split, ShardedBlock, compress_id with
NCCL-reduced Grams) against the single-GPU mirror and the oracle. This project has one GPU, so the
group lists device 0 once (a 1-rank NCCL communicator: the NCCL code path) or several times (several
contexts on one GPU: the host-reduction path) -- the sharding, the merged split, the gathered
EuclideanNorm weights and the reduced Grams are exercised either way."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
@pytest.mark.parametrize("d,N,n,eps", [(3, 30_000, 100, 1e-6), (8, 20_000, 512, 1e-2)])
def test_sharded_trial_matches_single_gpu(oracle, devices, d, N, n, eps):
    from paper_1409_2802_b200 import kernid as H
    seed = H.derive_seed(1, 0, 0)
    single = H.compress_trial(d, N, n, 2.0, seed, H.EUCLIDEAN_NORM, 0.05, H.derive_seed(seed, 0, 1), eps)
    sharded, nccl = H.sharded_compress_trial(devices, d, N, n, 2.0, seed, 0.05, H.derive_seed(seed, 0, 1), eps)
    assert nccl == (len(devices) == 1)
    assert sharded.n_targets == single.n_targets
    assert np.array_equal(sharded.sample, single.sample)  # weights gathered in global target order
    assert sharded.rank == single.rank and np.array_equal(sharded.skeleton, single.skeleton)
    assert sharded.rel_error == pytest.approx(single.rel_error, rel=1e-9)
    assert sharded.rel_error_fro == pytest.approx(single.rel_error_fro, rel=1e-9)
    # and the oracle pipeline on the whole block
    t = oracle.prepare_trial(d, N, n, 2.0, seed)
    K = oracle.kernel_matrix(t.targets, t.sources, t.h)
    assert np.array_equal(sharded.sample,
                          oracle.sample_rows(oracle.SCHEME_EUCLIDEAN, K.shape[0], 0.05, H.derive_seed(seed, 0, 1),
                                             oracle.row_norms(K)))
    ref = oracle.compress_id(K, sharded.sample, eps=eps)
    assert np.array_equal(ref.skeleton, sharded.skeleton)
    floor = 1e-13 / max(ref.rel_error, 1e-300)
    assert abs(sharded.rel_error - ref.rel_error) <= max(1e-9, floor) * ref.rel_error
