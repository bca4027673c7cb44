"""Host logic of bench.py's partitioned batch (SURVEY.md §8(e) sequence-batch sharding; BASELINE
configs[2] "1/2/4/8 B200"): the LPT partition into ranks x waves, on CPU, including a world-size-2
gloo run where each rank derives its own share from the same costs."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _costs(n=64, seed=0):
    rng = np.random.default_rng(seed)
    return rng.integers(0, 900, n)          # Stage-1 pair counts per sequence (c3: ~150-600)


@pytest.mark.parametrize("world,cap,W", [(1, 43, 2), (2, 43, 1), (4, 43, 1), (8, 43, 1), (1, 20, 4), (1, 64, 1)])
def test_bins_cover_every_sequence_once_within_the_cap(world, cap, W):
    costs = _costs()
    bins, w = bench.bin_waves(costs, world, cap)
    assert w == W and len(bins) == world * W
    flat = sorted(i for b in bins for i in b)
    assert flat == list(range(costs.size))                   # a partition: each sequence exactly once
    assert max(len(b) for b in bins) <= cap                  # every wave fits the KV budget
    loads = [sum(int(costs[i]) + 1 for i in b) for b in bins]
    assert max(loads) - min(loads) <= int(costs.max()) + 1   # LPT: within one item of balance


def test_wave_count_grows_until_the_cap_holds():
    costs = np.zeros(100, np.int64)
    costs[:3] = 10_000                                       # three heavy sequences
    bins, W = bench.bin_waves(costs, 1, 30)
    assert W >= 4 and max(len(b) for b in bins) <= 30


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bins, W = bench.bin_waves(_costs(), world, 43)
    mine = bins[rank * W:(rank + 1) * W]
    got = [None] * world
    dist.all_gather_object(got, mine)
    ms, pairs = bench.reduce_max_sum(dist, "cpu", 1.0 + rank, 100 * (rank + 1))
    q.put((rank, got, ms, pairs))
    dist.destroy_process_group()


def test_two_ranks_take_disjoint_shares_of_the_same_plan():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(60)
    for rank, got, ms, pairs in res:
        flat = sorted(i for share in got for wave in share for i in wave)
        assert flat == list(range(64))
        assert ms == 2.0 and pairs == 300.0                   # max over ranks of the step time; sum of pairs


def test_dual_ceiling_picks_the_binding_bound():
    """roofline.dual: distinct bytes against the HBM peak vs staged (T + P) slice bytes against the
    L2 -> shared-memory rate; the larger time is the bound and frac_of_bound its fraction."""
    peak = bench.measured_peaks()[0]
    blk = 4 << 20                                             # one 32B-shape block, all layers, K and V
    # low sharing: (T + P) / U = 1.5 -> the HBM time is the larger one
    U, T, P = 1000, 500, 1000
    t_hbm = U * blk / (peak * 1e9)
    d = bench.dual_ceiling(U, T, P, U * blk, 1e3 * t_hbm / 0.9)
    assert d["bound"] == "hbm" and abs(d["frac_of_bound"] - 0.9) < 1e-9
    assert d["staged_bytes"] == (T + P) * blk and abs(d["staged_over_distinct"] - 1.5) < 1e-12
    # heavy sharing: (T + P) / U = 4 -> the staged bytes bind
    T, P = 1000, 3000
    t_l2 = (T + P) * blk / (bench.L2_DELIVERY_GBS * 1e9)
    assert t_l2 > t_hbm
    d = bench.dual_ceiling(U, T, P, U * blk, 1e3 * t_l2 / 0.5)
    assert d["bound"] == "l2_delivery" and abs(d["frac_of_bound"] - 0.5) < 1e-9
    assert abs(d["l2_frac"] - 0.5) < 1e-9
