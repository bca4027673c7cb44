"""World-size-2 gloo tests of the multi-GPU host logic (no GPU here; NCCL replaced by gloo).

* sequence sharding: LPT assignment covers every sequence once and balances cost; per-rank
  counters all-reduce to the single-process totals;
* KV-head sharding: each rank computes the partial squared sums of its head slice, an all-reduce
  sums them, FINALIZE with the global h reproduces the unsharded distances (the oracle stands in
  for the kernel on both sides, so this checks the decomposition and the collective plumbing).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth import kv, traces


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _seq_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2507_21433_b200.sharding import lpt_assign
    _init(rank, world, port)
    b = traces.make_batch(3, 6, 1500, 32, 16, vocab=600, len_lo=8, len_hi=40)
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    full = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.5)
    costs = [int((full["pairs"]["seq"] == s).sum()) + 1 for s in range(6)]
    mine = lpt_assign(costs, world)[rank]
    # this rank's sub-batch
    sub = traces.TraceBatch(tokens=np.concatenate([b.seq_tokens(s) for s in mine]),
                            seq_tok_off=np.concatenate([[0], np.cumsum([b.seq_tokens(s).size for s in mine])]),
                            gen_start=b.gen_start[mine], final=b.final[mine], delim_ids=b.delim_ids, vocab=b.vocab)
    sseg = oracle.segment_steps(sub.tokens, sub.seq_tok_off, sub.gen_start, sub.final, sub.delim_ids)
    stab, _ = traces.identity_table(sub, 16)
    r = oracle.step_candidates(sub.tokens, sub.seq_tok_off, sseg, sub.delim_ids, stab, 16, 0.5)
    cnt = torch.tensor([r["matches"]["seq"].size, r["pairs"]["seq"].size, r["target_off"].size - 1, len(mine)],
                       dtype=torch.int64)
    dist.all_reduce(cnt)
    if rank == 0:
        q.put((cnt.tolist(), [full["matches"]["seq"].size, full["pairs"]["seq"].size, full["target_off"].size - 1, 6]))
    dist.destroy_process_group()


def _head_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2507_21433_b200.sharding import head_shard
    _init(rank, world, port)
    sh = kv.KVShape(3, 5, 16, 8)                       # 5 heads over 2 ranks -> 3 + 2 (uneven)
    b = traces.make_batch(1, 1, 400, 0, 8, vocab=300)
    tab, nbk = traces.identity_table(b, 8)
    s_, l_, p_ = kv.table_blocks(b.seq_tok_off, tab, 8)
    hl, h0 = head_shard(sh.num_kv_heads, world, rank)
    k, v, ls, bs = kv.host_pool(sh, nbk, h_local=hl)
    kv.fill_blocks_host(k, v, ls, bs, sh, b.tokens, b.seq_tok_off, s_, l_, p_, 5, 0.05, h_local=hl, head_offset=h0)
    rng = np.random.default_rng(0)
    a, c = rng.integers(0, nbk, 40), rng.integers(0, nbk, 40)
    sk, sv = oracle.partial_sq(k, v, ls, bs, 3, hl, 16, 8, a, c)       # PARTIAL on this rank's heads
    part = torch.from_numpy(np.stack([sk, sv], -1).copy())
    dist.all_reduce(part)                                             # the NCCL all-reduce of the GPU path
    D = oracle.finalize(part[..., 0].numpy(), part[..., 1].numpy(), 3, 8, sh.num_kv_heads)   # FINALIZE, global h
    if rank == 0:
        kf, vf, lsf, bsf = kv.host_pool(sh, nbk)
        kv.fill_blocks_host(kf, vf, lsf, bsf, sh, b.tokens, b.seq_tok_off, s_, l_, p_, 5, 0.05)
        Df = oracle.block_distance(kf, vf, lsf, bsf, 3, 5, 5, 16, 8, a, c)
        q.put((D, Df))
    dist.destroy_process_group()


def _run(fn):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    mp.start_processes(fn, args=(2, port, q), nprocs=2, join=True, start_method="spawn")
    return q.get(timeout=60)


def test_lpt_assignment_properties():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2507_21433_b200.sharding import head_shard, lpt_assign
    costs = [9, 1, 7, 3, 3, 8, 2, 2]
    parts = lpt_assign(costs, 3)
    assert sorted(i for p in parts for i in p) == list(range(8))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)
    assert [head_shard(10, 4, r) for r in range(4)] == [(3, 0), (3, 3), (2, 6), (2, 8)]
    assert [head_shard(8, 8, r) for r in range(8)] == [(1, r) for r in range(8)]


def test_sequence_sharding_counters_gloo():
    got, exp = _run(_seq_worker)
    assert got == exp


def test_head_sharded_partial_allreduce_gloo():
    D, Df = _run(_head_worker)
    assert np.allclose(D, Df, rtol=1e-13, atol=0)
