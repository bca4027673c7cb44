#!/usr/bin/env python
"""Bandwidth probe of memshare_block_distance on synthetic pair lists (tuning tool, not a test).

Pool: the c2 pool (776 blocks x 4 MiB, 32B KV shape). Pair lists:
  c2       -- the real c2 candidate pairs (L2 reuse across targets)
  disjoint -- pairs (2i, 2i+1): every block read once, no reuse (pure HBM stream, 3.25 GB)
  chain    -- pairs (i, i+1): every block read twice (once as target, once as source)
  subset   -- disjoint pairs over the c2 pair list's distinct blocks only
Prints kernel time (CUDA events, 20 reps) and GB/s of distinct bytes.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import Caps, MemSharePath  # noqa: E402
from synth import workloads  # noqa: E402


def run(path, pairs_np, toff_np, reps=20):
    dev = path.dev
    P, T = pairs_np.size, toff_np.size - 1
    path.set_caps(Caps(step=path.caps.step, match=path.caps.match, pair=P, target=T))
    path.pairs.copy_(torch.as_tensor(pairs_np.view(np.uint8), device=dev))
    path.target_off[:T + 1].copy_(torch.as_tensor(toff_np, device=dev))
    path.num_pairs.fill_(P)
    path.num_targets.fill_(T)
    for _ in range(3):
        path.distance_call(1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        path.distance_call(1.0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    U = np.unique(np.concatenate([pairs_np["target_phys"], pairs_np["source_phys"]])).size
    slice_b = 16 * 8 * 128 * 2
    gbs = U * 64 * 2 * slice_b / (ms / 1e3) / 1e9
    return ms, U, gbs, P, T


def make_pairs(tp, sp, tl=None):
    n = len(tp)
    a = np.zeros(n, L.PAIR_DTYPE)
    a["target_phys"], a["source_phys"] = tp, sp
    a["target_logical"] = np.arange(n) if tl is None else tl
    a["source_logical"] = 0
    # group by target: target_idx increments when target_phys changes
    tidx = np.concatenate([[0], np.cumsum(np.diff(np.asarray(tp)) != 0)]).astype(np.int32)
    a["target_idx"] = tidx
    toff = np.concatenate([[0], np.flatnonzero(np.diff(tidx)) + 1, [n]]).astype(np.int64)
    return a, toff


def real_pairs(seed):
    w = workloads.c2(seed=seed)
    k, v, ls, bs = w.device_pool("cuda")
    b, sh = w.batch, w.shape
    path = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                        w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                        sh.head_dim, sh.block_size)
    path.autosize(w.tau_s)
    path.segment()
    path.candidates(w.tau_s)
    c = path.read_candidates()
    pr = c["pairs"]
    real = np.zeros(pr["seq"].size, L.PAIR_DTYPE)
    for f in L.PAIR_DTYPE.names:
        real[f] = pr[f]
    return path, real, c["target_off"]


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--seed2-only":      # for ncu captures
        path, real, toff = real_pairs(2)
        print(run(path, real, toff, reps=3))
        return
    for seed in (1, 2):
        path, real, toff = real_pairs(seed)
        ms, U, gbs, P, T = run(path, real, toff)
        print(f"{'c2 seed%d' % seed:18s} P={P:4d} T={T:4d} U={U:4d}  {ms * 1e3:8.1f} us  {gbs:8.1f} GB/s (distinct bytes)",
              flush=True)
        del path
        torch.cuda.empty_cache()
    w = workloads.c2(seed=0)
    k, v, ls, bs = w.device_pool("cuda")
    b, sh = w.batch, w.shape
    path = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                        w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                        sh.head_dim, sh.block_size)
    path.autosize(w.tau_s)
    path.segment()
    path.candidates(w.tau_s)
    c = path.read_candidates()
    pr = c["pairs"]
    real = np.zeros(pr["seq"].size, L.PAIR_DTYPE)
    for f in L.PAIR_DTYPE.names:
        real[f] = pr[f]
    nb = w.num_blocks
    cases = {"c2": (real, c["target_off"])}
    cases["disjoint"] = make_pairs(np.arange(0, nb - 1, 2), np.arange(1, nb, 2))
    cases["chain"] = make_pairs(np.arange(0, nb - 1), np.arange(1, nb))
    dist_blocks = np.unique(np.concatenate([pr["target_phys"], pr["source_phys"]]))
    m = dist_blocks.size // 2 * 2
    cases["subset"] = make_pairs(dist_blocks[0:m:2], dist_blocks[1:m:2])
    perm = np.random.default_rng(0).permutation(nb)
    cases["disjoint_shuffled"] = make_pairs(perm[0:nb - 1:2], perm[1:nb:2])
    for name, (pairs_np, toff) in cases.items():
        ms, U, gbs, P, T = run(path, pairs_np, toff)
        print(f"{name:18s} P={P:4d} T={T:4d} U={U:4d}  {ms * 1e3:8.1f} us  {gbs:8.1f} GB/s (distinct bytes)", flush=True)


if __name__ == "__main__":
    main()
