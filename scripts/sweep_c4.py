#!/usr/bin/env python
"""Threshold sweep on the c4 configuration (BASELINE.json configs[3]: Phi-4-reasoning-plus KV
shape, 40 layers x 10 KV heads x 128, a batch of 128 AIME-length synthetic traces L ~ U[8192,
16620]), over the WHOLE batch.

The 128 traces do not fit one GPU (~430 GB of KV); they run as bench.py's waves (the same LPT
plan, <= 140 GB of KV each). While a wave's pool is resident every (tau_s, tau_b) point gets one
full a1-a7 pass (state restored first), timed with CUDA events on the launching stream (median of
--reps), and its outcome is read back; the per-point numbers are summed over the waves: Stage-1
matches, candidate pairs, targets, accepted targets, freed blocks and the affected-token ratio
(changed targets x d / total tokens), to set beside Table 2's MemShare affected
ratios (8.3-27.4 %). tau_b is an absolute distance ceiling (R21); the
generator's closed form puts exact copies at ~0.063 and one mutated token at ~0.32 for this shape.

  python scripts/sweep_c4.py [--seqs 128] [--reps 3]   -> one JSON line per point (stdout)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import MemSharePath  # noqa: E402
from synth import workloads  # noqa: E402

TAU_S = [0.7, 0.8, 0.9, 0.95]
TAU_B = [0.05, 0.1, 0.15, 0.25, 0.4, 0.6, 0.9, 1.2]
KEYS = ("matches", "pairs", "targets", "accepted", "freed_blocks", "affected_tokens", "round_us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=128)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    bins, W, _ = bench.plan_waves("c4", args.seqs, 1, args.seed, dev)
    acc = {(ts, tb): dict.fromkeys(KEYS, 0) for ts in TAU_S for tb in TAU_B}
    total_tokens = 0
    st = torch.cuda.current_stream()
    for idx in bins:
        w = workloads.batch("c4", idx, args.seed)
        sh, b = w.shape, w.batch
        total_tokens += int(b.tokens.size)
        k, v, ls, bs = w.device_pool(dev)
        p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount,
                         w.free_list, w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads,
                         sh.num_kv_heads, sh.head_dim, sh.block_size)
        p.autosize(min(TAU_S), slack=1.05)              # the lowest tau_s has the most matches / pairs
        pristine = p.state.clone()

        def one(ts, tb):
            p.state.copy_(pristine)
            p.segment()
            p.candidates(ts)
            p.distance_call(tb)
            p.remap()

        for ts in TAU_S:
            for tb in TAU_B:
                one(ts, tb)
                torch.cuda.synchronize()
                times = []
                for _ in range(args.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    one(ts, tb)
                    e1.record(st)
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1) * 1e3)
                assert p.read_status() == 0, L.status_string(p.read_status())
                c = p.counts()
                dec = p.read_distance()["decisions"]
                s = p.read_state()
                a = acc[(ts, tb)]
                for key, val in (("matches", c["matches"]), ("pairs", c["pairs"]), ("targets", c["targets"]),
                                 ("accepted", int(np.count_nonzero(dec["accepted"]))),
                                 ("freed_blocks", s["num_freed"]), ("affected_tokens", s["affected"]),
                                 ("round_us", float(np.median(times)))):
                    a[key] += val
        del p, k, v
        torch.cuda.empty_cache()
    print(json.dumps({"config": "configs[3] c4", "shape": "Phi-4-reasoning-plus (N=40, h=10, d_h=128, d=16)",
                      "seqs": args.seqs, "waves": len(bins), "tokens": total_tokens,
                      "default_tau_b": round(workloads.default_tau_b(workloads.BATCHES["c4"][2], 0.05), 6),
                      "note": "per point: sums over the waves; round_us = sum of the waves' a1-a7 times"}), flush=True)
    for ts in TAU_S:
        for tb in TAU_B:
            a = acc[(ts, tb)]
            print(json.dumps({"tau_s": ts, "tau_b": tb, **{k_: a[k_] for k_ in KEYS if k_ != "round_us"},
                              "affected_ratio": round(a["affected_tokens"] / total_tokens, 5),
                              "round_us": round(a["round_us"], 1),
                              "pairs_per_s": round(a["pairs"] / (a["round_us"] * 1e-6))}), flush=True)


if __name__ == "__main__":
    main()
