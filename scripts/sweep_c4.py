#!/usr/bin/env python
"""Threshold sweep on the c4 configuration (BASELINE.json configs[3]: Phi-4-reasoning-plus KV
shape, 40 layers x 10 KV heads x 128, AIME-length synthetic traces L ~ U[8192, 16620]).

For every (tau_s, tau_b) point one full a1-a7 pass (state restored first) is timed with CUDA
events on the launching stream (median of --reps) and its outcome is read back: Stage-1 matches,
candidate pairs, targets, accepted targets, freed blocks and the affected-token ratio (PAPER.md:421:
changed targets x d / total tokens), to set beside Table 2's MemShare affected ratios (8.3-27.4 %,
PAPER.md:386-399). tau_b is an absolute distance ceiling (R21); the generator's closed
form puts exact copies at ~0.063 and one mutated token at ~0.32 for this shape.

  python scripts/sweep_c4.py [--seqs 16] [--reps 5]   -> one JSON line per point (stdout)
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

from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import MemSharePath  # noqa: E402
from synth import workloads  # noqa: E402

TAU_S = [0.7, 0.8, 0.9, 0.95]
TAU_B = [0.05, 0.1, 0.15, 0.25, 0.4, 0.6, 0.9, 1.2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    w = workloads.c4(num_seqs=args.seqs, seed=args.seed)
    sh, b = w.shape, w.batch
    k, v, ls, bs = w.device_pool("cuda")
    p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                     w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                     sh.head_dim, sh.block_size)
    p.autosize(min(TAU_S), slack=1.05)              # the lowest tau_s has the most matches / pairs
    pristine = p.state.clone()
    total_tokens = int(b.tokens.size)
    st = torch.cuda.current_stream()
    print(json.dumps({"config": "configs[3] c4", "shape": "Phi-4-reasoning-plus (N=40, h=10, d_h=128, d=16)",
                      "seqs": args.seqs, "tokens": total_tokens, "pool_GB": round(w.pool_bytes() / 1e9, 2),
                      "default_tau_b": round(w.tau_b, 6)}), flush=True)

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
            us = float(np.median(times))
            print(json.dumps({"tau_s": ts, "tau_b": tb, "matches": c["matches"], "pairs": c["pairs"],
                              "targets": c["targets"], "accepted": int(np.count_nonzero(dec["accepted"])),
                              "freed_blocks": s["num_freed"], "affected_tokens": s["affected"],
                              "affected_ratio": round(s["affected"] / total_tokens, 5),
                              "round_us": round(us, 1), "pairs_per_s": round(c["pairs"] / (us * 1e-6))}), flush=True)


if __name__ == "__main__":
    main()
