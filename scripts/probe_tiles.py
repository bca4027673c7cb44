#!/usr/bin/env python
"""Tuning probe (not a test): memshare_block_distance on the c2 pair lists of seeds 0-4
(ALIGNED and CROSS) and synthetic lists; prints the whole call and the streaming kernel alone
(library profiling hook), as time, GB/s of distinct bytes and fraction of the measured HBM peak,
plus element-pairs/s against the measured ALU ceiling for the L2-heavy lists.

  python scripts/probe_tiles.py [--seeds 0,1,2,3,4] [--cross] [--json out.jsonl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import MemSharePath  # noqa: E402
from synth import workloads  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6544.7
ALU = 13.4e12     # measured FHFMA.BF16 + FFMA2 element pairs / s (scripts/alu_peak.cu)


def timed(path, tau_b, reps=30):
    ev = lambda: torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        path.distance_call(tau_b)
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    for _ in range(reps):
        path.distance_call(tau_b)
    e1.record()
    torch.cuda.synchronize()
    call_ms = e0.elapsed_time(e1) / reps
    kb, ke = ev(), ev()
    kb.record()
    ke.record()
    torch.cuda.synchronize()
    L.profile_distance_events(kb, ke)
    ks = []
    for _ in range(reps):
        path.distance_call(tau_b)
        torch.cuda.synchronize()
        ks.append(kb.elapsed_time(ke))
    L.profile_distance_events(None, None)
    return call_ms, float(np.median(ks))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", default="0,1,2,3,4")
    ap.add_argument("--cross", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    out = open(args.json, "a") if args.json else None
    for seed in [int(x) for x in args.seeds.split(",")]:
        w = workloads.c2(seed=seed)
        k, v, ls, bs = w.device_pool("cuda")
        b, sh = w.batch, w.shape
        path = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount,
                            w.free_list, w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads,
                            sh.num_kv_heads, sh.head_dim, sh.block_size)
        for pairing in ([L.PAIR_ALIGNED, L.PAIR_CROSS] if args.cross else [L.PAIR_ALIGNED]):
            path.autosize(w.tau_s, pairing=pairing)
            path.segment()
            path.candidates(w.tau_s, pairing=pairing)
            c = path.read_candidates()
            pr = c["pairs"]
            P, T = pr["seq"].size, c["target_off"].size - 1
            U = np.unique(np.concatenate([pr["target_phys"], pr["source_phys"]])).size
            call_ms, k_ms = timed(path, w.tau_b)
            assert path.read_status() == 0
            byts = U * sh.block_bytes
            ep = P * sh.num_layers * 2 * sh.slice_elems
            rec = {"seed": seed, "pairing": "cross" if pairing else "aligned", "P": P, "T": T, "U": U,
                   "call_us": call_ms * 1e3, "kernel_us": k_ms * 1e3,
                   "call_frac": byts / (call_ms / 1e3) / 1e9 / PEAK, "kernel_frac": byts / (k_ms / 1e3) / 1e9 / PEAK,
                   "kernel_alu_frac": ep / (k_ms / 1e3) / ALU, "pairs_per_s_call": P / (call_ms / 1e3)}
            print(json.dumps({k_: (round(v_, 4) if isinstance(v_, float) else v_) for k_, v_ in rec.items()}),
                  flush=True)
            if out:
                out.write(json.dumps(rec) + "\n")
        del path, k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
