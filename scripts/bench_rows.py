#!/usr/bin/env python
"""Measurement of the SURVEY.md §8(f) rows (f1-f4) and the CROSS pairing mode on B200.

Each row is timed with CUDA events on the launching stream (warm, after a synchronize on both
sides) and reported against the HBM roofline with its algorithmic bytes:

  f1 paged decode attention  bytes = sum_s len_s * h * d_h * 2 (K and V) * 2 B  (+ q/out)
  f1 KV append               bytes = 2 (K,V) * N * S * h * d_h * 2 B read + the same written
  f2 cosine block metric     bytes = U * B_blk (distinct blocks)  -- same stream as Euclidean
  CROSS pairing              bytes = U * B_blk; units = scored pairs
  f3 all-pairs matrix        bytes = W * B_blk (the window's blocks); units = W(W-1)/2 pairs
  f4 similarity ratio        latency only (reads the Stage-1 matches)

Prints one JSON line per row (stdout). Not part of the product; inputs are synthetic (synth/).
  python scripts/bench_rows.py [--rows f1,f2,cross,f3,f4]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import Caps, MemSharePath  # noqa: E402
from synth import decode as sd  # noqa: E402
from synth import workloads  # noqa: E402


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"])
    return 6650.0


PEAK = peak()
FLUSH = None
# CUDA-core ceiling of the distance inner loop (one FHFMA.BF16 + half an FFMA2 per bf16 element
# pair), measured on this pool's B200 by scripts/alu_peak.cu (registers only, 16-64 warps/SM)
ALU_PEAK = 13.4e12


def EP(sh):
    """element pairs per block pair (K and V, all layers)"""
    return sh.num_layers * 2 * sh.block_size * sh.num_kv_heads * sh.head_dim


def flush_l2():
    """Evict L2 by READING a 512 MB buffer (a write-based flush would leave ~126 MB of dirty lines
    whose write-back then competes with the timed kernel's reads)."""
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.ones(64 << 20, dtype=torch.int64, device="cuda")
    FLUSH.sum()


def time_us(fn, reps=30, flush=False, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    st = torch.cuda.current_stream()
    for _ in range(reps):
        if flush:
            flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def graph_us(p, fn, n_rep=200):
    """Per-replay device time of `fn` captured as one CUDA graph (no host launch gaps)."""
    fn()
    torch.cuda.synchronize()
    g = p.capture(fn)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n_rep):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n_rep


def emit(row, **kv):
    rec = {"row": row, **kv}
    if "bytes" in kv and "us" in kv:
        gbs = kv["bytes"] / (kv["us"] * 1e-6) / 1e9
        rec["GB/s"] = round(gbs, 1)
        rec["frac_of_peak"] = round(gbs / PEAK, 4)
        rec["peak_gbs"] = PEAK
    print(json.dumps(rec), flush=True)


def path_for(w, caps=None):
    k, v, ls, bs = w.device_pool("cuda")
    b, sh = w.batch, w.shape
    p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                     w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                     sh.head_dim, sh.block_size, caps=caps)
    torch.cuda.synchronize()
    return p


def distinct_bytes(p, sh):
    pr = p.read_candidates()["pairs"]
    U = int(np.unique(np.concatenate([pr["target_phys"], pr["source_phys"]])).size)
    return U, U * sh.num_layers * 2 * sh.block_size * sh.num_kv_heads * sh.head_dim * 2, int(pr["seq"].size)


def row_f2_cross(rows):
    w = workloads.c2()
    sh = w.shape
    p = path_for(w)
    if "f2" in rows:
        p.autosize(w.tau_s)
        p.segment()
        p.candidates(w.tau_s)
        U, byts, P = distinct_bytes(p, sh)
        eu = time_us(lambda: p.distance_call(w.tau_b))
        co = time_us(lambda: p.distance_call(w.tau_b, metric=L.METRIC_COSINE))
        assert p.read_status() == 0
        emit("a5-a6 euclidean (reference point)", workload="c2 aligned", pairs=P, distinct_blocks=U, bytes=byts, us=eu,
             pairs_per_s=P / (eu * 1e-6))
        emit("f2 cosine block metric", workload="c2 aligned", pairs=P, distinct_blocks=U, bytes=byts, us=co,
             pairs_per_s=P / (co * 1e-6))
    if "cross" in rows:
        p.autosize(w.tau_s, pairing=L.PAIR_CROSS)
        p.segment()
        p.candidates(w.tau_s, pairing=L.PAIR_CROSS)
        U, byts, P = distinct_bytes(p, sh)
        t = time_us(lambda: p.distance_call(w.tau_b))
        assert p.read_status() == 0
        slices = P + int(p.counts()["targets"])
        emit("f2 CROSS pairing distance", workload="c2 cross", pairs=P, distinct_blocks=U, bytes=byts, us=t,
             pairs_per_s=P / (t * 1e-6), slice_reads_per_layer=slices,
             ingest_GBps=round(slices * sh.num_layers * 2 * 32768 / (t * 1e-6) / 1e9, 1),
             elem_pairs_per_s=P * EP(sh) / (t * 1e-6), frac_of_alu_peak=round(P * EP(sh) / (t * 1e-6) / ALU_PEAK, 4))
    if "f4" in rows:
        p.set_caps(Caps(step=p.caps.step, match=max(1024, p.num_tokens), pair=p.caps.pair, target=p.caps.target))
        p.segment()
        p.candidates(0.8, top_k=1)
        t_eager = time_us(lambda: p.similarity_ratio(), reps=100)      # includes the host-side launch gaps
        t = graph_us(p, lambda: p.similarity_ratio())
        red = p.similarity_ratio().cpu().numpy()
        emit("f4 similarity ratio", workload="c2 tau_s=0.8", us=t, eager_call_us=t_eager,
             redundant_steps=int(red.sum()), steps=int(p.counts()["steps"]),
             note="us: one graph replay of the call (output zeroing + the count kernel); eager_call_us: "
                  "events around the eager Python call, dominated by host launch gaps")
    del p
    torch.cuda.empty_cache()


def row_f3(rows):
    w = workloads.c2()
    sh = w.shape
    Wn = 96                       # window of full blocks after the prompt: 96*95/2 = 4560 pairs
    b0 = 8
    p = path_for(w, caps=Caps(step=w.num_tokens, match=1024, pair=Wn * (Wn - 1) // 2, target=Wn))
    t_ap_eager = time_us(lambda: p.all_pairs([b0], [b0 + Wn]), reps=50)   # host launch gaps included
    bb = torch.tensor([b0], dtype=torch.int32, device="cuda")
    be = torch.tensor([b0 + Wn], dtype=torch.int32, device="cuda")
    t_ap = graph_us(p, lambda: p.all_pairs(bb, be))
    p.all_pairs([b0], [b0 + Wn])
    U, byts, P = distinct_bytes(p, sh)
    t = time_us(lambda: p.distance_call(w.tau_b))
    assert p.read_status() == 0
    emit("f3 all-pairs block matrix", workload=f"c2 window of {Wn} blocks", pairs=P, distinct_blocks=U, bytes=byts,
         us=t, pairs_per_s=P / (t * 1e-6), all_pairs_enum_us=t_ap, all_pairs_enum_eager_us=t_ap_eager,
         elem_pairs_per_s=P * EP(sh) / (t * 1e-6), frac_of_alu_peak=round(P * EP(sh) / (t * 1e-6) / ALU_PEAK, 4),
         note="bytes = distinct blocks once; every source is re-read from L2 by later targets")
    del p
    torch.cuda.empty_cache()


def row_f1(rows):
    # QwQ-32B decode shape: 40 query heads, 8 KV heads, d_h 128, block 16; 32 x 12,288-token CoTs
    S, n, N, h, dh, d, hq = 32, 12288, 4, 8, 128, 16, 40
    nbs = -(-n // d)
    nb = S * nbs + 8
    sl = d * h * dh
    dev = torch.device("cuda")
    k = torch.randn(N * nb * sl, dtype=torch.bfloat16, device=dev)
    v = torch.randn(N * nb * sl, dtype=torch.bfloat16, device=dev)
    rng = np.random.default_rng(0)
    table = torch.as_tensor(rng.permutation(nb)[:S * nbs].reshape(S, nbs).astype(np.int32), device=dev)
    lens_h = rng.integers(n // 2, n + 1, S).astype(np.int32)
    lens = torch.as_tensor(lens_h, device=dev)
    q = torch.as_tensor(sd.gaussian_bf16(rng, (S, hq, dh)).view(np.int16), device=dev)
    out = torch.empty(S, hq, dh, dtype=torch.float32, device=dev)
    dims = L.Dims(N, h, h, dh, d)
    pool = L.KVPool(k.data_ptr(), v.data_ptr(), nb * sl, sl, nb, 0)
    ws = torch.empty(L.paged_attention_workspace_size(dims, S, hq, n), dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    layer = [0]

    def call():
        L.check(L.paged_attention_decode(pool, dims, layer[0] % N, q, hq, table, nbs, lens, S, n,
                                         1 / math.sqrt(dh), out, ws, st))
        layer[0] += 1
    t = time_us(call, reps=40, flush=True)
    assert st.item() == 0
    byts = int(lens_h.astype(np.int64).sum()) * h * dh * 2 * 2 + S * hq * dh * (2 + 4)
    emit("f1 paged decode attention", workload=f"QwQ-32B decode shape (hq {hq}, h {h}, d_h {dh}), {S} seqs, "
         f"len U[{n // 2},{n}], one layer, random block placement", bytes=byts, us=t,
         tokens_per_s=float(lens_h.sum()) / (t * 1e-6))
    del k, v
    torch.cuda.empty_cache()
    # KV append: one decode token for 256 sequences into a 64-layer pool
    S2, N2 = 256, 64
    nb2 = S2 * 4 + 64
    k2 = torch.zeros(N2 * nb2 * sl, dtype=torch.bfloat16, device=dev)
    v2 = torch.zeros_like(k2)
    dims2 = L.Dims(N2, h, h, dh, d)
    tab2 = torch.full((S2, 4), -1, dtype=torch.int32, device=dev)
    tab2[:, 0] = torch.arange(S2, dtype=torch.int32, device=dev)
    seq_len0 = torch.full((S2,), 1, dtype=torch.int32, device=dev)     # appends land in the private block
    rc = torch.zeros(nb2, dtype=torch.int32, device=dev)
    rc[:S2] = 1
    fl = torch.arange(S2, nb2, dtype=torch.int32, device=dev)
    fc = torch.tensor([nb2 - S2], dtype=torch.int64, device=dev)
    nk = torch.randn(N2 * S2 * h * dh, dtype=torch.bfloat16, device=dev)
    nv = torch.randn_like(nk)
    ws2 = torch.empty(max(1, L.kv_append_workspace_size(S2)), dtype=torch.uint8, device=dev)
    seq_len = seq_len0.clone()

    def app():
        seq_len.copy_(seq_len0)
        L.check(L.kv_append(k2, v2, nb2 * sl, sl, nb2, dims2, tab2, 4, S2, seq_len, None, rc, fl, fc, nk, nv, ws2, st))
    t2 = time_us(app, reps=50, flush=True)
    assert st.item() == 0
    byts2 = 2 * 2 * N2 * S2 * h * dh * 2
    emit("f1 KV append", workload=f"{S2} seqs x {N2} layers x {h} heads x {dh}, one token each", bytes=byts2, us=t2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="f1,f2,cross,f3,f4")
    rows = set(ap.parse_args().rows.split(","))
    torch.cuda.set_device(0)
    if rows & {"f2", "cross", "f4"}:
        row_f2_cross(rows)
    if "f3" in rows:
        row_f3(rows)
    if "f1" in rows:
        row_f1(rows)


if __name__ == "__main__":
    main()
