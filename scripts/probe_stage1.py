#!/usr/bin/env python
"""Phase timing of the stage1 kernel on c2 (tuning tool): run with MEMSHARE_DEBUG_SKIP=8."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MEMSHARE_DEBUG_SKIP", "8")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import MemSharePath  # noqa: E402
from synth import workloads  # noqa: E402

w = workloads.c2(seed=0)
b, sh = w.batch, w.shape
path = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                    w.free_count, None, None, 0, 0, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                    sh.head_dim, sh.block_size)
path.autosize(w.tau_s)
for _ in range(300):
    path.segment()
    path.candidates(w.tau_s)
torch.cuda.synchronize()
buf = np.zeros(2048 * 16, np.uint64)
L.lib.memshare_debug_stage1_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.lib.memshare_debug_stage1_times(buf.ctypes.data, buf.size) == 0
t = buf.reshape(2048, 16).astype(np.int64)
G = int(path.seq_step_off[-1].item())
act = t[:min(G, 148)]
t0 = act[:, 0].min()
names = ["start", "table", "stream+select", "sort", "stash", "prepare", "count", "pre-last", "last-elected", "scans"]
rel = act[:, :10] - t0
print("steps", G, "CTAs", act.shape[0])
end = rel[:, 7].argmax()
print("slowest CTA (by pre-last):", end, "phases (us from kernel start):", (rel[end, :8] / 1e3).round(2).tolist())
print("median CTA phases:", (np.median(rel[:, :8], axis=0) / 1e3).round(2).tolist())
lastc = np.argmax(t[:148, 8])
print("last-CTA scan: elected at", (t[lastc, 8] - t0) / 1e3, "us, scans done at", (t[lastc, 9] - t0) / 1e3, "us")
for i, n in enumerate(names[:8]):
    d = (rel[:, i + 1] - rel[:, i]) / 1e3 if i < 7 else None
    if d is not None:
        print(f"  {n:14s} -> {names[i + 1]:14s}: median {np.median(d):6.2f} us  max {d.max():6.2f} us")

d1 = (act[:, 10] - act[:, 1]) / 1e3
d2 = (act[:, 11] - act[:, 10]) / 1e3
d3 = (act[:, 2] - act[:, 11]) / 1e3
print("table->stage hist: median %.2f max %.2f; stream: median %.2f max %.2f; select: median %.2f max %.2f" %
      (np.median(d1), d1.max(), np.median(d2), d2.max(), np.median(d3), d3.max()))

print("raw stamps 10..14 of 4 CTAs:\n", (act[:4, 10:15] - t0))
a12 = act[:, 12]; a13 = act[:, 13]; a14 = act[:, 14]
ok = (a12 > 0) & (a14 > a12)
if not ok.any():
    ok = None
if ok is not None: print("thread0 first run: loads %.2f us, process %.2f us (median over CTAs); max loads %.2f, max process %.2f" %
      (np.median((a13 - a12)[ok]) / 1e3, np.median((a14 - a13)[ok]) / 1e3, ((a13 - a12)[ok]).max() / 1e3, ((a14 - a13)[ok]).max() / 1e3))
if ok is not None: print("stream start offset from kernel start (median, max):", np.median((a12 - t0)[ok]) / 1e3, ((a12 - t0)[ok]).max() / 1e3)

if ok is not None:
  cyc = act[:, 15][ok]; ns = (a14 - a13)[ok]
  print("effective SM clock during processing: median %.0f MHz" % np.median(cyc / np.maximum(ns, 1) * 1e3))

tk = np.zeros(2048 * 32, np.int64)
L.lib.memshare_debug_stage1_tok.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.lib.memshare_debug_stage1_tok(tk.ctypes.data, tk.size)
tk = tk.reshape(2048, 32)
for c in (1, 60, 122, 135):
    row = tk[c]
    st = row[31]
    d = np.diff(np.concatenate([[st], row[:30][row[:30] > 0]]))
    print("CTA", c, "per-token cycles:", d[:16].tolist())
