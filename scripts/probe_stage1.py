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
for _ in range(5):
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
