#!/usr/bin/env python
"""Phase timing of the stage1 kernel in an ONLINE round on c2 (tuning tool): the one CTA that
owns the current (last) step, MEMSHARE_DEBUG_SKIP=8 (globaltimer stamps)."""
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
if "--hot" in sys.argv:                       # keep the SM clock up: a busy GPU right before
    x = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(200):
        x @ x
for _ in range(50):
    path.segment()
    path.candidates(w.tau_s, cur_mode=L.CUR_LAST)
torch.cuda.synchronize()
buf = np.zeros(2048 * 16, np.uint64)
L.lib.memshare_debug_stage1_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.lib.memshare_debug_stage1_times(buf.ctypes.data, buf.size) == 0
t = buf.reshape(2048, 16).astype(np.int64)
G = int(path.seq_step_off[-1].item())
cs = int(os.environ.get("CS", "8"))
ncl = 148 // cs
n = ncl * cs
t0 = t[:n, 0].min()
owner = 0                                    # LAST mode: sequence 0 -> cluster 0
for r in range(cs):
    rr = (t[owner + r] - t0) / 1e3
    print(f"rank {r}: start {rr[0]:.2f} table {rr[1]:.2f} staged {rr[10]:.2f} loop-end {rr[7]:.2f}")
r = (t[owner] - t0) / 1e3
names = {0: "start", 1: "table", 10: "hist staged", 14: "tokens staged", 11: "stream done", 2: "select", 3: "sort", 4: "stash",
         5: "prepare", 6: "count", 7: "loop end"}
print("steps", G, "owner CTA", owner)
for k in (0, 1, 10, 14, 11, 2, 3, 4, 5, 6, 7):
    print(f"  {names[k]:12s} {r[k]:7.2f} us")
cyc = t[owner, 13] - t[owner, 12]
ns = t[owner, 11] - t[owner, 10]
print(f"stream: {cyc} SM cycles in {ns} ns -> {cyc / max(ns, 1):.3f} GHz")
lastc = int(np.argmax(t[:n, 8]))
print("last CTA", lastc, "elected", (t[lastc, 8] - t0) / 1e3, "scans done", (t[lastc, 9] - t0) / 1e3)
print("other CTAs loop end: median %.2f max %.2f" % (np.median((t[:n, 7] - t0) / 1e3), ((t[:n, 7] - t0) / 1e3).max()))
