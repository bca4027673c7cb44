#!/usr/bin/env python
"""Stage-1 (offline c2) warm vs L2-cold timing and per-phase stamps (tuning tool).

candidates() (encode + stage1 with the fused fill) is timed with CUDA events (a) back to back and
(b) after a 512 MB read that evicts L2 (as the distance kernel's KV stream does inside a step).
The stage1 phase stamps (MEMSHARE_DEBUG_SKIP=8, globaltimer) of the last call of each mode are
printed per phase: median / max over CTAs and the last step's CTA.
"""
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
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
L.lib.memshare_debug_stage1_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
G = None
names = {0: "start", 1: "table", 10: "hist-idx", 14: "tok-staged", 11: "streamed", 2: "selected", 3: "sorted",
         4: "stashed", 5: "prepared", 6: "counted", 8: "prefixed", 9: "scanned", 7: "end"}
order = [0, 1, 10, 14, 11, 2, 3, 4, 5, 6, 8, 9, 7]
for mode in ("warm", "cold"):
    ts, tseg = [], []
    for it in range(200):
        if mode == "cold":
            flush.sum()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(st)
        path.segment()
        e1.record(st)
        path.candidates(w.tau_s)
        e2.record(st)
        torch.cuda.synchronize()
        if it >= 20:
            tseg.append(e0.elapsed_time(e1) * 1e3)
            ts.append(e1.elapsed_time(e2) * 1e3)
    buf = np.zeros(2048 * 16, np.uint64)
    assert L.lib.memshare_debug_stage1_times(buf.ctypes.data, buf.size) == 0
    G = int(path.seq_step_off[-1].item())
    t = buf.reshape(2048, 16).astype(np.int64)[:G]
    t0 = t[:, 0].min()
    print(f"[{mode}] segment {np.median(tseg):.1f} us, candidates (encode+stage1) {np.median(ts):.1f} us; steps {G}")
    for a_, b_ in zip(order[:-1], order[1:]):
        d = (t[:, b_] - t[:, a_]) / 1e3
        d = d[np.abs(d) < 1e6]
        print(f"   {names[a_]:>10s} -> {names[b_]:<10s} median {np.median(d):6.2f}  max {d.max():6.2f}  last-CTA {d[-1]:6.2f} us")
    cnt = (t[:, 6] - t0) / 1e3
    print("   counted at (us from kernel start), every 17th step:", cnt[::17].round(2).tolist(), "last", round(cnt[-1], 2))
    pre = (t[:, 8] - t0) / 1e3
    valid = np.abs(pre) < 1e6
    cm = np.maximum.accumulate(np.concatenate([[0.0], cnt[:-1]]))      # latest predecessor publish
    lag = (pre - np.maximum(cm, cnt))[valid]
    print("   top counted:", sorted(zip(cnt.round(2).tolist(), range(G)))[-5:])
    for c in [int(x) for x in np.argsort(cnt)[-4:]] + [G - 1]:
        ph = [(names[b_], round((t[c, b_] - t[c, a_]) / 1e3, 2)) for a_, b_ in zip(order[:6], order[1:7])]
        print(f"   step {c} counted {cnt[c]:.2f}:", ph)
    pl = (t[:, 15] - t[:, 6]) / 1e3
    print(f"   counted -> polled (lane 0): median {np.median(pl[valid]):.2f} max {pl[valid].max():.2f}; last CTA {pl[-1]:.2f}; "
          f"last CTA polled at {(t[-1, 15] - t0) / 1e3:.2f}, prefixed at {(t[-1, 8] - t0) / 1e3:.2f}")
    tk = np.zeros(2048 * 32, np.int64)
    L.lib.memshare_debug_stage1_tok.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.lib.memshare_debug_stage1_tok(tk.ctypes.data, tk.size)
    tk = tk.reshape(2048, 32)[:G]
    for c in (G - 1, G // 2):
        row = tk[c][tk[c] > 0]
        if row.size:
            qs = row & 0xFFF
            tm = ((row >> 12) - (t0 & 0xFFFFFFFFFF)) / 1e3
            j = int(np.argmax(tm))
            q = int(qs[j])
            print(f"   CTA {c}: last waited-for step {q} seen at {tm[j]:.2f} us; that step counted at {cnt[q]:.2f}, "
                  f"prefixed at {(t[q, 8] - t0) / 1e3:.2f}; waits: {sorted(zip(tm.round(2).tolist(), qs.tolist()))[-4:]}")
    print(f"   prefix lag after the later of (own count, last predecessor count): median {np.median(lag):.2f} max {lag.max():.2f} us")
    print(f"   start offsets: median {np.median(t[:, 0] - t0) / 1e3:.2f} max {(t[:, 0] - t0).max() / 1e3:.2f}; "
          f"end max {(t[:, 7] - t0).max() / 1e3:.2f} us (last CTA {(t[-1, 7] - t0) / 1e3:.2f})")
