"""Tuning probe (not part of the product): kernel list of one online round (cur_mode LAST / RANGE)
on the c2 workload. Run under ncu --metrics gpu__time_duration.sum for per-kernel times, or
plain for graph-replay latency of each phase."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_21433_b200 import _lib as L  # noqa: E402
from paper_2507_21433_b200.pipeline import MemSharePath  # noqa: E402
from synth import workloads  # noqa: E402

dev = torch.device("cuda", 0)
w = workloads.c2()
sh = w.shape
k, v, ls, bs = w.device_pool(dev)
b = w.batch
path = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                    w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                    sh.head_dim, sh.block_size, device=dev)
path.autosize(w.tau_s)
torch.cuda.synchronize()
mode = sys.argv[1] if len(sys.argv) > 1 else "time"
offline = "offline" in sys.argv
cm = L.CUR_ALL if offline else L.CUR_LAST
pristine = path.state.clone()
phases = {"restore": lambda: path.state.copy_(pristine, non_blocking=True), "segment": path.segment,
          "candidates": lambda: path.candidates(w.tau_s, cur_mode=cm),
          "distance": lambda: path.distance_call(w.tau_b), "remap": path.remap}
if mode == "ncu":
    for _ in range(3):
        for f in phases.values():
            f()
    torch.cuda.synchronize()
else:
    for name, f in phases.items():
        f()
        torch.cuda.synchronize()
        g = path.capture(f)
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(500):
            g.replay()
        e.record()
        torch.cuda.synchronize()
        print(f"{name:18s} {a.elapsed_time(e) / 500 * 1e3:7.1f} us / graph replay")
    def allp():
        for f in phases.values():
            f()
    g = path.capture(allp)
    for _ in range(20):
        g.replay()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(500):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    print(f"{'all':18s} {a.elapsed_time(e) / 500 * 1e3:7.1f} us / graph replay")

if mode == "stamps":
    # MEMSHARE_DEBUG_SKIP=8: phase stamps of stage1 in CUR_LAST mode (globaltimer ns)
    import ctypes
    for _ in range(50):
        path.segment()
        path.candidates(w.tau_s, cur_mode=L.CUR_LAST)
    torch.cuda.synchronize()
    buf = np.zeros(2048 * 16, np.uint64)
    L.lib.memshare_debug_stage1_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.lib.memshare_debug_stage1_times(buf.ctypes.data, buf.size)
    t = buf.reshape(2048, 16).astype(np.int64)[:148]
    t0 = t[:, 0][t[:, 0] > 0].min()
    G = int(path.seq_step_off[-1].item())
    act = (G - 1) % 148
    print("G", G, "active CTA", act)
    print("active CTA stamps (us):", [(round((x - t0) / 1e3, 2) if x > 0 else None) for x in t[act, :12]])
    print("CTA start spread (us):", (t[:, 0].max() - t0) / 1e3, " pre-last max:", (t[:, 7].max() - t0) / 1e3)
    lastc = np.argmax(t[:, 8])
    print("last CTA", lastc, "elected", (t[lastc, 8] - t0) / 1e3, "scans done", (t[lastc, 9] - t0) / 1e3)
