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
phases = {"segment": path.segment, "candidates_last": lambda: path.candidates(w.tau_s, cur_mode=L.CUR_LAST),
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
