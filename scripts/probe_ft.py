#!/usr/bin/env python
"""Tuning probe (not a test): per-CTA timing of the fused a5-a7 tail (-DMS_FT_PROF variant):

  MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_ftprof.so python scripts/probe_ft.py [--seed S]

Per CTA: producer done, consumers done, finaliser done (us from the first CTA start), the number
of targets it finalised, the finaliser's batches and its time inside warp_finalize."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2507_21433_b200 import _lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seed", type=int, default=0)
ap.add_argument("--config", default="c2")
args = ap.parse_args()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
ns = argparse.Namespace(collective="nccl", no_graph=False, steps=1, warmup=3)
w = bench.single_workload(args.config, args.seed)
r = bench.Run(w, dev, ns)
r.prepare()
for _ in range(5):
    r.full()
torch.cuda.synchronize()
r.full()
torch.cuda.synchronize()
f = L.lib.memshare_debug_ft_prof
f.argtypes = [ctypes.c_void_p]
buf = np.zeros((1024, 8), np.uint64)
assert f(buf.ctypes.data) == 0
n = 148
b = buf[:n].astype(np.int64)
t0 = b[:, 0].min()
us = lambda c: (b[:, c] - t0) / 1e3
print("pairs", r.counts["pairs"], "targets", r.counts["targets"])
for name, c in (("producer done", 1), ("consumers done", 2), ("finaliser done", 3)):
    v = us(c)
    print(f"{name:15s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f} us")
print("finalisations per CTA: max", b[:, 4].max(), "hist", np.bincount(b[:, 4]).tolist())
print("batches per CTA: median", np.median(b[:, 5]), "max", b[:, 5].max())
tf = b[:, 7] / 1e3
print("time in warp_finalize per CTA: max %.2f us, mean per finalisation %.2f us" %
      (tf.max(), tf.sum() / max(1, b[:, 4].sum())))
first = us(6)[b[:, 4] > 0]
print("first finalisation: min %.2f med %.2f" % (first.min(), np.median(first)))
late = np.argsort(us(3))[-5:]
for c in late:
    print(f"  CTA {c}: producer {us(1)[c]:.2f} consumers {us(2)[c]:.2f} finaliser {us(3)[c]:.2f} nfin {b[c, 4]}")
