#!/usr/bin/env python
"""Tuning probe (not a test): device timeline of one graph-replayed round (bench.py's c2 step, and
an online LAST round) from the -DMS_TIMELINE variant library:

  MEMSHARE_LIB=$PWD/paper_2507_21433_b200/libmemshare_tl.so python scripts/probe_timeline.py

Per kernel: first CTA resident, first CTA past griddepcontrol.wait, last CTA done (us from the
round's first kernel)."""
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

NAMES = {0: "flag_reset", 1: "seg", 2: "encode", 3: "stage1", 4: "fill", 5: "ticket_reset", 6: "distance_st",
         7: "finalize", 8: "remap", 9: "chain_link"}
TUS = ("segment", "candidates", "distance", "remap")


def read(reset):
    out = np.zeros((16, 4), np.uint64)
    for tu in TUS:
        f = getattr(L.lib, f"memshare_debug_tl_{tu}")
        f.argtypes = [ctypes.c_void_p, ctypes.c_int]
        buf = np.zeros((16, 4), np.uint64)
        f(buf.ctypes.data, int(reset))
        m = buf[:, 2] > 0
        out[m] = buf[m]
    return out


def show(title, tl, reps):
    act = [i for i in range(16) if tl[i, 2] > 0]
    t0 = min(int(tl[i, 0]) for i in act)
    print(title)
    for i in act:
        s, w, e = (int(tl[i, j]) - t0 for j in range(3))
        print(f"  {NAMES.get(i, i):13s} resident {s / 1e3:8.2f}  past-wait {w / 1e3:8.2f}  done {e / 1e3:8.2f}  "
              f"(run {(e - w) / 1e3:7.2f} us)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--fused", action="store_true", help="a5-a7 as memshare_block_distance_remap")
    args = ap.parse_args()
    if args.fused:
        os.environ["MEMSHARE_BENCH_FUSED"] = "1"
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    ns = argparse.Namespace(collective="nccl", no_graph=False, steps=1, warmup=3)
    w = bench.single_workload("c2", args.seed)
    r = bench.Run(w, dev, ns)
    r.prepare()
    for _ in range(5):
        r.full()
    torch.cuda.synchronize()
    read(True)
    r.full()
    torch.cuda.synchronize()
    show("offline c2 step (one graph)", read(True), 1)
    p = r.path

    def online():
        r.restore()
        p.segment()
        p.candidates(w.tau_s, cur_mode=L.CUR_LAST)
        r.distance()
        r.remap_phase()
    online()
    torch.cuda.synchronize()
    g = p.capture(online)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    read(True)
    g.replay()
    torch.cuda.synchronize()
    show("online LAST round (one graph)", read(True), 1)

    # the busiest online round: each sequence's step with the most Stage-1 survivors (cur_mode RANGE)
    mt = p.read_candidates()["matches"]
    r.restore()
    p.segment()
    p.candidates(w.tau_s)
    torch.cuda.synchronize()
    mt = p.read_candidates()["matches"]
    busiest = np.zeros(w.batch.num_seqs, np.int32)
    for sq in range(w.batch.num_seqs):
        st = mt["step"][mt["seq"] == sq]
        if st.size:
            busiest[sq] = np.bincount(st).argmax()
    bb = torch.as_tensor(busiest, device=dev)
    be = bb + 1

    def busy():
        r.restore()
        p.segment()
        p.candidates(w.tau_s, cur_mode=L.CUR_RANGE, cur_begin=bb, cur_end=be)
        r.distance()
        r.remap_phase()
    busy()
    torch.cuda.synchronize()
    gb = p.capture(busy)
    for _ in range(5):
        gb.replay()
    torch.cuda.synchronize()
    read(True)
    gb.replay()
    torch.cuda.synchronize()
    show(f"busiest online round (RANGE, {int(p.num_pairs.item())} pairs, one graph)", read(True), 1)


if __name__ == "__main__":
    main()
