#!/usr/bin/env python
"""Tuning probe (not part of the product): is the c3 distance call power-capped when it runs back
to back? Builds rank 0's wave 0 of bench.py's c3 plan (as scripts/ncu_capture.py does) and times
the a5-a6 call (memshare_block_distance) with CUDA events
  * back to back (as the bench's timed loop runs it), and
  * with an idle gap of --gap-ms after each call (the GPU cools between calls, like an ncu replay),
sampling board power and the throttle reasons with NVML during each phase. Prints one JSON line.

  python scripts/probe_power.py [--config c3] [--calls 20] [--gap-ms 50]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class Power:
    def __init__(self, idx=0):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        self.samples, self.reasons, self.stop_ = [], 0, False
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()

    def run(self):
        while not self.stop_:
            try:
                self.samples.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.005)

    def stop(self):
        self.stop_ = True
        self.t.join()
        s = sorted(self.samples)
        return {"power_w_median": s[len(s) // 2] if s else None, "power_w_max": s[-1] if s else None,
                "sw_power_cap": bool(self.reasons & 0x4), "reasons_mask": self.reasons, "samples": len(s)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--gap-ms", type=float, default=50.0)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from synth import workloads
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    ns = argparse.Namespace(collective="nccl", no_graph=True, steps=1, warmup=3)
    n = workloads.BATCHES[args.config][1]
    bins, _, _ = bench.plan_waves(args.config, n, 1, 0, dev)
    w = workloads.batch(args.config, bins[0], 0)
    r = bench.Run(w, dev, ns)
    r.path.segment()
    r.path.candidates(w.tau_s)
    for _ in range(3):
        r.path.distance_call(w.tau_b)
    torch.cuda.synchronize()
    alg, U, kvb = r.alg_bytes()
    peak = bench.measured_peaks()[0]

    def phase(gap_ms):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.calls)]
        pw = Power()
        for a, b in ev:
            a.record()
            r.path.distance_call(w.tau_b)
            b.record()
            if gap_ms > 0:
                torch.cuda.synchronize()
                time.sleep(gap_ms / 1e3)
        torch.cuda.synchronize()
        p = pw.stop()
        ms = np.array([a.elapsed_time(b) for a, b in ev])
        return {"ms_median": float(np.median(ms)), "ms_min": float(ms.min()),
                "frac_median": alg / (np.median(ms) / 1e3) / 1e9 / peak, **p}

    out = {"config": args.config, "wave": 0, "algorithmic_bytes": alg, "distinct_blocks": U,
           "back_to_back": phase(0.0), f"gap_{args.gap_ms:g}ms": phase(args.gap_ms)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
