#!/usr/bin/env python
"""Evidence helper (not a test): one memshare_block_distance call on exactly the workload bench.py
times, for an ncu capture of its streaming kernel.

  ncu --set full -k regex:distance_st_kernel -s 1 -c 1 -o out python scripts/ncu_capture.py --config c3 --wave 0

builds rank 0's wave `--wave` of bench.py's plan (LPT partition of the batch; --config c2: the
single CoT), warms up (the first distance call, skipped with -s 1) and runs one more call.
`--summarize out.ncu-rep [...] --key K` instead writes profiles/ncu_distance_<config>.json from
captures: DRAM bytes per launch and per step (sum over the waves), L2 -> SM bytes, time."""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def capture(args):
    import torch

    import bench
    from synth import workloads
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    ns = argparse.Namespace(collective="nccl", no_graph=True, steps=1, warmup=3)
    if args.config in bench.BATCH_CONFIGS:
        n = args.batch_seqs or workloads.BATCHES[args.config][1]
        bins, W, _ = bench.plan_waves(args.config, n, args.gpus, 0, dev)
        w = workloads.batch(args.config, bins[args.wave], 0)
    else:
        w = bench.single_workload(args.config, 0)
    r = bench.Run(w, dev, ns)
    r.path.segment()
    r.path.candidates(w.tau_s)
    r.path.distance_call(w.tau_b)          # skipped by ncu -s 1
    torch.cuda.synchronize()
    r.path.distance_call(w.tau_b)          # the captured launch
    torch.cuda.synchronize()
    alg, U, kvb = r.alg_bytes()
    print(json.dumps({"config": args.config, "wave": args.wave, "pairs": r.counts["pairs"], "distinct_blocks": U,
                      "algorithmic_bytes": alg}))


def summarize(args):
    out = {"config": args.config, "key": args.key, "kernel": None, "launches": [], "source": args.source}
    for rep in args.summarize:
        txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                                       "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                                       "l1tex__m_xbar2l1tex_read_bytes.sum"]).decode()
        rows = list(csv.reader(io.StringIO(txt)))
        hdr, units, vals = rows[0], rows[1], rows[2]
        get = lambda m: float(vals[hdr.index(m)].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-3, "ns": 1e-3, "us": 1, "ms": 1e3,
                 "usecond": 1, "msecond": 1e3}
        unit = lambda m: scale[units[hdr.index(m)]]
        out["kernel"] = vals[hdr.index("Kernel Name")]
        out["launches"].append({"report": os.path.basename(rep),
                                "dram_read_bytes": get("dram__bytes_read.sum") * unit("dram__bytes_read.sum"),
                                "dram_write_bytes": get("dram__bytes_write.sum") * unit("dram__bytes_write.sum"),
                                "l2_to_sm_bytes": get("l1tex__m_xbar2l1tex_read_bytes.sum")
                                * unit("l1tex__m_xbar2l1tex_read_bytes.sum"),
                                "gpu_time_us_cold": get("gpu__time_duration.sum") * unit("gpu__time_duration.sum")})
    tot = sum(x["dram_read_bytes"] + x["dram_write_bytes"] for x in out["launches"])
    out["dram_bytes_per_step"] = tot
    out["dram_bytes_per_launch"] = tot / len(out["launches"])
    json.dump(out, open(os.path.join(ROOT, "profiles", f"ncu_distance_{args.config}.json"), "w"), indent=1)
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--wave", type=int, default=0)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--batch-seqs", type=int, default=0)
    ap.add_argument("--summarize", nargs="*")
    ap.add_argument("--key", default="")
    ap.add_argument("--source", default="")
    args = ap.parse_args()
    summarize(args) if args.summarize else capture(args)


if __name__ == "__main__":
    main()
