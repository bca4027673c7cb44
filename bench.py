#!/usr/bin/env python
"""Benchmark of the MemShare KV-block reuse path on B200 (BASELINE.json metric:
"candidate KV-block pairs scored/s and HBM GB/s (% of peak) at 1/2/4/8 B200").

One STEP = one full pass of the hot path (a1 segment -> a2-a4 Stage 1 + pairs -> a5-a6 block
distance + selection -> a7 remap) over the WHOLE batch of the configuration; the block table,
refcounts and free list are restored from a pristine device copy before every step, so every
step does identical work. Inputs are resident in HBM when the timed region starts; every KV pool
is far larger than the 126 MB L2 (no flush needed).

Default workload: configs[2] "c3" = QwQ-32B KV shape, a batch of 64 synthetic 12,288-token CoTs,
STRONG scaling over N GPUs (offline batch inference, all problems submitted at
once). The batch is partitioned by sequence -- no data-path collective: before
the timed region every rank runs a1-a4 over all 64 traces (no KV needed) to get each sequence's
Stage-1 pair count, and the sequences go to N x W bins by longest-processing-time on those
counts (`sharding.lpt_assign`); rank r owns bins r*W .. r*W+W-1 as W WAVES, W = the fewest waves
whose KV pools fit one GPU (N = 1: two waves of ~32 sequences, 103 GB each; N >= 2: one). A wave
is built (trace, paged table, KV pool generated on the device), warmed up and timed for K steps;
the rank's step time is the sum of its waves' step times, the job's the max over ranks.
Each wave also checks a parity sample against the CPU oracle (a1-a4 and the remap bit-exact,
sampled targets' distances within 1e-5 and decisions by the tie / threshold rules); a failure
prints the JSON line and exits 1.

Other workloads: --config c2 (configs[1], one 12,406-token CoT per GPU, weak scaling: every rank
runs the same sequence), c4 (configs[3], 128 Phi-4 AIME-length traces), c5 (configs[4], 512 x
16,384-token CoTs), tiny.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "candidate KV-block pairs scored/s"
UNIT = "pairs/s"
BATCH_CONFIGS = ("c3", "c4", "c5")
POOL_BUDGET = 140e9          # KV bytes one wave may take on a 180 GB B200 (the rest: workspaces, CUDA)


def gpu_launches_per_step(num_tokens, sms=148, fused_tail=False):
    """Our kernels per round: flag reset, seg, encode, stage1, (fill), ticket reset, distance,
    finalize, remap (inside finalize's last CTA when a5-a7 is the fused
    memshare_block_distance_remap call). The library fuses the fill into stage1 for an offline
    round over at most 100 x 8 x SMs tokens (one CoT-sized batch); MEMSHARE_FUSED_FILL=0 disables
    it."""
    fused = num_tokens <= 100 * 8 * sms and os.environ.get("MEMSHARE_FUSED_FILL", "1") != "0"
    return (7 if fused_tail else 8) + (0 if fused else 1)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0, help="timed steps (0 = config default: c2 300, batches 10)")
    ap.add_argument("--warmup", type=int, default=0, help="warm-up steps (0 = config default, >= 3)")
    ap.add_argument("--config", default="c3", choices=["c3", "c2", "c4", "c5", "tiny"])
    ap.add_argument("--batch-seqs", type=int, default=0, help="c3/c4/c5: use the first n sequences of the batch")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="seq", choices=["seq", "headshard"])
    ap.add_argument("--collective", default="p2p", choices=["p2p", "nccl"],
                    help="headshard, N>1: 'p2p' = FINALIZE reads every rank's partial sums over NVLink from "
                         "symmetric memory (memshare_block_distance_finalize_peers); 'nccl' = all-reduce + FINALIZE")
    ap.add_argument("--seed", type=int, default=int(os.environ.get("MEMSHARE_SEED", "0")))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-online", action="store_true")
    ap.add_argument("--seed-sweep", default="0,1,2,3,4",
                    help="c2: also time these seeds' pair lists (the paper's 5 runs) and report mean / min / max "
                         "beside the --seed line ('' = off)")
    ap.add_argument("--breakdown", action="store_true", help="also time each ABI call separately (stderr)")
    ap.add_argument("--no-graph", action="store_true", help="launch the calls directly instead of CUDA-graph replay")
    a = ap.parse_args()
    batch = a.config in BATCH_CONFIGS
    if a.steps <= 0:
        a.steps = 10 if batch else 300
    if a.warmup <= 0:
        a.warmup = 3 if batch else 20
    a.warmup = max(3, a.warmup)
    return a


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def single_workload(cfg, seed):
    from synth import workloads
    if cfg == "c2":
        # weak scaling: every rank runs configs[1] itself (identical per-GPU work); other seeds give
        # 192-622 pairs, which would make the max-over-ranks time measure seed variance, not scaling
        return workloads.c2(seed=seed)
    return workloads.tiny(eta=0.05)


def describe(cfg, w, world, mode, extra=None):
    sh = w.shape
    text = {"c2": "configs[1]: DeepSeek-R1-Distill-Qwen-32B KV shape, 1 x 12,406-token synthetic CoT per GPU "
                  "(128-token prompt, MATH-500-like planted redundancy; every rank runs the same sequence: "
                  "identical per-GPU work)",
            "tiny": "configs[0]: tiny T0 fixture",
            "c3": "configs[2]: QwQ-32B KV shape, batch of 12,288-token synthetic CoTs (MATH-500-like planted "
                  "redundancy), partitioned over the GPUs by sequence (LPT on Stage-1 pair counts), waves of "
                  "<= 140 GB of KV per GPU",
            "c4": "configs[3]: Phi-4-reasoning-plus KV shape, batch of AIME-length synthetic traces "
                  "(L ~ U[8192, 16620]), partitioned over the GPUs by sequence (LPT), waves",
            "c5": "configs[4]: 32B KV shape, batch of 16,384-token synthetic CoTs, partitioned over the GPUs by "
                  "sequence (LPT), waves"}[cfg]
    d = {"workload": text,
         "kv_shape": {"layers": sh.num_layers, "kv_heads": sh.num_kv_heads, "head_dim": sh.head_dim,
                      "block_size": sh.block_size, "kv_dtype": "bf16"},
         "tau_s": w.tau_s, "tau_b": round(w.tau_b, 6), "eta": w.eta, "pairing": "aligned",
         "stage1": "offline (every step current)",
         "parallelism": (f"seq-shard dp{world}" if mode == "seq" else f"kv-head-shard hs{world}"),
         "l2": "inputs larger than L2 (pool %.2f GB per wave vs 126 MB L2); no flush" % (w.pool_bytes() / 1e9)}
    if extra:
        d.update(extra)
    return d


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100",
                                       "-i", str(gpu_index)], stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        self.windows = []
        self.t0 = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.windows.append((self.t0, time.time()))

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = time.mktime(time.strptime(parts[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                rows.append((ts, float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        os.unlink(self.f.name)
        inwin = [r for r in rows if any(t0 - 1 <= r[0] <= t1 + 1 for t0, t1 in self.windows)] or rows
        if not inwin:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inwin for i, x in enumerate(r[3]) if x.lower() == "active"})
        return {"sm_mhz": float(np.median([r[1] for r in inwin])), "sm_max_mhz": max(r[2] for r in inwin),
                "reasons": reasons, "samples": len(inwin)}


# ----------------------------------------------------------------------------- oracle (CPU baselines)
def oracle_pass(w, k_pool, v_pool, max_pairs=600, budget_s=20.0):
    """The oracle as it stands on the host: a1-a4 in full, then a5-a6 on whole target groups in
    order (at most `max_pairs` pairs / `budget_s` seconds), then a7 on those decisions. Only the KV
    blocks those pairs touch are copied from the device pool to the host (not timed)."""
    import torch

    import oracle
    b, sh = w.batch, w.shape
    t0 = time.perf_counter()
    st = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    oc = oracle.step_candidates(b.tokens, b.seq_tok_off, st, b.delim_ids, w.table, sh.block_size, w.tau_s)
    t1 = time.perf_counter()
    pr, toff = oc["pairs"], oc["target_off"]
    T = int(np.searchsorted(toff, max_pairs, side="right") - 1) if toff[-1] > max_pairs else toff.size - 1
    T = max(T, min(1, toff.size - 1))
    P = int(toff[T])
    blocks = np.unique(np.concatenate([pr["target_phys"][:P], pr["source_phys"][:P]]))
    slice_e = sh.block_size * sh.num_kv_heads * sh.head_dim
    idx = torch.as_tensor(blocks, device=k_pool.device, dtype=torch.long)
    kh = k_pool.view(sh.num_layers, w.num_blocks, slice_e).index_select(1, idx).view(torch.int16).cpu().numpy()
    vh = v_pool.view(sh.num_layers, w.num_blocks, slice_e).index_select(1, idx).view(torch.int16).cpu().numpy()
    kh, vh = kh.view(np.uint16).ravel(), vh.view(np.uint16).ravel()
    pos = {int(x): i for i, x in enumerate(blocks)}
    tp = np.array([pos[int(x)] for x in pr["target_phys"][:P]], np.int32)
    sp = np.array([pos[int(x)] for x in pr["source_phys"][:P]], np.int32)
    ls, bs = blocks.size * slice_e, slice_e
    t1b = time.perf_counter()
    D_parts, t, ts = [], 0, time.perf_counter()
    while t < T and time.perf_counter() - ts < budget_s:
        t_end = min(T, t + 16)
        p0, p1 = toff[t], toff[t_end]
        D_parts.append(oracle.block_distance(kh, vh, ls, bs, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                                             sh.head_dim, sh.block_size, tp[p0:p1], sp[p0:p1]))
        t = t_end
    P = int(toff[t])
    D = np.concatenate(D_parts) if D_parts else np.zeros(0)
    best, acc, _ = oracle.select(D, toff[:t + 1], pr["source_logical"][:P], w.tau_b)
    dec = oracle.decisions({k: v[:P] for k, v in pr.items()}, toff[:t + 1], D, best, acc)
    t2 = time.perf_counter()
    oracle.remap(w.table, w.refcount, w.free_list, w.free_count, dec, sh.block_size)
    t3 = time.perf_counter()
    t_cpu = (t1 - t0) + (t3 - t1b)                       # the block copy from the GPU is not oracle work
    return {"pairs": P, "targets": t, "all_pairs": int(pr["seq"].size), "t_front": t1 - t0, "t_stage2": t2 - t1b,
            "t_remap": t3 - t2, "t_total": t_cpu}


def oracle_job(job):
    """One host process of the all-cores CPU baseline: the oracle on ONE sequence (a1-a4 in full,
    a5-a6 on its first whole target groups up to `max_pairs` pairs, a7), its KV blocks generated on
    the host by the generator twin into a compact pool (not timed). Returns (pairs, seconds)."""
    cfg, seq_index, seed, max_pairs = job
    sys.path.insert(0, ROOT)
    import oracle
    from synth import kv, workloads
    w = workloads.c2(seed=seed) if cfg == "c2" else workloads.batch(cfg, [seq_index], seed)
    b, sh = w.batch, w.shape
    t0 = time.perf_counter()
    st = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    oc = oracle.step_candidates(b.tokens, b.seq_tok_off, st, b.delim_ids, w.table, sh.block_size, w.tau_s)
    t_front = time.perf_counter() - t0
    pr, toff = oc["pairs"], oc["target_off"]
    if toff.size < 2:
        return 0, t_front
    T = int(np.searchsorted(toff, max_pairs, side="right") - 1) if toff[-1] > max_pairs else toff.size - 1
    T = max(T, 1)
    P = int(toff[T])
    blocks = np.unique(np.concatenate([pr["target_phys"][:P], pr["source_phys"][:P]]))
    pos = {int(x): i for i, x in enumerate(blocks)}
    s_, l_, p_ = w.blocks()
    sel = np.isin(p_, blocks)
    k, v, ls, bs = kv.host_pool(sh, blocks.size)
    kv.fill_blocks_host(k, v, ls, bs, sh, b.tokens, b.seq_tok_off, s_[sel], l_[sel],
                        np.array([pos[int(x)] for x in p_[sel]], np.int32), w.seed, w.eta)
    tp = np.array([pos[int(x)] for x in pr["target_phys"][:P]], np.int32)
    sp = np.array([pos[int(x)] for x in pr["source_phys"][:P]], np.int32)
    t1 = time.perf_counter()
    D = oracle.block_distance(k, v, ls, bs, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads, sh.head_dim,
                              sh.block_size, tp, sp)
    best, acc, _ = oracle.select(D, toff[:T + 1], pr["source_logical"][:P], w.tau_b)
    dec = oracle.decisions({k_: v_[:P] for k_, v_ in pr.items()}, toff[:T + 1], D, best, acc)
    oracle.remap(w.table, w.refcount, w.free_list, w.free_count, dec, sh.block_size)
    return P, t_front + (time.perf_counter() - t1)


def all_cores_baseline(cfg, seed, seq_indices, max_pairs=128):
    """The oracle on every host core at once (one process per core, disjoint sequences,
    BASELINE.md §4): aggregate pairs / the slowest process's time."""
    import multiprocessing as mp
    n = os.cpu_count() or 1
    jobs = [(cfg, seq_indices[i % len(seq_indices)], seed + (i // len(seq_indices) if cfg == "c2" else 0), max_pairs)
            for i in range(n)]
    with mp.get_context("spawn").Pool(n) as pool:
        res = pool.map(oracle_job, jobs)
    pairs = sum(r[0] for r in res)
    worst = max(r[1] for r in res)
    return {"value": pairs / worst if worst > 0 else None, "unit": UNIT, "cores": n, "kind": "oracle",
            "sample": (f"{n} oracle processes (fp64, one per host core) on {n} different sequences of the {cfg} "
                       f"workload: a1-a4 in full, a5-a7 on up to {max_pairs} pairs each; {pairs} pairs in "
                       f"{worst:.2f} s (slowest process)"), "cpu": host_cpu_model()}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm), as it stands, on host cores."""
    if rank != 0:
        return
    import oracle
    from synth import workloads
    oracle.build()
    if args.config in BATCH_CONFIGS:
        w = workloads.batch(args.config, [0], args.seed)        # a bounded sample: the batch's sequence 0
    else:
        w = single_workload(args.config, args.seed)
    k, v, ls, bs = w.host_pool()
    sh = w.shape
    st = oracle.segment_steps(w.batch.tokens, w.batch.seq_tok_off, w.batch.gen_start, w.batch.final, w.batch.delim_ids)
    oc = oracle.step_candidates(w.batch.tokens, w.batch.seq_tok_off, st, w.batch.delim_ids, w.table, sh.block_size,
                                w.tau_s)
    pr, toff = oc["pairs"], oc["target_off"]
    T = toff.size - 1
    # calibrate: seconds per target group (a5-a6 on all pairs of a target)
    t0 = time.perf_counter()
    oracle.block_distance(k, v, ls, bs, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads, sh.head_dim,
                          sh.block_size, pr["target_phys"][:4], pr["source_phys"][:4])
    per_pair = (time.perf_counter() - t0) / 4
    budget = 150.0 / max(1, args.steps + args.warmup)
    n_t = max(1, min(T, int(budget / (per_pair * max(1.0, pr["seq"].size / max(T, 1))))))
    cursor = 0
    times, pairs_done = [], []
    for it in range(args.warmup + args.steps):
        ts = [(cursor + i) % T for i in range(n_t)]
        cursor = (cursor + n_t) % T
        sel = np.concatenate([np.arange(toff[t], toff[t + 1]) for t in ts])
        sub_off = np.concatenate([[0], np.cumsum([toff[t + 1] - toff[t] for t in ts])])
        t0 = time.perf_counter()
        D = oracle.block_distance(k, v, ls, bs, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads, sh.head_dim,
                                  sh.block_size, pr["target_phys"][sel], pr["source_phys"][sel])
        oracle.select(D, sub_off, pr["source_logical"][sel], w.tau_b)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
            pairs_done.append(sel.size)
    total_t = float(np.sum(times))
    value = float(np.sum(pairs_done)) / total_t
    sample = (f"a5-a6 (oracle_block_distance + oracle_select, fp64, 1 thread) on {n_t} target group(s) "
              f"(~{np.mean(pairs_done):.1f} pairs) per step, rotating over the {pr['seq'].size} pairs of "
              f"{'sequence 0 of the ' if args.config in BATCH_CONFIGS else 'the '}{args.config} workload; "
              f"a1-a4/a7 excluded from the steps")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / max(1, args.steps),
            "higher_is_better": True, "scaling": "strong" if args.config in BATCH_CONFIGS else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": describe(args.config, w, 1, "seq"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": host_cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- one device-resident workload
class Run:
    """One workload resident on this GPU: the path, its CUDA graphs and the measurements of a
    round (a1-a7) over it. `mode` headshard: this rank holds a slice of the KV heads."""

    def __init__(self, w, dev, args, world=1, rank=0, mode="seq", dist=None):
        import torch

        from paper_2507_21433_b200 import _lib as L
        from paper_2507_21433_b200.pipeline import MemSharePath
        self.torch, self.L, self.w, self.dev, self.args, self.dist = torch, L, w, dev, args, dist
        sh = w.shape
        self.h_local, h_off = sh.num_kv_heads, 0
        if mode == "headshard":
            from paper_2507_21433_b200.sharding import head_shard
            self.h_local, h_off = head_shard(sh.num_kv_heads, world, rank)
        k, v, ls, bs = w.device_pool(dev, h_local=self.h_local, head_offset=h_off)
        b = w.batch
        self.path = p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount,
                                     w.free_list, w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers,
                                     self.h_local, sh.num_kv_heads, sh.head_dim, sh.block_size, device=dev)
        self.counts = p.autosize(w.tau_s)
        self.mode = mode
        self.collective = "none" if world == 1 or mode != "headshard" else args.collective
        self.symm = self.peer_ptrs = None
        if mode == "headshard":
            p.alloc_partial()
        if self.collective == "p2p":
            try:
                import torch.distributed._symmetric_memory as symm
                buf = symm.empty(p.partial_sq.numel(), dtype=torch.float32, device=dev)
                self.symm = symm.rendezvous(buf, dist.group.WORLD.group_name)
                p.partial_sq = buf                      # PARTIAL writes into this rank's symmetric buffer
                self.peer_ptrs = torch.tensor(list(self.symm.buffer_ptrs), dtype=torch.int64, device=dev)
            except Exception as e:                      # no symmetric memory on this node: NCCL all-reduce
                print(f"bench: symmetric memory unavailable ({e!r}); using the NCCL all-reduce", file=sys.stderr)
                self.collective = "nccl"
        self.world = world
        # a5-a6 then a7 as separate calls (the roofline times the a5-a6 call alone);
        # MEMSHARE_BENCH_FUSED=1 times memshare_block_distance_remap (a5-a7 in one call: the remap in
        # the finalisation kernel's last CTA; same offline step, busiest online round -1.5 us)
        self.fused = mode != "headshard" and os.environ.get("MEMSHARE_BENCH_FUSED", "0") == "1"
        torch.cuda.synchronize()
        self.pristine = p.state.clone()
        self.stream = torch.cuda.current_stream(dev)

    def ev(self):
        return self.torch.cuda.Event(enable_timing=True)

    def restore(self):              # table + refcounts + free list + free count: one device copy
        self.path.state.copy_(self.pristine, non_blocking=True)

    def distance(self):
        """a5-a6 (a5-a7 when fused)."""
        p, L, w = self.path, self.L, self.w
        if self.fused:
            p.distance_remap(w.tau_b)
            return
        if self.mode != "headshard":
            p.distance_call(w.tau_b)
            return
        p.distance_call(w.tau_b, L.DIST_PARTIAL)
        if self.collective == "p2p":
            self.symm.barrier(channel=0)                 # every rank's partial sums are written
            p.finalize_peers(w.tau_b, self.peer_ptrs, self.world)
            self.symm.barrier(channel=1)                 # every rank has read them (buffer reusable)
        else:
            if self.collective == "nccl":
                self.dist.all_reduce(p.partial_sq[:self.counts["pairs"] * w.shape.num_layers * 2])
            p.distance_call(w.tau_b, L.DIST_FINALIZE)

    def remap_phase(self):
        """a7 (inside the a5-a7 call when fused)."""
        if not self.fused:
            self.path.remap()

    def prepare(self):
        p, w = self.path, self.w

        def front():                 # restore the round's initial state, a1, a2-a4
            self.restore()
            p.segment()
            p.candidates(w.tau_s)

        for fn in (front, self.distance, self.remap_phase):     # eager warm-up (module load, attributes)
            fn()
        self.torch.cuda.synchronize()
        if self.args.no_graph or self.collective != "none":    # collectives / symmetric-memory barriers: eager
            self.run = (front, self.distance, self.remap_phase)
            self.full = None
        else:
            # the timed step: the whole round as ONE graph (a serving loop's replay); the a5-a6 timing
            # pass replays one graph per phase with events between them (graph boundaries cost ~4 us)
            self.run = tuple(p.capture(fn).replay for fn in (front, self.distance)) + (
                (lambda: None) if self.fused else p.capture(p.remap).replay,)

            def whole():
                front()
                self.distance()
                self.remap_phase()
            self.full = p.capture(whole).replay

    def step(self, d_ev=None):
        self.run[0]()
        if d_ev is not None:
            d_ev[0].record(self.stream)
        self.run[1]()
        if d_ev is not None:
            d_ev[1].record(self.stream)
        self.run[2]()

    def alg_bytes(self):
        """Algorithmic bytes of the distance call: U distinct blocks x B_blk + pair / target
        metadata."""
        pr = self.path.read_candidates()["pairs"]
        U = int(np.unique(np.concatenate([pr["target_phys"], pr["source_phys"]])).size)
        sh = self.w.shape
        blk_b = sh.num_layers * 2 * sh.block_size * self.h_local * sh.head_dim * 2
        P, T = self.counts["pairs"], self.counts["targets"]
        return U * blk_b + P * (24 + 4 + 1) + T * (8 + 32), U, U * blk_b

    def timed(self, clocks):
        """W warm-up steps, then EXACTLY K steps (the whole round as one graph replay each) between
        a barrier + synchronize pair -> ms per step; then K more steps replayed phase by phase with
        CUDA events around the a5-a6 call on its stream -> its mean ms. Returns both."""
        torch, args = self.torch, self.args
        one = self.full if self.full is not None else self.step
        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize()
        assert self.path.read_status() == 0, f"device status {self.L.status_string(self.path.read_status())}"
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()
        clocks.mark_start()
        e0, e1 = self.ev(), self.ev()
        e0.record(self.stream)
        for i in range(args.steps):
            one()
        e1.record(self.stream)
        torch.cuda.synchronize()
        clocks.mark_end()
        if self.dist is not None:
            self.dist.barrier()
        ms = e0.elapsed_time(e1) / args.steps
        d_events = [(self.ev(), self.ev()) for _ in range(args.steps)]
        clocks.mark_start()
        for i in range(args.steps):
            self.step(d_events[i])
        torch.cuda.synchronize()
        clocks.mark_end()
        assert self.path.read_status() == 0
        return ms, float(np.mean([a.elapsed_time(b) for a, b in d_events]))

    def kernel_only(self, n):
        """The streaming kernel alone: the library's profiling hook records events around it."""
        kb, ke = self.ev(), self.ev()
        kb.record(self.stream)
        ke.record(self.stream)
        self.torch.cuda.synchronize()
        self.L.profile_distance_events(kb, ke)
        ks = []
        for i in range(n + 2):
            self.run[0]()
            self.distance()
            self.run[2]()
            self.torch.cuda.synchronize()
            if i >= 2:
                ks.append(kb.elapsed_time(ke))
        self.L.profile_distance_events(None, None)
        return float(np.mean(ks))

    def online(self):
        """PAPER.md:317 evaluates each step as it finishes: CUR_LAST = the newly finished step of
        every sequence against its history; RANGE = each sequence's busiest step (most Stage-1
        survivors in the offline pass). One graph replay of a1-a7 per round, table restored."""
        torch, L, p, w = self.torch, self.L, self.path, self.w
        mt = p.read_candidates()["matches"]
        busiest = np.zeros(w.batch.num_seqs, np.int32)
        for sq in range(w.batch.num_seqs):
            st = mt["step"][mt["seq"] == sq]
            if st.size:
                busiest[sq] = np.bincount(st).argmax()

        def replay_us(fn, n_on=200):
            fn()
            torch.cuda.synchronize()
            og = p.capture(fn)
            for _ in range(10):
                og.replay()
            torch.cuda.synchronize()
            o0, o1 = self.ev(), self.ev()
            o0.record(self.stream)
            for _ in range(n_on):
                og.replay()
            o1.record(self.stream)
            torch.cuda.synchronize()
            return 1e3 * o0.elapsed_time(o1) / n_on

        def time_round(cur_mode, cb=None, ce=None, restores=1):
            # the round a serving loop runs: a1-a4, then a5-a7 as the one fused call
            # (memshare_block_distance_remap) unless the bench's own path is head-sharded
            def online_round():
                for _ in range(restores):
                    self.restore()
                p.segment()
                p.candidates(w.tau_s, cur_mode=cur_mode, cur_begin=cb, cur_end=ce)
                if self.mode == "headshard":
                    self.distance()
                    self.remap_phase()
                else:
                    p.distance_remap(w.tau_b)
            us = replay_us(online_round)
            return us, int(p.num_pairs.item())

        last_us, last_pairs = time_round(L.CUR_LAST)
        bb = torch.as_tensor(busiest, device=self.dev)
        busy_us, busy_pairs = time_round(L.CUR_RANGE, bb, bb + 1)
        # the state reset every replayed round carries: its marginal cost inside the round's graph
        # (a round with two resets minus the round with one)
        last2_us, _ = time_round(L.CUR_LAST, restores=2)
        restore_us = max(0.0, last2_us - last_us)
        self.restore()
        torch.cuda.synchronize()
        return {"round_us": last_us - restore_us, "pairs_per_round": last_pairs,
                "busiest_round_us": busy_us - restore_us, "busiest_pairs_per_round": busy_pairs,
                "current_steps_per_round": w.batch.num_seqs, "rounds": 200,
                "raw_round_us": last_us, "raw_busiest_round_us": busy_us, "state_restore_us": restore_us,
                "note": "online (PAPER.md:317): one graph replay of a1-a4 + the fused a5-a7 call "
                        "(memshare_block_distance_remap) with one current step per sequence -- round_us: the last "
                        "finished step (cur_mode LAST); busiest_round_us: the step with the most Stage-1 "
                        "survivors (cur_mode RANGE); both net of the table/refcount/free-list restore each "
                        "replay carries (state_restore_us: its marginal cost in the graph, a round with two "
                        "restores minus one; raw_* include it)"}

    def e2e(self, n_steps):
        """The same round through the public API with HOST buffers: one pinned H2D of the round's
        inputs (MemSharePath's layout), the four calls, one D2H of counters + decisions and of the
        rewritten block table; the host reads every round's counters. Replayed as one CUDA graph
        with two rounds in flight (double-buffered pinned results). Returns (ms, h2d, d2h)."""
        torch, p, w = self.torch, self.path, self.w
        from paper_2507_21433_b200.pipeline import pack_inputs
        b = w.batch
        host_in, _ = pack_inputs(b.tokens, b.seq_tok_off, b.gen_start, b.final, w.table, w.refcount, w.free_list,
                                 w.free_count)
        h_in = torch.from_numpy(host_in).pin_memory()
        assert h_in.numel() == p.inputs.numel()
        h2d = h_in.numel() * 4
        n_head = 2 + p.table.numel()
        outs = [(torch.empty(p.outputs.numel(), dtype=torch.uint8).pin_memory(),
                 torch.empty(n_head, dtype=torch.int32).pin_memory()) for _ in range(2)]
        d2h = outs[0][0].numel() + outs[0][1].numel() * 4
        P = self.counts["pairs"]

        def round_body(j):
            def body():
                p.inputs.copy_(h_in, non_blocking=True)
                p.segment()
                p.candidates(w.tau_s)
                self.distance()
                self.remap_phase()
                outs[j][0].copy_(p.outputs, non_blocking=True)
                outs[j][1].copy_(p.state[:n_head], non_blocking=True)
            return body

        def consume(j):
            o = outs[j][0][:64].view(torch.int64)
            assert int(o[1]) == P, "e2e round result"

        if not self.args.no_graph and self.collective == "none":
            gs = []
            for j in range(2):
                round_body(j)()
                torch.cuda.synchronize()
                gs.append(p.capture(round_body(j)))
            done = [torch.cuda.Event(), torch.cuda.Event()]
            inflight = [False, False]
            cursor = [0]

            def e2e_step():
                j = cursor[0] & 1
                cursor[0] += 1
                if inflight[j]:
                    done[j].synchronize()
                    consume(j)
                gs[j].replay()
                done[j].record(torch.cuda.current_stream(self.dev))
                inflight[j] = True

            def drain():
                for j in range(2):
                    if inflight[j]:
                        done[j].synchronize()
                        consume(j)
                        inflight[j] = False
        else:
            body0 = round_body(0)

            def e2e_step():
                body0()
                torch.cuda.current_stream(self.dev).synchronize()
                consume(0)

            def drain():
                pass

        for _ in range(3):
            e2e_step()
        drain()
        if self.dist is not None:
            self.dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = self.ev(), self.ev()
        a0.record(self.stream)
        for _ in range(n_steps):
            e2e_step()
        drain()
        a1.record(self.stream)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / n_steps, int(h2d), int(d2h)

    def parity_sample(self, n_targets=8, seed=0):
        """This rank's parity sample against the CPU oracle (test infrastructure, run after the
        timed region): segmentation, Stage-1 matches and block pairs bit-exact; the distances of
        `n_targets` sampled whole targets within 1e-5 relative and their decisions by the tie /
        threshold rules; the remap bit-exact on the GPU's own decisions."""
        import torch

        import oracle
        p, w = self.path, self.w
        b, sh = w.batch, w.shape
        self.restore()
        p.round(w.tau_s, w.tau_b)
        torch.cuda.synchronize()
        out = {"ok": False, "status": p.read_status()}
        try:
            assert out["status"] == 0, "device status"
            st = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
            gs = p.read_steps()
            for k in ("step_start", "step_end", "step_nbag", "seq_step_off"):
                assert np.array_equal(np.asarray(gs[k]), np.asarray(st[k])), k
            oc = oracle.step_candidates(b.tokens, b.seq_tok_off, st, b.delim_ids, w.table, sh.block_size, w.tau_s)
            gc = p.read_candidates()
            for k in ("seq", "step", "cand_step", "rank"):
                assert np.array_equal(gc["matches"][k], oc["matches"][k]), "matches." + k
            assert np.array_equal(gc["matches"]["cosine"].view(np.uint64), oc["matches"]["cosine"].view(np.uint64))
            for k in oc["pairs"]:
                assert np.array_equal(gc["pairs"][k], oc["pairs"][k]), "pairs." + k
            toff, pr = oc["target_off"], oc["pairs"]
            gd = p.read_distance()
            T = toff.size - 1
            rng = np.random.default_rng(seed)
            tsel = np.sort(rng.choice(T, size=min(n_targets, T), replace=False)) if T else np.zeros(0, np.int64)
            psel = np.concatenate([np.arange(toff[t], toff[t + 1]) for t in tsel]) if tsel.size else np.zeros(0, int)
            if psel.size:
                blocks = np.unique(np.concatenate([pr["target_phys"][psel], pr["source_phys"][psel]]))
                slice_e = sh.block_size * self.h_local * sh.head_dim
                idx = torch.as_tensor(blocks, device=self.dev, dtype=torch.long)
                kh = p.k_pool.view(sh.num_layers, w.num_blocks, slice_e).index_select(1, idx)
                vh = p.v_pool.view(sh.num_layers, w.num_blocks, slice_e).index_select(1, idx)
                kh = kh.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).ravel()
                vh = vh.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).ravel()
                pos = {int(x): i for i, x in enumerate(blocks)}
                tp = np.array([pos[int(x)] for x in pr["target_phys"][psel]], np.int32)
                sp = np.array([pos[int(x)] for x in pr["source_phys"][psel]], np.int32)
                D = oracle.block_distance(kh, vh, blocks.size * slice_e, slice_e, sh.num_layers, self.h_local,
                                          sh.num_kv_heads, sh.head_dim, sh.block_size, tp, sp)
                g = gd["distance"][psel].astype(np.float64)
                zero = D == 0.0
                assert np.all(g[zero] == 0.0), "identical blocks must give 0"
                rel = np.abs(g[~zero] - D[~zero]) / D[~zero]
                out["max_rel_err"] = float(rel.max()) if rel.size else 0.0
                assert out["max_rel_err"] <= 1e-5, "distance rel err"
                sub_off = np.concatenate([[0], np.cumsum([toff[t + 1] - toff[t] for t in tsel])])
                best, acc, _ = oracle.select(D, sub_off, pr["source_logical"][psel], w.tau_b)
                exact = near_tie = near_thr = 0
                for j, t in enumerate(tsel):
                    p0, p1 = sub_off[j], sub_off[j + 1]
                    src = gd["decisions"]["source_logical"][t]
                    m = np.nonzero(pr["source_logical"][psel][p0:p1] == src)[0]
                    assert m.size == 1, "decision source"
                    dmin = D[p0:p1].min()
                    assert D[p0 + m[0]] <= dmin * (1 + 1e-5), "decision outside the tie set"
                    same_src = p0 + m[0] == best[j]
                    same_acc = bool(gd["decisions"]["accepted"][t]) == bool(acc[j])
                    if not same_acc:
                        assert abs(D[best[j]] - np.float32(w.tau_b)) <= 1e-4 * w.tau_b, "accept away from tau_b"
                    exact += int(same_src and same_acc)
                    near_tie += int(not same_src)
                    near_thr += int(not same_acc)
                # SURVEY.md §5 parity counts (reading R29): decisions equal to the oracle's, and those
                # allowed to differ (a near tie / a distance within 1e-4 of tau_b)
                out["decisions"] = {"exact": exact, "near_tie": near_tie, "near_threshold": near_thr}
            s = p.read_state()
            st_o, tab, rc, fl, fc, nf, af = oracle.remap(w.table, w.refcount, w.free_list, w.free_count,
                                                         gd["decisions"], sh.block_size)
            assert st_o == 0 and np.array_equal(s["table"], tab) and np.array_equal(s["refcount"], rc), "remap"
            assert np.array_equal(s["free_list"], fl) and s["free_count"] == fc and s["num_freed"] == nf, "free list"
            out.update(ok=True, pairs=int(pr["seq"].size), sampled_targets=int(tsel.size), sampled_pairs=int(psel.size))
        except AssertionError as e:
            out["error"] = str(e) or "assertion"
        self.restore()
        torch.cuda.synchronize()
        return out

    def free(self):
        self.path = None
        self.torch.cuda.synchronize()
        self.torch.cuda.empty_cache()


def init_dist(world, local):
    import torch
    import torch.distributed as dist
    # MEMSHARE_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0 over gloo, to exercise the
    # multi-rank code path (barriers, max-over-ranks timing, pair sums) on a one-GPU box
    shared_gpu = os.environ.get("MEMSHARE_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared_gpu else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        return gpu, dev, dist
    return gpu, dev, None


def reduce_max_sum(dist, dev, mx, sm):
    import torch
    t = torch.tensor([float(mx), float(sm)], dtype=torch.float64, device=dev)
    if dist is None:
        return float(t[0]), float(t[1])
    a, b = t[:1].clone(), t[1:].clone()
    dist.all_reduce(a, op=dist.ReduceOp.MAX)
    dist.all_reduce(b, op=dist.ReduceOp.SUM)
    return float(a[0]), float(b[0])


def live_copy_gbs(dev):
    """This box's copy bandwidth, measured the way MEASURED_PEAKS.json's hbm_gbs is (torch copy of
    1 Gi bf16 elements, read + write bytes, best of 10, CUDA events): context for box-to-box spread
    of the roofline fraction (the fraction itself uses the driver-measured peak)."""
    import torch
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 2 * (1 << 30) / (best / 1e3) / 1e9


# L2 -> shared-memory delivery of a TMA ring with 32 KiB copies (one per stage) from an L2-resident
# source on this pool's B200: 16.2-16.7 TB/s (scripts/tma_sweep.cu 32, lean producer; 19.4 TB/s
# with 64 KiB copies), profiles/r1_tuning_log.md "L2 -> SM delivery ceiling"
L2_DELIVERY_GBS = 16500.0


def dual_ceiling(U, T, P, kv_bytes, d_ms):
    """The distance kernel stages T + P slices per (layer, K|V) (each target once, each pair's source
    once) of which U are distinct: its time is bounded by max(distinct bytes / HBM peak, staged bytes
    / L2 delivery ceiling). Returns the staged bytes, the L2-delivery fraction and the fraction of the
    larger of the two bounds."""
    peak, _ = measured_peaks()
    per_block = kv_bytes / max(U, 1)
    staged = (T + P) * per_block
    t_hbm = kv_bytes / (peak * 1e9)
    t_l2 = staged / (L2_DELIVERY_GBS * 1e9)
    return {"staged_bytes": staged, "staged_over_distinct": (T + P) / max(U, 1),
            "l2_delivery_gbs": staged / (d_ms / 1e3) / 1e9, "l2_delivery_peak_gbs": L2_DELIVERY_GBS,
            "l2_frac": staged / (d_ms / 1e3) / 1e9 / L2_DELIVERY_GBS,
            "bound": "l2_delivery" if t_l2 > t_hbm else "hbm",
            "frac_of_bound": max(t_hbm, t_l2) / (d_ms / 1e3)}


def roofline(alg_bytes, d_ms, kernel_only_ms, kv_bytes, U, P, traffic, kernel_name, live=None, T=None):
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (d_ms / 1e3) / 1e9
    r = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
         "traffic": traffic, "kernel": kernel_name, "kernel_ms": d_ms, "algorithmic_bytes": alg_bytes,
         "pairs_per_s_a5a6": P / (d_ms / 1e3), "kv_bytes": kv_bytes, "distinct_blocks": U, "peak_source": peak_src,
         "frac_of_nominal_8000": achieved / 8000.0,
         "note": ("achieved/kernel_ms: CUDA events around the whole a5-a7 call (memshare_block_distance_remap: "
                  "ticket reset + streaming kernel + finalize with the remap in its last CTA; conservative: the "
                  "remap is inside)" if "remap" in kernel_name else
                  "achieved/kernel_ms: CUDA events around the whole a5-a6 call (ticket reset + streaming kernel "
                  "+ finalize, conservative)") +
                 " over K steps replayed phase by phase right after the timed loop (which replays each step as one "
                 "graph); kernel_only_*: events around the streaming kernel alone (library profiling hook, eager "
                 "calls)"}
    if kernel_only_ms:
        r["kernel_only_ms"] = kernel_only_ms
        r["kernel_only_frac"] = alg_bytes / (kernel_only_ms / 1e3) / 1e9 / peak
    if live:
        r["live_copy_gbs"] = live
        r["frac_of_live_copy"] = achieved / live
    if T is not None:
        r["dual"] = dual_ceiling(U, T, P, kv_bytes, d_ms)
        r["dual"]["note"] = ("the HBM fraction counts distinct bytes; the kernel also re-stages shared sources "
                             "from L2 (T+P slices per layer and K|V): staged bytes against the TMA L2 -> smem "
                             "rate of 32 KiB copies (16.5 TB/s, scripts/tma_sweep.cu); the larger of the two "
                             "times is the kernel's bound")
    return r


def committed_traffic(cfg, key):
    """DRAM bytes per launch of the distance kernel from the committed ncu capture of this
    workload (profiles/ncu_distance_<cfg>.json), if its key matches."""
    prof = os.path.join(ROOT, "profiles", f"ncu_distance_{cfg}.json")
    if not os.path.exists(prof):
        return None
    try:
        pj = json.load(open(prof))
    except (ValueError, OSError):
        return None
    if "key" not in pj:
        return pj.get("dram_bytes_per_launch") if cfg not in BATCH_CONFIGS else None
    return pj.get("dram_bytes_per_step") if pj["key"] == key else None


# ----------------------------------------------------------------------------- our arm: one workload per GPU
def run_single(args, rank, world, local):
    import torch
    gpu, dev, dist = init_dist(world, local)
    w = single_workload(args.config, args.seed)
    r = Run(w, dev, args, world, rank, args.mode, dist)
    r.prepare()
    alg_bytes, U, kv_bytes = r.alg_bytes()
    P, T = r.counts["pairs"], r.counts["targets"]
    if args.breakdown:
        p = r.path
        calls = {"restore (state copy)": r.restore, "segment_steps": p.segment,
                 "step_candidates": lambda: p.candidates(w.tau_s),
                 "block_distance": lambda: p.distance_call(w.tau_b), "remap": p.remap}
        for name, fn in calls.items():
            for _ in range(5):
                fn()
            ea, eb = r.ev(), r.ev()
            ea.record(r.stream)
            for _ in range(100):
                fn()
            eb.record(r.stream)
            torch.cuda.synchronize()
            print(f"breakdown {name}: {ea.elapsed_time(eb) / 100 * 1e3:.1f} us (eager launches)", file=sys.stderr)
        r.restore()
        torch.cuda.synchronize()
    clocks = ClockSampler(gpu)
    time.sleep(0.3)
    ms_step, d_ms = r.timed(clocks)
    ck = clocks.stop()
    step_freed, step_affected = int(r.path.num_freed.item()), int(r.path.affected.item())
    kernel_only_ms = r.kernel_only(max(5, min(args.steps, 50))) if args.mode == "seq" else None
    ms_step, pairs_all = reduce_max_sum(dist, dev, ms_step, P)
    if args.mode == "headshard":
        pairs_all = float(P)             # every rank scores the same pairs (strong scaling)
    value = pairs_all / (ms_step / 1e3)
    online = r.online() if args.mode == "seq" and not args.no_online else None
    e2e = None
    if not args.no_e2e:
        e_ms, h2d, d2h = r.e2e(max(10, min(args.steps, 200)))
        e_ms, _ = reduce_max_sum(dist, dev, e_ms, 0)
        e2e = {"value": pairs_all / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
               "note": "public API (MemSharePath over the C ABI); per step: one pinned H2D of the round's inputs "
                       "(tokens, offsets, block table, refcounts, free list), the 4 calls, D2H of counters + "
                       "decisions and of the rewritten table, the host reads each round's counters; the KV pool "
                       "is the device-resident serving cache; the round is replayed as one CUDA graph, two rounds "
                       "in flight (double-buffered pinned results)"}
    parity = r.parity_sample() if not args.no_parity else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        o = oracle_pass(w, r.path.k_pool, r.path.v_pool)
        one = {"value": o["pairs"] / o["t_total"], "cores": 1,
               "sample": (f"oracle (fp64, single thread) on the {args.config} workload: a1-a4 in full, a5-a7 on "
                          f"{o['pairs']} of {o['all_pairs']} pairs ({o['targets']} whole targets)")}
        cpu = all_cores_baseline(args.config, args.seed, [0])
        cpu["single_core"] = one
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak" if args.mode == "seq" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": describe(args.config, w, world, args.mode,
                           {"seqs_per_gpu": w.batch.num_seqs, "tokens_per_gpu": w.num_tokens,
                            **({"collective": r.collective} if r.collective != "none" else {})}),
        "roofline": roofline(alg_bytes, d_ms, kernel_only_ms, kv_bytes, U, P,
                             committed_traffic(args.config, f"{args.config}_seed{args.seed}"),
                             "distance_st_kernel (memshare_block_distance_remap)" if r.fused
                             else "distance_st_kernel (memshare_block_distance)", live=live_copy_gbs(dev), T=T),
        "per_step": {"pairs": P, "targets": T, "steps": r.counts["steps"], "matches": r.counts["matches"],
                     "freed_blocks": step_freed, "affected_tokens": step_affected},
        "gpu_launches": gpu_launches_per_step(w.num_tokens, torch.cuda.get_device_properties(dev).multi_processor_count,
                                              r.fused) * args.steps,
        "clocks": ck, "e2e": e2e, "cpu_baseline": cpu, "online": online, "parity": parity,
    }
    if args.config == "c2" and args.mode == "seq" and args.seed_sweep:
        line["seed_stats"] = seed_sweep(args, dev, [int(x) for x in args.seed_sweep.split(",")], dist)
    line["roofline"]["kernel_share_of_step"] = d_ms / ms_step
    return line, dist, (parity is None or parity["ok"])


def seed_sweep(args, dev, seeds, dist):
    """The c2 step on other seeds' traces (five runs): pairs per second and the
    distance call's fraction of the HBM peak per seed, and their mean / min / max. Each seed is a
    different trace with a different amount of source sharing (192-622 pairs over 241-404 blocks)."""
    from synth import workloads
    per = []
    for sd in seeds:
        w = workloads.c2(seed=sd)
        r = Run(w, dev, args, 1, 0, "seq", dist)
        r.prepare()
        alg, U, kvb = r.alg_bytes()
        clocks = ClockSampler(dev.index or 0)
        ms, d_ms = r.timed(clocks)
        clocks.stop()
        per.append({"seed": sd, "pairs": r.counts["pairs"], "targets": r.counts["targets"], "distinct_blocks": U,
                    "ms_per_step": ms, "pairs_per_s": r.counts["pairs"] / (ms / 1e3),
                    "distance_frac": alg / (d_ms / 1e3) / 1e9 / measured_peaks()[0],
                    "dual": dual_ceiling(U, r.counts["targets"], r.counts["pairs"], kvb, d_ms)})
        r.free()
    st = lambda k: {"mean": float(np.mean([x[k] for x in per])), "min": float(min(x[k] for x in per)),
                    "max": float(max(x[k] for x in per))}
    fb = [x["dual"]["frac_of_bound"] for x in per]
    return {"seeds": seeds, "pairs_per_s": st("pairs_per_s"), "distance_frac": st("distance_frac"),
            "frac_of_dual_bound": {"mean": float(np.mean(fb)), "min": float(min(fb)), "max": float(max(fb))},
            "per_seed": per}


# ----------------------------------------------------------------------------- our arm: a partitioned batch
def stage1_costs(cfg, n, seed, dev):
    """Per-sequence Stage-1 pair counts of the first n sequences of batch `cfg` (a1-a4 on this GPU,
    no KV pool; chunks of 64 sequences). Every rank computes the same numbers."""
    import torch

    from paper_2507_21433_b200.pipeline import MemSharePath
    from synth import workloads
    _, _, shape, _, _, _ = workloads.BATCHES[cfg]
    costs = np.zeros(n, np.int64)
    for c0 in range(0, n, 64):
        idx = list(range(c0, min(n, c0 + 64)))
        w = workloads.batch(cfg, idx, seed)
        b = w.batch
        p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                         w.free_count, None, None, 0, 0, w.num_blocks, shape.num_layers, shape.num_kv_heads,
                         shape.num_kv_heads, shape.head_dim, shape.block_size, device=dev)
        p.autosize(w.tau_s)                       # sizes the buffers (count-then-fill), then fill
        p.segment()
        p.candidates(w.tau_s)
        pr = p.read_candidates()["pairs"]
        assert p.read_status() == 0
        costs[c0:c0 + len(idx)] = np.bincount(pr["seq"], minlength=len(idx))[:len(idx)]
        del p
        torch.cuda.empty_cache()
    return costs


def bin_waves(costs, world, cap):
    """Host logic of the partition: LPT bins of the sequences over world x W (rank r's waves are
    bins r*W .. r*W+W-1), W = the fewest waves per rank with at most `cap` sequences in any wave.
    A sequence without Stage-1 pairs still costs a1-a4 (cost + 1)."""
    from paper_2507_21433_b200.sharding import lpt_assign
    n = len(costs)
    W = max(1, math.ceil(math.ceil(n / world) / cap))
    while True:
        bins = lpt_assign([int(c) + 1 for c in costs], world * W)
        if max(len(b) for b in bins) <= cap:
            return bins, W
        W += 1


def plan_waves(cfg, n, world, seed, dev):
    """The partition of the first n sequences of batch `cfg`: Stage-1 pair counts on this GPU, then
    bin_waves with the wave size capped by POOL_BUDGET of KV per GPU."""
    from synth import workloads
    _, _, shape, _, length, _ = workloads.BATCHES[cfg]
    seq_bytes = max(-(-length(seed, i) // shape.block_size) for i in range(n)) * shape.block_bytes
    cap = max(1, int(POOL_BUDGET // seq_bytes))
    costs = stage1_costs(cfg, n, seed, dev)
    bins, W = bin_waves(costs, world, cap)
    return bins, W, costs


def run_batch(args, rank, world, local):
    import torch

    from synth import workloads
    gpu, dev, dist = init_dist(world, local)
    cfg = args.config
    ci, n_total, shape, _, _, _ = workloads.BATCHES[cfg]
    n = args.batch_seqs if 0 < args.batch_seqs <= n_total else n_total
    t_plan = time.perf_counter()
    bins, W, costs = plan_waves(cfg, n, world, args.seed, dev)
    t_plan = time.perf_counter() - t_plan
    my_waves = bins[rank * W:(rank + 1) * W]
    clocks = ClockSampler(gpu)
    time.sleep(0.3)
    waves, ms_step, e_ms, parity_ok = [], 0.0, 0.0, True
    tot = {"pairs": 0, "targets": 0, "steps": 0, "matches": 0, "alg": 0, "kv": 0, "U": 0, "d_ms": 0.0, "k_ms": 0.0,
           "freed": 0, "affected": 0, "tokens": 0, "h2d": 0, "d2h": 0, "launches": 0}
    online, first_w, fused_tail = None, None, True
    for wi, idx in enumerate(my_waves):
        if not idx:
            continue
        w = workloads.batch(cfg, idx, args.seed)
        first_w = first_w or w
        r = Run(w, dev, args, world, rank, "seq", dist)
        fused_tail = r.fused
        r.prepare()
        alg, U, kvb = r.alg_bytes()
        m, d_ms = r.timed(clocks)
        ms_step += m
        freed, affected = int(r.path.num_freed.item()), int(r.path.affected.item())
        k_ms = r.kernel_only(5)
        if wi == 0 and rank == 0 and not args.no_online:
            online = r.online()
        wave_e2e = None
        if not args.no_e2e:
            wave_e2e, h2d, d2h = r.e2e(max(5, min(args.steps, 20)))
            e_ms += wave_e2e
            tot["h2d"] += h2d
            tot["d2h"] += d2h
        par = r.parity_sample(seed=1000 * rank + wi) if not args.no_parity else None
        parity_ok &= par is None or par["ok"]
        c = r.counts
        for k_, v_ in (("pairs", c["pairs"]), ("targets", c["targets"]), ("steps", c["steps"]),
                       ("matches", c["matches"]), ("alg", alg), ("kv", kvb), ("U", U), ("d_ms", d_ms),
                       ("k_ms", k_ms), ("freed", freed), ("affected", affected), ("tokens", w.num_tokens),
                       ("launches", gpu_launches_per_step(w.num_tokens,
                                                          torch.cuda.get_device_properties(dev).multi_processor_count,
                                                          r.fused))):
            tot[k_] += v_
        waves.append({"rank": rank, "wave": wi, "seqs": len(idx), "tokens": w.num_tokens, "pairs": c["pairs"],
                      "targets": c["targets"], "distinct_blocks": U, "ms_per_step": m, "distance_ms": d_ms,
                      "kernel_only_ms": k_ms, "distance_frac": alg / (d_ms / 1e3) / 1e9 / measured_peaks()[0],
                      "dual": dual_ceiling(U, c["targets"], c["pairs"], kvb, d_ms),
                      "e2e_ms_per_step": wave_e2e, "parity": par, "pool_gb": w.pool_bytes() / 1e9})
        r.free()
        del r, w
    ck = clocks.stop()
    # job time per step = the slowest rank's summed wave times; pairs summed over ranks
    job_ms, pairs_all = reduce_max_sum(dist, dev, ms_step, tot["pairs"])
    value = pairs_all / (job_ms / 1e3)
    e2e = None
    if not args.no_e2e:
        e_job, _ = reduce_max_sum(dist, dev, e_ms, 0)
        e2e = {"value": pairs_all / (e_job / 1e3), "unit": UNIT, "h2d_bytes_per_step": tot["h2d"],
               "d2h_bytes_per_step": tot["d2h"], "ms_per_step": e_job,
               "note": "public API (MemSharePath over the C ABI) per wave while its KV pool is resident: one pinned "
                       "H2D of the wave's inputs (tokens, offsets, block table, refcounts, free list), the 4 calls, "
                       "D2H of counters + decisions and of the rewritten table, the host reads each round's "
                       "counters; a step = every wave of the rank (sum of the waves' e2e step times), max over ranks; "
                       "bytes per step are this rank's"}
    # every rank's wave records to rank 0
    all_waves = waves
    ok_all = parity_ok
    if dist is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, (waves, parity_ok))
        all_waves = [x for g in gathered for x in g[0]]
        ok_all = all(g[1] for g in gathered)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = all_cores_baseline(cfg, args.seed, list(range(min(n, os.cpu_count() or 1))))
    fr = [x["distance_frac"] for x in all_waves]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": job_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": describe(cfg, first_w, world, "seq",
                           {"batch_seqs": n, "batch_tokens": int(sum(workloads.BATCHES[cfg][4](args.seed, i)
                                                                     for i in range(n))),
                            "waves_per_gpu": W, "partition": "LPT on per-sequence Stage-1 pair counts "
                                                              "(sharding.lpt_assign), computed before the timed region",
                            "plan_s": round(t_plan, 2), "baseline_config": f"configs[{ci}]"}),
        "roofline": roofline(tot["alg"], tot["d_ms"], tot["k_ms"], tot["kv"], tot["U"], tot["pairs"],
                             committed_traffic(cfg, f"{cfg}_{n}seq_{world}gpu_seed{args.seed}"),
                             "distance_st_kernel (memshare_block_distance_remap)" if fused_tail
                             else "distance_st_kernel (memshare_block_distance)", live=live_copy_gbs(dev),
                             T=tot["targets"]),
        "per_step": {"pairs": int(pairs_all), "pairs_rank0": tot["pairs"], "targets_rank0": tot["targets"],
                     "steps_rank0": tot["steps"], "matches_rank0": tot["matches"], "freed_blocks_rank0": tot["freed"],
                     "affected_tokens_rank0": tot["affected"]},
        "waves": all_waves,
        "load_balance": {"rank_ms": None, "lpt_costs_total": int(costs.sum())},
        "gpu_launches": tot["launches"] * args.steps,
        "clocks": ck, "e2e": e2e, "cpu_baseline": cpu, "online": online,
        "parity": {"ok": bool(ok_all), "checked_waves": sum(1 for x in all_waves if x.get("parity")),
                   "what": "per wave: a1-a4 and the remap bit-exact vs the oracle; 8 sampled targets' distances "
                           "within 1e-5 and their decisions by the tie / threshold rules"},
    }
    line["roofline"]["kernel_share_of_step"] = tot["d_ms"] / max(ms_step, 1e-9)
    line["roofline"]["frac_per_wave"] = {"min": min(fr) if fr else None, "max": max(fr) if fr else None}
    if dist is not None:
        rank_ms = [None] * world
        dist.all_gather_object(rank_ms, ms_step)
        line["load_balance"]["rank_ms"] = rank_ms
    else:
        line["load_balance"]["rank_ms"] = [ms_step]
    return line, dist, ok_all


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return 0
    if args.config in BATCH_CONFIGS:
        line, dist, ok = run_batch(args, rank, world, local)
    else:
        line, dist, ok = run_single(args, rank, world, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
