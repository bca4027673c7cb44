#!/usr/bin/env python
"""Benchmark of the MemShare KV-block reuse path on B200 (BASELINE.json metric:
"candidate KV-block pairs scored/s and HBM GB/s (% of peak) at 1/2/4/8 B200").

One STEP = one full pass of the hot path (a1 segment -> a2-a4 Stage 1 + pairs -> a5-a6 block
distance + selection -> a7 remap) over one batch (configs[1] = "c2": one 12,406-token
synthetic CoT with DeepSeek-R1-Distill-Qwen-32B's KV shape) per GPU. Before each step the block
table / refcounts / free list are restored from a pristine device copy (a few KB), so every step
does identical work. Inputs are resident in HBM; the 3.25 GB KV pool (1.38 GB of distinct blocks
read per step) is far larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
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
# our kernels per step: seg, encode, stage1, [fill], distance, finalize, remap (+ 2 memset nodes);
# the fill kernel runs only when stage1 does not fuse it (the library fuses it for an offline
# round over a single CoT-sized batch: <= 100 x 8 x SMs tokens, no cluster; MEMSHARE_FUSED_FILL=0 disables)
def gpu_launches_per_step(num_tokens, sms=148):
    fused = num_tokens <= 100 * 8 * sms and os.environ.get("MEMSHARE_FUSED_FILL", "1") != "0"
    # flag reset, seg, encode, stage1, (fill), ticket reset, distance, finalize, remap
    return 8 if fused else 9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c2", choices=["c2", "tiny", "c3", "c4", "c5"])
    ap.add_argument("--seqs-per-gpu", type=int, default=0, help="c3/c4: sequences per GPU (0 = config default)")
    ap.add_argument("--wave", type=int, default=0,
                    help="c3/c5: which wave of the batch (rank r of N holds sequences (wave*N + r)*seqs ...); a "
                         "64-sequence batch on 1 GPU is waves 0 and 1 of 32")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="seq", choices=["seq", "headshard"])
    ap.add_argument("--collective", default="p2p", choices=["p2p", "nccl"],
                    help="headshard, N>1: 'p2p' = FINALIZE reads every rank's partial sums over NVLink from "
                         "symmetric memory (memshare_block_distance_finalize_peers); 'nccl' = all-reduce + FINALIZE")
    ap.add_argument("--seed", type=int, default=int(os.environ.get("MEMSHARE_SEED", "0")))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--breakdown", action="store_true", help="also time each ABI call separately (stderr)")
    ap.add_argument("--no-graph", action="store_true", help="launch the calls directly instead of CUDA-graph replay")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def make_workload(cfg, seed, rank, seqs, wave=0, world=1):
    from synth import workloads
    if cfg == "c2":
        # weak scaling: every rank runs configs[1] itself (identical per-GPU work); other seeds give
        # 192-622 pairs, which would make the max-over-ranks time measure seed variance, not scaling
        return workloads.c2(seed=seed)
    if cfg == "tiny":
        return workloads.tiny(eta=0.05)
    if cfg == "c3":
        return workloads.c3(num_seqs=seqs or 8, seed=seed, first_seq=(wave * world + rank) * (seqs or 8))
    if cfg == "c4":
        return workloads.c4(num_seqs=seqs or 8, seed=seed + rank)
    if cfg == "c5":
        return workloads.c5(num_seqs=seqs or 32, seed=seed, first_seq=(wave * world + rank) * (seqs or 32))
    raise ValueError(cfg)


def describe(cfg, w, world, mode):
    sh = w.shape
    return {"workload": {"c2": "configs[1]: DeepSeek-R1-Distill-Qwen-32B KV shape, 1 x 12,406-token synthetic CoT "
                                "per GPU (128-token prompt, MATH-500-like planted redundancy; every rank runs the "
                                "same sequence: identical per-GPU work)",
                         "tiny": "configs[0]: tiny T0 fixture",
                         "c3": "configs[2]: QwQ-32B KV shape, 12,288-token CoTs",
                         "c4": "configs[3]: Phi-4-reasoning-plus KV shape, AIME-length traces",
                         "c5": "configs[4]: 32B KV shape, 16,384-token CoTs (512 over 8 GPUs = 2 waves of 32 per "
                               "GPU; this line is one wave)"}[cfg],
            "kv_shape": {"layers": sh.num_layers, "kv_heads": sh.num_kv_heads, "head_dim": sh.head_dim,
                         "block_size": sh.block_size, "kv_dtype": "bf16"},
            "seqs_per_gpu": w.batch.num_seqs, "tokens_per_gpu": w.num_tokens, "tau_s": w.tau_s,
            "tau_b": round(w.tau_b, 6), "eta": w.eta, "pairing": "aligned", "stage1": "offline (every step current)",
            "parallelism": (f"seq-shard dp{world}" if mode == "seq" else f"kv-head-shard hs{world}"),
            "l2": "inputs larger than L2 (pool %.2f GB/GPU vs 126 MB L2); no flush" % (w.pool_bytes() / 1e9),
            **({"first_seq": int(getattr(w, "first_seq", 0))} if cfg in ("c3", "c5") else {})}


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
        self.t0 = self.t1 = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

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
        inwin = [r for r in rows if self.t0 - 1 <= r[0] <= self.t1 + 1] or rows
        if not inwin:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inwin for i, x in enumerate(r[3]) if x.lower() == "active"})
        return {"sm_mhz": float(np.median([r[1] for r in inwin])), "sm_max_mhz": max(r[2] for r in inwin),
                "reasons": reasons, "samples": len(inwin)}


# ----------------------------------------------------------------------------- oracle
def oracle_pass(w, k_pool, v_pool, max_pairs=600, budget_s=20.0):
    """The oracle as it stands on the host: a1-a4 in full, then a5-a6 on whole target groups in
    order (at most `max_pairs` pairs / `budget_s` seconds; all of c2), then a7 on those decisions.
    Only the KV blocks those pairs touch are copied from the device pool to the host."""
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


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the oracle (this tier's reference arm), as it stands, on host cores."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    w = make_workload(args.config, args.seed, 0, args.seqs_per_gpu, args.wave)
    k, v, ls, bs = w.host_pool()
    sh = w.shape
    st = oracle.segment_steps(w.batch.tokens, w.batch.seq_tok_off, w.batch.gen_start, w.batch.final, w.batch.delim_ids)
    oc = oracle.step_candidates(w.batch.tokens, w.batch.seq_tok_off, st, w.batch.delim_ids, w.table, sh.block_size,
                                w.tau_s)
    pr, toff = oc["pairs"], oc["target_off"]
    T = toff.size - 1
    # calibrate: seconds per target group (a5-a6 on all pairs of a target)
    t0 = time.perf_counter()
    one = oracle.block_distance(k, v, ls, bs, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads, sh.head_dim,
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
              f"(~{np.mean(pairs_done):.1f} pairs) per step, rotating over the {pr['seq'].size} pairs of the "
              f"{args.config} workload; a1-a4/a7 excluded from the steps")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": describe(args.config, w, 1, "seq"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": host_cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

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
    from paper_2507_21433_b200 import _lib as L
    from paper_2507_21433_b200.pipeline import MemSharePath, pack_inputs

    w = make_workload(args.config, args.seed, rank if args.mode == "seq" else 0, args.seqs_per_gpu, args.wave,
                      world if args.mode == "seq" else 1)
    sh = w.shape
    h_local, h_off = sh.num_kv_heads, 0
    if args.mode == "headshard":
        from paper_2507_21433_b200.sharding import head_shard
        h_local, h_off = head_shard(sh.num_kv_heads, world, rank)
    k, v, ls, bs = w.device_pool(dev, h_local=h_local, head_offset=h_off)
    b = w.batch
    path = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                        w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, h_local, sh.num_kv_heads,
                        sh.head_dim, sh.block_size, device=dev)
    counts = path.autosize(w.tau_s)
    if args.mode == "headshard":
        path.alloc_partial()
    # headshard across GPUs: the cross-rank reduction fused into FINALIZE over peer memory
    symm_hdl, peer_ptrs, collective = None, None, ("none" if world == 1 or args.mode != "headshard" else args.collective)
    if collective == "p2p":
        try:
            import torch.distributed._symmetric_memory as symm
            buf = symm.empty(path.partial_sq.numel(), dtype=torch.float32, device=dev)
            symm_hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
            path.partial_sq = buf                      # PARTIAL writes into this rank's symmetric buffer
            peer_ptrs = torch.tensor(list(symm_hdl.buffer_ptrs), dtype=torch.int64, device=dev)
        except Exception as e:                         # no symmetric memory on this node: NCCL all-reduce
            print(f"bench: symmetric memory unavailable ({e!r}); using the NCCL all-reduce", file=sys.stderr)
            collective = "nccl"

    def headshard_distance():
        path.distance_call(w.tau_b, L.DIST_PARTIAL)
        if collective == "p2p":
            symm_hdl.barrier(channel=0)                # every rank's partial sums are written
            path.finalize_peers(w.tau_b, peer_ptrs, world)
            symm_hdl.barrier(channel=1)                # every rank has read them (buffer reusable)
        else:
            if collective == "nccl":
                dist.all_reduce(path.partial_sq[:counts["pairs"] * sh.num_layers * 2])
            path.distance_call(w.tau_b, L.DIST_FINALIZE)
    torch.cuda.synchronize()
    pristine = path.state.clone()
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def restore():               # table + refcounts + free list + free count: one device copy
        path.state.copy_(pristine, non_blocking=True)

    def front():                 # restore the round's initial state, a1, a2-a4
        restore()
        path.segment()
        path.candidates(w.tau_s)

    def middle():                # a5-a6 (the HBM-bound kernel)
        if args.mode == "headshard":
            headshard_distance()
        else:
            path.distance_call(w.tau_b)

    def back():                  # a7
        path.remap()

    for fn in (front, middle, back):      # eager warm-up (module load, attributes)
        fn()
    torch.cuda.synchronize()
    if args.no_graph or collective != "none":    # collectives / symmetric-memory barriers run eagerly
        run = (front, middle, back)
    else:                                  # one CUDA graph per phase; events between replays
        run = tuple(path.capture(fn).replay for fn in (front, middle, back))

    def step(d_ev=None):
        run[0]()
        if d_ev is not None:
            d_ev[0].record(stream)
        run[1]()
        if d_ev is not None:
            d_ev[1].record(stream)
        run[2]()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert path.read_status() == 0, f"device status {L.status_string(path.read_status())}"
    # distinct physical blocks per step (algorithmic bytes of the distance kernel)
    pr = path.read_candidates()["pairs"]
    U = int(np.unique(np.concatenate([pr["target_phys"], pr["source_phys"]])).size)
    P, T = counts["pairs"], counts["targets"]
    slice_b = sh.block_size * h_local * sh.head_dim * 2
    blk_b = sh.num_layers * 2 * slice_b
    kv_bytes = U * blk_b
    meta_bytes = P * (24 + 4 + 1) + T * (8 + 32)
    alg_bytes = kv_bytes + meta_bytes

    if args.breakdown:
        calls = {"restore (state copy)": restore, "segment_steps": path.segment,
                 "step_candidates": lambda: path.candidates(w.tau_s),
                 "block_distance": lambda: path.distance_call(w.tau_b), "remap": path.remap}
        for name, fn in calls.items():
            for _ in range(5):
                fn()
            ea, eb = ev(), ev()
            ea.record(stream)
            for _ in range(100):
                fn()
            eb.record(stream)
            torch.cuda.synchronize()
            print(f"breakdown {name}: {ea.elapsed_time(eb) / 100 * 1e3:.1f} us (eager launches)", file=sys.stderr)
        restore()
        torch.cuda.synchronize()

    clocks = ClockSampler(gpu)
    time.sleep(0.3)
    d_events = [(ev(), ev()) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    e0, e1 = ev(), ev()
    e0.record(stream)
    for i in range(args.steps):
        step(d_events[i])
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark_end()
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    d_ms = float(np.mean([a.elapsed_time(b_) for a, b_ in d_events]))
    ck = clocks.stop()
    assert path.read_status() == 0
    # counters of the last timed (offline) step, read before the online / e2e legs overwrite them
    step_freed, step_affected = int(path.num_freed.item()), int(path.affected.item())

    # the streaming kernel alone (the timed region's events bracket the whole a5-a6 call: ticket
    # memset + streaming kernel + finalize): the library's profiling hook records a pair of
    # events around the streaming kernel of eager calls, same buffers and launch configuration
    kernel_only_ms = None
    if args.mode == "seq":
        kb, ke = ev(), ev()
        kb.record(stream)
        ke.record(stream)
        torch.cuda.synchronize()
        L.profile_distance_events(kb, ke)
        ks = []
        for i in range(max(5, min(args.steps, 50))):
            run[0]()
            path.distance_call(w.tau_b)
            run[2]()
            torch.cuda.synchronize()
            if i >= 2:
                ks.append(kb.elapsed_time(ke))
        L.profile_distance_events(None, None)
        kernel_only_ms = float(np.mean(ks))

    # max over ranks of the step time; sum of pairs over ranks
    t = torch.tensor([ms_total, float(P)], dtype=torch.float64, device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        ms_total, pairs_all = float(tmax[0]), float(t[1])
    else:
        pairs_all = float(P)
    if args.mode == "headshard":
        pairs_all = float(P)             # every rank scores the same pairs (strong scaling)
    ms_step = ms_total / args.steps
    value = pairs_all / (ms_step / 1e3)

    # ---------------------------------------------------------------- online round latency
    # PAPER.md:317 evaluates each step as it finishes: CUR_LAST = the newly finished step of every
    # sequence against its history (one graph replay per round; table restored each round).
    online = None
    if args.mode == "seq":
        # the busiest step of each sequence (most Stage-1 survivors in the offline pass) as RANGE
        mt = path.read_candidates()["matches"]
        busiest = np.zeros(w.batch.num_seqs, np.int32)
        for sq in range(w.batch.num_seqs):
            st = mt["step"][mt["seq"] == sq]
            if st.size:
                busiest[sq] = np.bincount(st).argmax()

        def time_round(cur_mode, cb=None, ce=None):
            def online_round():
                restore()
                path.segment()
                path.candidates(w.tau_s, cur_mode=cur_mode, cur_begin=cb, cur_end=ce)
                path.distance_call(w.tau_b)
                path.remap()
            online_round()
            torch.cuda.synchronize()
            og = path.capture(online_round)
            for _ in range(10):
                og.replay()
            torch.cuda.synchronize()
            o_pairs = int(path.num_pairs.item())
            o0, o1 = ev(), ev()
            n_on = max(50, min(args.steps, 500))
            o0.record(stream)
            for _ in range(n_on):
                og.replay()
            o1.record(stream)
            torch.cuda.synchronize()
            return 1e3 * o0.elapsed_time(o1) / n_on, o_pairs, n_on

        last_us, last_pairs, n_on = time_round(L.CUR_LAST)
        bb = torch.as_tensor(busiest, device=dev)
        busy_us, busy_pairs, _ = time_round(L.CUR_RANGE, bb, bb + 1)
        online = {"round_us": last_us, "pairs_per_round": last_pairs,
                  "busiest_round_us": busy_us, "busiest_pairs_per_round": busy_pairs,
                  "current_steps_per_round": w.batch.num_seqs, "rounds": n_on,
                  "note": "online (PAPER.md:317): one graph replay of a1-a7 with one current step per sequence -- "
                          "round_us: the last finished step (cur_mode LAST); busiest_round_us: the step with the "
                          "most Stage-1 survivors (cur_mode RANGE)"}
        restore()
        torch.cuda.synchronize()

    # ---------------------------------------------------------------- e2e through the public API
    e2e = None
    if not args.no_e2e:
        # one pinned upload of the round's inputs (trace + serving state, MemSharePath's layout) and
        # one pinned read-back each of the outputs (counters + decisions) and the state head
        # (free count + rewritten block table)
        host_in, _ = pack_inputs(b.tokens, b.seq_tok_off, b.gen_start, b.final, w.table, w.refcount, w.free_list,
                                 w.free_count)
        h_in = torch.from_numpy(host_in).pin_memory()
        assert h_in.numel() == path.inputs.numel()
        h2d = h_in.numel() * 4
        n_head = 2 + path.table.numel()
        # two pinned result sets: with graph replay the host keeps two rounds in flight and reads
        # round i's results (from set i % 2) before it launches round i + 2 into the same set
        outs = [(torch.empty(path.outputs.numel(), dtype=torch.uint8).pin_memory(),
                 torch.empty(n_head, dtype=torch.int32).pin_memory()) for _ in range(2)]
        d2h = outs[0][0].numel() + outs[0][1].numel() * 4

        def round_body(j):
            def body():
                path.inputs.copy_(h_in, non_blocking=True)
                path.segment()
                path.candidates(w.tau_s)
                if args.mode == "headshard":
                    headshard_distance()
                else:
                    path.distance_call(w.tau_b)
                path.remap()
                outs[j][0].copy_(path.outputs, non_blocking=True)
                outs[j][1].copy_(path.state[:n_head], non_blocking=True)
            return body

        def consume(j):                 # the host reads the round's result
            o = outs[j][0][:64].view(torch.int64)
            assert int(o[1]) == P, "e2e round result"

        e2e_graph = not args.no_graph and collective == "none"
        if e2e_graph:
            # a serving loop replays the round as one CUDA graph: memcpy nodes read the pinned
            # host inputs / write the pinned host outputs at replay time, the ABI calls in between
            gs = []
            for j in range(2):
                round_body(j)()
                torch.cuda.synchronize()
                gs.append(path.capture(round_body(j)))
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
                done[j].record(torch.cuda.current_stream(dev))
                inflight[j] = True

            def e2e_drain():
                for j in range(2):
                    if inflight[j]:
                        done[j].synchronize()
                        consume(j)
                        inflight[j] = False
        else:
            body0 = round_body(0)

            def e2e_step():
                body0()
                torch.cuda.current_stream(dev).synchronize()
                consume(0)

            def e2e_drain():
                pass

        for _ in range(max(3, args.warmup // 4)):
            e2e_step()
        e2e_drain()
        n_e2e = max(10, min(args.steps, 200))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a0, a1 = ev(), ev()
        a0.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        e2e_drain()
        a1.record(stream)
        torch.cuda.synchronize()
        e_ms = a0.elapsed_time(a1) / n_e2e
        te = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = float(te[0])
        e2e = {"value": pairs_all / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms, "steps": n_e2e,
               "note": "public API (MemSharePath over the C ABI); per step: one pinned H2D of the round's inputs "
                       "(tokens, offsets, block table, refcounts, free list), the 4 calls, D2H of counters + "
                       "decisions and of the rewritten table, the host reads each round's counters; the KV pool "
                       "is the device-resident serving cache" + ("; the round (H2D + calls + D2H) is replayed as one "
                       "CUDA graph captured through MemSharePath.capture, two rounds in flight (double-buffered "
                       "pinned results: round i's are read before round i+2 is launched)" if e2e_graph else
                       "; calls launched eagerly, a host sync per round")}

    # ---------------------------------------------------------------- cpu baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_pass(w, path.k_pool, path.v_pool)
        cpu = {"value": r["pairs"] / r["t_total"], "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": (f"oracle (fp64, single thread) on the {args.config} workload: a1-a4 in full, a5-a7 on "
                          f"{r['pairs']} of {r['all_pairs']} pairs ({r['targets']} whole targets); front "
                          f"{r['t_front']:.2f}s, stage2 {r['t_stage2']:.2f}s, remap {r['t_remap']:.3f}s"),
               "cpu": host_cpu_model(), "host_cores": os.cpu_count()}

    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (d_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_distance_{args.config}.json")
    if os.path.exists(prof):                   # the committed ncu capture of this exact workload
        try:
            pj = json.load(open(prof))
            if int(pj.get("seqs_per_gpu", w.batch.num_seqs)) == w.batch.num_seqs and args.mode == "seq":
                traffic = pj.get("dram_bytes_per_launch")
        except (ValueError, OSError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak" if args.mode == "seq" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {**describe(args.config, w, world, args.mode),
                   **({"collective": {"p2p": "FINALIZE reads all ranks' partial sums over NVLink (symmetric memory)",
                                      "nccl": "NCCL all-reduce of partial sums, then FINALIZE"}[collective]}
                      if collective != "none" else {})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "distance_st_kernel (memshare_block_distance)",
                     "kernel_ms": d_ms, "kernel_share_of_step": d_ms / ms_step, "algorithmic_bytes": alg_bytes,
                     "pairs_per_s_a5a6": P / (d_ms / 1e3),
                     "kv_bytes": kv_bytes, "distinct_blocks": U, "peak_source": peak_src,
                     "frac_of_nominal_8000": achieved / 8000.0,
                     "note": "achieved/kernel_ms: CUDA events around the whole a5-a6 call inside the timed loop "
                             "(ticket memset + streaming kernel + finalize, conservative); kernel_only_*: events "
                             "around the streaming kernel alone (library profiling hook, eager calls after the "
                             "timed loop)",
                     **({"kernel_only_ms": kernel_only_ms,
                         "kernel_only_frac": alg_bytes / (kernel_only_ms / 1e3) / 1e9 / peak}
                        if kernel_only_ms else {})},
        "per_step": {"pairs": P, "targets": T, "steps": counts["steps"], "matches": counts["matches"],
                     "freed_blocks": step_freed, "affected_tokens": step_affected},
        "gpu_launches": gpu_launches_per_step(w.num_tokens, torch.cuda.get_device_properties(dev).multi_processor_count)
        * args.steps,
        "clocks": {"sm_mhz": ck["sm_mhz"], "sm_max_mhz": ck["sm_max_mhz"], "reasons": ck["reasons"],
                   "samples": ck["samples"]},
        "e2e": e2e, "cpu_baseline": cpu, "online": online,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
