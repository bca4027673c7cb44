"""Child process of tests/test_gpu_progress.py (environment knobs are read once per process).

  python tests/_progress_child.py last_many|range|last_long_step|contended

Runs one round through the C ABI and the full oracle parity check (test_gpu_path.full_parity);
prints "ok" on success.
"""
import ctypes
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth import kv, traces, workloads  # noqa: E402

SMALL = kv.KVShape(8, 4, 64, 16)

HOLD_SRC = r"""
#include <cuda_runtime.h>
__global__ void hold(volatile int* flag) {
  extern __shared__ int pad[];
  if (threadIdx.x == 0) {
    pad[0] = 1;
    while (*flag == 0) __nanosleep(2000);
  }
  __syncthreads();
}
extern "C" int hold_launch(int blocks, int* flag, void* stream) {
  cudaFuncSetAttribute(hold, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  hold<<<blocks, 1024, 200 * 1024, (cudaStream_t)stream>>>(flag);
  return (int)cudaGetLastError();
}
"""


def holder():
    """A kernel on its own stream that keeps `blocks` SMs busy (one 1024-thread, 200 KB CTA per SM)
    until the host flips a mapped flag."""
    d = tempfile.mkdtemp()
    src, so = os.path.join(d, "hold.cu"), os.path.join(d, "libhold.so")
    open(src, "w").write(HOLD_SRC)
    subprocess.check_call(["nvcc", "-O2", "-shared", "-cudart", "shared", "-Xcompiler", "-fPIC", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-o", so, src])
    return ctypes.CDLL(so)


def main(case):
    import torch
    from test_gpu_path import full_parity
    if case == "last_many":
        # 40 sequences with 8-CTA clusters: 18 clusters launched for 40 work items, fewer co-resident
        w = workloads.small(SMALL, 40, 900, seed=40, gen_start=16)
        full_parity(w, tau_s=0.5, cur_mode=oracle.CUR_LAST)
    elif case == "range":
        w = workloads.small(SMALL, 3, 3000, seed=3)
        full_parity(w, cur_mode=oracle.CUR_RANGE, cb=[0, 5, 10], ce=[4, 30, 11])
        w = workloads.small(SMALL, 30, 1200, seed=5, gen_start=16)
        full_parity(w, tau_s=0.5, cur_mode=oracle.CUR_RANGE, cb=[1] * 30, ce=[9] * 30)
    elif case == "last_long_step":
        # the last step has > 2048 content tokens, so its count table is the
        # shared global one; only cluster rank 0 may fill it
        rng = np.random.default_rng(4)
        long_step = rng.integers(10, 900, 6000).astype(np.int32)
        toks = np.concatenate([long_step, [1], rng.integers(10, 900, 3000), [1], long_step[:5000], [1],
                               long_step, [1]]).astype(np.int32)
        b = traces.TraceBatch(tokens=toks, seq_tok_off=np.array([0, toks.size]), gen_start=np.zeros(1, np.int32),
                              final=np.ones(1, np.uint8), delim_ids=np.array([1], np.int32), vocab=1000)
        w = workloads._paged("long_last", SMALL, b, 1, 0.05, 0.5)
        for _ in range(3):                     # run-to-run: a race would show as varying counts
            full_parity(w, cur_mode=oracle.CUR_LAST)
    elif case == "contended":
        import time
        from _gpu_util import make_path
        from test_gpu_path import check_round
        lib = holder()
        # one long CoT: ~600 steps > 148 Stage-1 CTAs (each CTA takes several work items) and ~30
        # segmentation tiles
        w = workloads.small(SMALL, 1, 60000, seed=9)
        p = make_path(w)
        p.autosize(w.tau_s)
        # one full round first: every kernel's module is loaded now (a lazy module load during the
        # contended round would wait for the device -- i.e. for the holder -- on the host thread)
        p.round(w.tau_s, w.tau_b)
        torch.cuda.synchronize()
        p = make_path(w)
        p.autosize(w.tau_s)
        torch.cuda.synchronize()
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")   # the holder polls this word
        one = torch.ones(1, dtype=torch.int32).pin_memory()
        side, dma = torch.cuda.Stream(), torch.cuda.Stream()
        torch.cuda.synchronize()
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        assert lib.hold_launch(sms - 8, ctypes.c_void_p(flag.data_ptr()), ctypes.c_void_p(side.cuda_stream)) == 0
        time.sleep(0.5)                                          # the holder occupies sms - 8 SMs
        print(f"holder running: {not side.query()}", flush=True)
        done = torch.cuda.Event()
        p.round(w.tau_s, w.tau_b)
        done.record()
        t0 = time.time()
        while not done.query() and time.time() - t0 < 30.0:
            time.sleep(0.01)
        finished_while_held = done.query()
        print(f"round finished while held: {finished_while_held} after {time.time() - t0:.2f} s; "
              f"holder still running: {not side.query()}", flush=True)
        with torch.cuda.stream(dma):                             # release the holder either way (copy engine)
            flag.copy_(one, non_blocking=True)
        side.synchronize()
        torch.cuda.synchronize()
        assert finished_while_held, "the round made no progress on the 8 free SMs"
        check_round(p, w, w.tau_s, w.tau_b)
    else:
        raise SystemExit(f"unknown case {case}")
    print("ok", flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
