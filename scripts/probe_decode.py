"""Tuning probe (not part of the product): decode attention bandwidth through a paged table.
Usage: python scripts/probe_decode.py [num_seqs] [seq_len]"""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2507_21433_b200 import _lib as L  # noqa: E402
from synth import decode as sd  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12288
N, h, dh, d, hq = 4, 8, 128, 16, 40
nbs = -(-n // d)
nb = S * nbs + 8
sl = d * h * dh
dev = torch.device("cuda")
k = torch.randn(N * nb * sl, dtype=torch.bfloat16, device=dev)
v = torch.randn(N * nb * sl, dtype=torch.bfloat16, device=dev)
rng = np.random.default_rng(0)
table = torch.as_tensor(rng.permutation(nb)[:S * nbs].reshape(S, nbs).astype(np.int32), device=dev)
lens = torch.full((S,), n, dtype=torch.int32, device=dev)
q = torch.randn(S, hq, dh, dtype=torch.bfloat16, device=dev)
out = torch.empty(S, hq, dh, dtype=torch.float32, device=dev)
dims = L.Dims(N, h, h, dh, d)
pool = L.KVPool(k.data_ptr(), v.data_ptr(), nb * sl, sl, nb, 0)
ws = torch.empty(L.paged_attention_workspace_size(dims, S, hq, n), dtype=torch.uint8, device=dev)
st = torch.zeros(1, dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def call(layer):
    L.check(L.paged_attention_decode(pool, dims, layer, q, hq, table, nbs, lens, S, n, 1 / math.sqrt(dh), out, ws, st))


for layer in range(N):
    call(layer)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
times = []
for it in range(20):
    flush.zero_()
    ev[0].record()
    call(it % N)
    ev[1].record()
    torch.cuda.synchronize()
    times.append(ev[0].elapsed_time(ev[1]) * 1e3)
byts = S * n * h * dh * 2 * 2
t = float(np.median(times))
print(f"S={S} n={n}: {t:.1f} us/layer, {byts / t / 1e3:.1f} GB/s of KV ({byts / 1e6:.1f} MB), status {st.item()}")
