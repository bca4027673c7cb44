"""The BASELINE.json configurations as concrete seeded inputs (input recipe only).

DESIGN.md §"Input recipe" states the recipe; SURVEY.md §8(d) "The five configs as concrete
inputs" is its source. A Workload holds host arrays (trace, paged block table, refcounts, free
list) and fills a layer-major bf16 KV pool on the host (numpy) or on the device (torch), through
the counter-hash generator twins. Nothing here computes a MemShare quantity.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import kv, traces


def default_tau_b(shape: kv.KVShape, eta: float) -> float:
    """tau_b = 2.5 * eta * sqrt(2 d_h / (d h)): 2.5x the expected distance of an
    exact copy under the generator's noise, well below the ~sqrt(2 d_h/(d h)) of unrelated blocks."""
    return 2.5 * eta * math.sqrt(2.0 * shape.head_dim / (shape.block_size * shape.num_kv_heads))


@dataclass
class Workload:
    name: str
    shape: kv.KVShape
    batch: traces.TraceBatch
    table: np.ndarray
    num_blocks: int
    refcount: np.ndarray
    free_list: np.ndarray
    free_count: int
    seed: int
    eta: float
    tau_s: float
    tau_b: float

    @property
    def num_tokens(self) -> int:
        return int(self.batch.tokens.size)

    def blocks(self):
        return kv.table_blocks(self.batch.seq_tok_off, self.table, self.shape.block_size)

    def pool_bytes(self, h_local: int | None = None) -> int:
        hl = h_local or self.shape.num_kv_heads
        return 2 * self.shape.num_layers * self.num_blocks * self.shape.block_size * hl * self.shape.head_dim * 2

    def host_pool(self, h_local=None, head_offset=0):
        k, v, ls, bs = kv.host_pool(self.shape, self.num_blocks, h_local)
        s_, l_, p_ = self.blocks()
        kv.fill_blocks_host(k, v, ls, bs, self.shape, self.batch.tokens, self.batch.seq_tok_off, s_, l_, p_,
                            self.seed, self.eta, h_local, head_offset)
        return k, v, ls, bs

    def device_pool(self, device="cuda", h_local=None, head_offset=0, stream=None):
        import torch
        hl = h_local or self.shape.num_kv_heads
        slice_elems = self.shape.block_size * hl * self.shape.head_dim
        n = self.shape.num_layers * self.num_blocks * slice_elems
        k = torch.zeros(n, dtype=torch.bfloat16, device=device)     # unreferenced blocks stay 0 (as on the host)
        v = torch.zeros(n, dtype=torch.bfloat16, device=device)
        s_, l_, p_ = self.blocks()
        dev = torch.device(device)
        t = lambda a, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
        kv.fill_blocks_dev(k, v, self.num_blocks * slice_elems, slice_elems, self.shape, t(self.batch.tokens),
                           t(self.batch.seq_tok_off, torch.int64), t(s_), t(l_), t(p_), self.seed, self.eta, hl,
                           head_offset, stream)
        return k, v, self.num_blocks * slice_elems, slice_elems


def _paged(name, shape, batch, seed, eta, tau_s, tau_b=None, identity=False, slack=0):
    if identity:
        table, nbk = traces.identity_table(batch, shape.block_size)
        refcount = np.zeros(nbk, np.int32)
        s_, l_, p_ = kv.table_blocks(batch.seq_tok_off, table, shape.block_size)
        refcount[p_] = 1
        free = np.setdiff1d(np.arange(nbk, dtype=np.int32), p_).astype(np.int32)
        free_list = np.full(nbk, -1, np.int32)
        free_list[:free.size] = free
        fc = int(free.size)
    else:
        table, nbk, refcount, free_list, fc = traces.shuffled_table(batch, shape.block_size, seed, slack)
    return Workload(name, shape, batch, table, nbk, refcount, free_list, fc, seed, eta, tau_s,
                    default_tau_b(shape, eta) if tau_b is None else tau_b)


def tiny(eta: float = 0.0, seed: int = 0) -> Workload:
    """configs[0]: 1 x 512 tokens, N=2, h=2, d_h=64, d=16, 32 blocks, 8 steps, 2 duplicates."""
    return _paged("tiny", kv.TINY, traces.tiny_t0(), seed, eta, 0.8, 0.5, identity=True)


def c2(seed: int = 0, eta: float = 0.05, tau_s: float = 0.8) -> Workload:
    """configs[1]: DeepSeek-R1-Distill-Qwen-32B KV shape, 1 x 12,406 tokens (128 prompt)."""
    b = traces.make_batch(seed, 1, 12406, 128, kv.QWEN32B.block_size)
    return _paged("c2_qwen32b_1x12406", kv.QWEN32B, b, seed, eta, tau_s)


def c3(num_seqs: int = 64, seed: int = 0, eta: float = 0.05, tau_s: float = 0.8, first_seq: int = 0) -> Workload:
    """configs[2]: QwQ-32B KV shape, batch of 12,288-token CoTs (a slice of the 64 for waves)."""
    b = traces.make_batch(seed * 1000 + first_seq, num_seqs, 12288, 128, kv.QWEN32B.block_size)
    w = _paged(f"c3_qwq32b_{num_seqs}x12288", kv.QWEN32B, b, seed, eta, tau_s)
    w.first_seq = first_seq
    return w


def c5(num_seqs: int = 32, seed: int = 0, eta: float = 0.05, tau_s: float = 0.8, first_seq: int = 0) -> Workload:
    """configs[4]: 32B KV shape, 512 x 16,384-token CoTs across 8 GPUs = 64 per GPU, run as waves of
    32 (137 GB of KV per wave); this builds one wave (sequences first_seq .. first_seq + num_seqs)."""
    b = traces.make_batch(seed * 1000 + 500 + first_seq, num_seqs, 16384, 128, kv.QWEN32B.block_size)
    w = _paged(f"c5_32b_{num_seqs}x16384", kv.QWEN32B, b, seed, eta, tau_s)
    w.first_seq = first_seq
    return w


def c4(num_seqs: int = 128, seed: int = 0, eta: float = 0.05, tau_s: float = 0.8) -> Workload:
    """configs[3]: Phi-4-reasoning-plus KV shape, AIME-length traces L ~ U[8192, 16620]."""
    rng = np.random.default_rng(seed + 4)
    lengths = rng.integers(8192, 16621, num_seqs)
    b = traces.make_batch(seed, num_seqs, lengths, 128, kv.PHI4.block_size, vocab=traces.PHI4_VOCAB)
    return _paged(f"c4_phi4_{num_seqs}xaime", kv.PHI4, b, seed, eta, tau_s)


# ---------------------------------------------------------------------------- partitionable batches
# configs[2..4] are batches of independent sequences that the bench splits over GPUs and waves.
# Sequence i of a batch is generated from its own seed, so any subset (a rank's share, a wave) is
# the same sequences wherever it runs.
BATCHES = {
    # name: (BASELINE configs index, sequences, shape, vocab, length of sequence i, seed of sequence i)
    "c3": (2, 64, kv.QWEN32B, traces.QWEN_VOCAB, lambda seed, i: 12288, lambda seed, i: seed * 1000 + i),
    "c4": (3, 128, kv.PHI4, traces.PHI4_VOCAB,
           lambda seed, i: int(np.random.default_rng(seed + 4).integers(8192, 16621, 128)[i]),
           lambda seed, i: seed * 1000 + 200 + i),
    "c5": (4, 512, kv.QWEN32B, traces.QWEN_VOCAB, lambda seed, i: 16384, lambda seed, i: seed * 1000 + 500 + i),
}


def batch_traces(config: str, indices, seed: int = 0) -> traces.TraceBatch:
    """Token traces of sequences `indices` of batch `config` (128-token prompt each)."""
    _, _, shape, vocab, length, sseed = BATCHES[config]
    return traces.concat([traces.make_batch(sseed(seed, int(i)), 1, length(seed, int(i)), 128, shape.block_size,
                                            vocab=vocab) for i in indices])


def batch(config: str, indices, seed: int = 0, eta: float = 0.05, tau_s: float = 0.8) -> Workload:
    """Workload (trace, paged table, KV generator state) of sequences `indices` of batch `config`."""
    _, n, shape, _, _, _ = BATCHES[config]
    idx = [int(i) for i in indices]
    assert all(0 <= i < n for i in idx), idx
    w = _paged(f"{config}_{len(idx)}of{n}", shape, batch_traces(config, idx, seed), seed, eta, tau_s)
    w.indices = idx
    return w


def small(shape: kv.KVShape, num_seqs: int, length: int, seed: int = 0, eta: float = 0.05, tau_s: float = 0.8,
          gen_start: int = 64, **kw) -> Workload:
    """Parity-size workloads: several tiles and ragged tails, oracle-checkable in seconds."""
    b = traces.make_batch(seed, num_seqs, length, gen_start, shape.block_size, **kw)
    return _paged(f"small_{num_seqs}x{length}", shape, b, seed, eta, tau_s, slack=3)
