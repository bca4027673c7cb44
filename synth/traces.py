"""Seeded synthetic reasoning traces (token ids only).

Recipe ("Synthetic workload generator"):

* content tokens: Zipf(s=1.0) over the vocabulary minus the delimiter id(s),
  mapped through a fixed seeded permutation so frequent ids are not just small ids;
* a step = U[len_lo, len_hi] content tokens followed by one delimiter token
  (steps "separated by delimiters like \\n\\n");
* after the first step, with probability ``p_copy`` a step is a near-copy of a
  uniformly chosen earlier step, each token resampled with probability
  m ~ U(0, m_max) drawn per copy (planted redundancy);
* copies are phase-aligned with their source: the previous step is padded with
  ``(start_src - start_copy) mod d`` fresh tokens before its delimiter, so the
  copy's full blocks line up with the source's;
* a prompt of ``gen_start`` tokens precedes the generated part; the sequence is
  cut at ``n_tokens`` and marked final.

The paper's redundancy band (20-40 % of steps similar at cosine 0.8, 10-30 % at
0.9) calibrates ``p_copy`` and ``m_max``.

Nothing here computes a MemShare quantity; ground-truth labels (``copy_of``,
step start positions) are recorded for tests only.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

QWEN_VOCAB = 152_064
PHI4_VOCAB = 100_352


@dataclass
class TraceBatch:
    tokens: np.ndarray          # int32 [total tokens], sequences concatenated
    seq_tok_off: np.ndarray     # int64 [S+1]
    gen_start: np.ndarray       # int32 [S]
    final: np.ndarray           # uint8 [S]
    delim_ids: np.ndarray       # int32 [num delimiters]
    vocab: int
    # ground truth (tests only): per sequence, start position of each generated
    # step and the index of the earlier step it copies (-1 = fresh)
    step_starts: list = field(default_factory=list)
    copy_of: list = field(default_factory=list)

    @property
    def num_seqs(self) -> int:
        return int(self.gen_start.shape[0])

    def seq_tokens(self, s: int) -> np.ndarray:
        return self.tokens[self.seq_tok_off[s]:self.seq_tok_off[s + 1]]


class _Zipf:
    """Zipf(s) over ``vocab`` ids minus ``excluded`` via inverse-CDF lookup."""

    def __init__(self, vocab: int, excluded, s: float = 1.0, perm_seed: int = 0x5EED):
        ids = np.setdiff1d(np.arange(vocab, dtype=np.int64), np.asarray(excluded, dtype=np.int64))
        prng = np.random.Generator(np.random.PCG64(perm_seed))
        self.ids = prng.permutation(ids).astype(np.int32)
        w = 1.0 / np.power(np.arange(1, ids.size + 1, dtype=np.float64), s)
        self.cdf = np.cumsum(w)
        self.cdf /= self.cdf[-1]

    def draw(self, rng: np.random.Generator, n: int) -> np.ndarray:
        u = rng.random(n)
        r = np.searchsorted(self.cdf, u, side="right")
        r = np.minimum(r, self.ids.size - 1)
        return self.ids[r]


_ZIPF_CACHE: dict = {}


def _zipf(vocab, excluded, s):
    key = (vocab, tuple(int(x) for x in excluded), s)
    if key not in _ZIPF_CACHE:
        _ZIPF_CACHE[key] = _Zipf(vocab, excluded, s)
    return _ZIPF_CACHE[key]


def make_sequence(rng: np.random.Generator, n_tokens: int, gen_start: int, block_size: int,
                  vocab: int = QWEN_VOCAB, delim: int = 271, p_copy: float = 0.3,
                  m_max: float = 0.2, len_lo: int = 32, len_hi: int = 160,
                  zipf_s: float = 1.0, phase_align: bool = True):
    """One trace of exactly ``n_tokens`` ids. Returns (tokens, step_starts, copy_of)."""
    z = _zipf(vocab, [delim], zipf_s)
    toks = list(z.draw(rng, gen_start)) if gen_start > 0 else []
    contents: list[np.ndarray] = []
    starts: list[int] = []
    copy_of: list[int] = []
    pending_delim = False
    while True:
        is_copy = bool(contents) and rng.random() < p_copy
        if is_copy:
            src = int(rng.integers(len(contents)))
            m = rng.uniform(0.0, m_max)
            content = contents[src].copy()
            mask = rng.random(content.size) < m
            if mask.any():
                content[mask] = z.draw(rng, int(mask.sum()))
            if phase_align:
                # pad the previous step (before its delimiter) so that
                # start_copy == start_src (mod d)
                start_if_no_pad = len(toks) + 1
                pad = (starts[src] - start_if_no_pad) % block_size
                if pad:
                    padding = z.draw(rng, pad)
                    toks.extend(padding.tolist())
                    contents[-1] = np.concatenate([contents[-1], padding])
        else:
            src = -1
            content = z.draw(rng, int(rng.integers(len_lo, len_hi + 1)))
        if pending_delim:
            toks.append(delim)
        if len(toks) >= n_tokens:
            break
        starts.append(len(toks))
        copy_of.append(src)
        contents.append(content)
        toks.extend(content.tolist())
        pending_delim = True
        if len(toks) >= n_tokens:
            break
    arr = np.asarray(toks[:n_tokens], dtype=np.int32)
    # drop ground-truth steps that start at/after the cut
    keep = [i for i, s0 in enumerate(starts) if s0 < n_tokens]
    return arr, np.asarray([starts[i] for i in keep], np.int64), np.asarray([copy_of[i] for i in keep], np.int64)


def make_batch(seed: int, num_seqs: int, lengths, gen_start: int, block_size: int,
               vocab: int = QWEN_VOCAB, delim: int = 271, **kw) -> TraceBatch:
    """``num_seqs`` independent final traces; ``lengths`` is an int or a list."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if np.isscalar(lengths):
        lengths = [int(lengths)] * num_seqs
    seqs, starts, copies = [], [], []
    for s in range(num_seqs):
        t, st, cp = make_sequence(rng, int(lengths[s]), gen_start, block_size, vocab, delim, **kw)
        seqs.append(t)
        starts.append(st)
        copies.append(cp)
    off = np.zeros(num_seqs + 1, np.int64)
    off[1:] = np.cumsum([len(t) for t in seqs])
    return TraceBatch(tokens=np.concatenate(seqs) if seqs else np.zeros(0, np.int32),
                      seq_tok_off=off,
                      gen_start=np.full(num_seqs, gen_start, np.int32),
                      final=np.ones(num_seqs, np.uint8),
                      delim_ids=np.asarray([delim], np.int32), vocab=vocab,
                      step_starts=starts, copy_of=copies)


def concat(batches) -> TraceBatch:
    """The sequences of several batches (same vocabulary and delimiters) as one batch, in order."""
    toks = [b.tokens for b in batches]
    off = np.zeros(sum(b.num_seqs for b in batches) + 1, np.int64)
    lens = [int(b.seq_tok_off[i + 1] - b.seq_tok_off[i]) for b in batches for i in range(b.num_seqs)]
    off[1:] = np.cumsum(lens)
    return TraceBatch(tokens=np.concatenate(toks).astype(np.int32) if toks else np.zeros(0, np.int32),
                      seq_tok_off=off, gen_start=np.concatenate([b.gen_start for b in batches]).astype(np.int32),
                      final=np.concatenate([b.final for b in batches]).astype(np.uint8),
                      delim_ids=batches[0].delim_ids, vocab=batches[0].vocab,
                      step_starts=[x for b in batches for x in b.step_starts],
                      copy_of=[x for b in batches for x in b.copy_of])


def tiny_t0() -> TraceBatch:
    """The hand-built T0 fixture (SURVEY.md §8(d) "tiny (T0)"; BASELINE.json configs[0]).

    1 sequence, 512 tokens, gen_start 0, 8 steps of exactly 64 tokens
    (63 content + 1 delimiter) at [64k, 64k+64); steps 5 and 7 are exact copies
    of steps 1 and 3; fresh steps use disjoint id ranges, so every unrelated
    cosine is exactly 0.
    """
    delim = 1
    steps = []
    for k in range(8):
        src = {5: 1, 7: 3}.get(k, k)
        steps.append(np.arange(63, dtype=np.int32) + 100 * (src + 1))
    toks = np.concatenate([np.concatenate([c, np.asarray([delim], np.int32)]) for c in steps])
    return TraceBatch(tokens=toks.astype(np.int32), seq_tok_off=np.asarray([0, 512], np.int64),
                      gen_start=np.zeros(1, np.int32), final=np.ones(1, np.uint8),
                      delim_ids=np.asarray([delim], np.int32), vocab=QWEN_VOCAB,
                      step_starts=[np.arange(8, dtype=np.int64) * 64],
                      copy_of=[np.asarray([-1, -1, -1, -1, -1, 1, -1, 3], np.int64)])


def identity_table(batch: TraceBatch, block_size: int, max_blocks: int | None = None):
    """Block table with logical block i of sequence s at physical s*max_blocks+i (T0 uses it)."""
    nblk = [-(-int(batch.seq_tok_off[s + 1] - batch.seq_tok_off[s]) // block_size) for s in range(batch.num_seqs)]
    mb = max_blocks or max(nblk + [1])
    table = np.full((batch.num_seqs, mb), -1, np.int32)
    for s in range(batch.num_seqs):
        table[s, :nblk[s]] = s * mb + np.arange(nblk[s])
    return table, batch.num_seqs * mb


def shuffled_table(batch: TraceBatch, block_size: int, seed: int, slack: int = 0):
    """Paged table: every logical block gets a distinct physical block drawn from a
    seeded permutation (PagedAttention's non-contiguous placement).
    Returns (table int32 [S, max_blocks], num_blocks, refcount int32, free_list int32,
    free_count)."""
    nblk = [-(-int(batch.seq_tok_off[s + 1] - batch.seq_tok_off[s]) // block_size) for s in range(batch.num_seqs)]
    mb = max(nblk + [1])
    used = int(sum(nblk))
    num_blocks = used + slack
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x7AB1E))
    perm = rng.permutation(num_blocks).astype(np.int32)
    table = np.full((batch.num_seqs, mb), -1, np.int32)
    pos = 0
    for s in range(batch.num_seqs):
        table[s, :nblk[s]] = perm[pos:pos + nblk[s]]
        pos += nblk[s]
    refcount = np.zeros(num_blocks, np.int32)
    refcount[perm[:used]] = 1
    free_list = np.full(num_blocks, -1, np.int32)
    free_list[:slack] = perm[used:]
    return table, num_blocks, refcount, free_list, slack
