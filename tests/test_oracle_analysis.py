"""Pins for the oracle's f3/f4 analysis functions.

f4 similarity ratio: PAPER.md:121-126 (Fig. 2); SPEC.md:280-288 (all identical -> (n-1)/n,
pairwise disjoint -> 0). f3 all-pairs matrix: PAPER.md:142-145; SPEC.md:276-279 (symmetric,
zero diagonal, entry = direct call).
"""
import collections

import numpy as np
import pytest

import oracle
from synth import kv, traces


def _counts(tokens, tau, delim=1):
    t = np.asarray(tokens, np.int32)
    seg = oracle.segment_steps(t, [0, t.size], [0], [1], [delim])
    tab = np.zeros((1, max(1, t.size // 16 + 1)), np.int32)
    r = oracle.step_candidates(t, [0, t.size], seg, [delim], tab, 16, tau, top_k=1)
    return oracle.similarity_ratio_counts(r["matches"], 1)[0], seg["step_start"].size


def test_all_identical_steps():
    step = list(range(10, 30)) + [1]
    n_red, n = _counts(step * 6, 0.9)
    assert (n_red, n) == (5, 6)                    # (n-1)/n


def test_pairwise_disjoint_steps():
    toks = []
    for k in range(6):
        toks += list(range(100 * (k + 1), 100 * (k + 1) + 20)) + [1]
    assert _counts(toks, 0.0)[0] == 0               # 0.0 (cosine 0 is not > 0)


@pytest.mark.parametrize("seed", range(4))
def test_ratio_brute_force(seed):
    b = traces.make_batch(seed, 1, 3000, 0, 16, vocab=300, len_lo=8, len_hi=40)
    tau = 0.6
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, tau, top_k=1)
    got = oracle.similarity_ratio_counts(r["matches"], 1)[0]
    dl = set(b.delim_ids.tolist())
    vecs = [collections.Counter(int(x) for x in b.tokens[a:e] if int(x) not in dl)
            for a, e in zip(seg["step_start"], seg["step_end"])]
    exp = 0
    for k in range(1, len(vecs)):
        best = -1.0
        for j in range(k):
            if not vecs[k] or not vecs[j]:
                continue
            keys = set(vecs[k]) | set(vecs[j])
            a = np.array([vecs[k].get(x, 0) for x in keys], float)
            c = np.array([vecs[j].get(x, 0) for x in keys], float)
            best = max(best, float(a @ c / np.sqrt((a @ a) * (c @ c))))
        exp += best > tau
    assert got == exp


def test_all_pairs_matrix_properties():
    b = traces.tiny_t0()
    tab, nbk = traces.identity_table(b, 16)
    r = oracle.all_pairs(b.seq_tok_off, [0], [32], tab, 16)
    p = r["pairs"]
    assert p["seq"].size == 32 * 31 // 2 and r["target_off"].size == 32
    k, v, ls, bs = kv.host_pool(kv.TINY, nbk)
    s_, l_, pp_ = kv.table_blocks(b.seq_tok_off, tab, 16)
    kv.fill_blocks_host(k, v, ls, bs, kv.TINY, b.tokens, b.seq_tok_off, s_, l_, pp_, 0, 0.05)
    D = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, p["target_phys"], p["source_phys"])
    M = np.zeros((32, 32))
    M[p["target_logical"], p["source_logical"]] = D
    M = M + M.T
    Dt = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, p["source_phys"], p["target_phys"])
    assert np.array_equal(D, Dt)                                       # symmetric
    diag = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, np.arange(32), np.arange(32))
    assert np.all(diag == 0)                                           # zero diagonal
    i, j = 17, 5
    assert M[i, j] == oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, [i], [j])[0]   # = direct call
    # copies (steps 5, 7 of 1, 3) are the near-zero off-diagonal entries
    assert M[20, 4] < 0.2 and M[21, 4] > 1.0


def test_all_pairs_windows_and_partial_blocks():
    # 2 sequences: 200 tokens (12 full blocks) window [2, 20) -> 10 blocks; 40 tokens (2 full) window [0, 1) -> none
    tab = np.arange(26, dtype=np.int32).reshape(2, 13)
    r = oracle.all_pairs([0, 200, 240], [2, 0], [20, 1], tab, 16)
    assert r["pairs"]["seq"].size == 10 * 9 // 2 and r["target_off"].size == 10
    assert r["pairs"]["target_logical"].max() == 11 and r["pairs"]["source_logical"].min() == 2
