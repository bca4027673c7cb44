"""Pins for the oracle's candidate block-pair expansion (a4).

PAPER.md:267 ('their corresponding KV cache blocks'), :319-320 ('pairwise distances between
candidate blocks'); SPEC.md:265, :298 (fully-filled, i-th with i-th); readings R13, R14, R25.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _t0(pairing):
    b = traces.tiny_t0()
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    return oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.8, pairing=pairing)


def test_tiny_aligned_golden():
    g = json.load(open(os.path.join(GOLD, "tiny_t0.json")))
    r = _t0(oracle.ALIGNED)
    p = r["pairs"]
    assert [[int(a), int(b)] for a, b in zip(p["target_logical"], p["source_logical"])] == g["aligned_pairs"]
    assert r["target_off"].tolist() == list(range(9))
    m = r["matches"]
    assert [(int(a), int(b), float(c)) for a, b, c in zip(m["step"], m["cand_step"], m["cosine"])] == \
        [(x["step"], x["cand_step"], x["cosine"]) for x in g["matches"]]


def test_tiny_cross_golden():
    r = _t0(oracle.CROSS)
    p = r["pairs"]
    exp = [(t, s) for t in range(20, 24) for s in range(4, 8)] + [(t, s) for t in range(28, 32) for s in range(12, 16)]
    assert list(zip(p["target_logical"].tolist(), p["source_logical"].tolist())) == exp
    assert r["target_off"].tolist() == list(range(0, 33, 4))


def _full_blocks(a, b, d):
    return list(range(-(-a // d), b // d))


@pytest.mark.parametrize("seed", range(4))
def test_cross_all_candidates_equals_brute_enumeration(seed):
    """tau_s = -1: every earlier non-void step is a candidate, so CROSS pairs are exactly
    (full block of the current step) x (full block of an earlier non-void step)."""
    b = traces.make_batch(seed, 2, 1200, 40, 16, vocab=300, len_lo=10, len_hi=60)
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, -1.0, pairing=oracle.CROSS)
    exp = []
    for s in range(2):
        lo, hi = seg["seq_step_off"][s], seg["seq_step_off"][s + 1]
        st, en, nb = seg["step_start"][lo:hi], seg["step_end"][lo:hi], seg["step_nbag"][lo:hi]
        for k in range(hi - lo):
            if nb[k] == 0:
                continue
            srcs = sorted(x for j in range(k) if nb[j] > 0 for x in _full_blocks(st[j], en[j], 16))
            for t in _full_blocks(st[k], en[k], 16):
                exp += [(s, t, x) for x in srcs]
    p = r["pairs"]
    got = list(zip(p["seq"].tolist(), p["target_logical"].tolist(), p["source_logical"].tolist()))
    assert got == exp
    assert np.all(p["target_phys"] == tab[p["seq"], p["target_logical"]])
    assert np.all(p["source_phys"] == tab[p["seq"], p["source_logical"]])


def test_aligned_pairs_from_matches_brute():
    b = traces.make_batch(5, 1, 9000, 128, 16)
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.8)
    m, p = r["matches"], r["pairs"]
    exp = {}
    for k, j in zip(m["step"].tolist(), m["cand_step"].tolist()):
        fk = _full_blocks(seg["step_start"][k], seg["step_end"][k], 16)
        fj = _full_blocks(seg["step_start"][j], seg["step_end"][j], 16)
        for i in range(min(len(fk), len(fj))):
            exp.setdefault(fk[i], []).append(fj[i])
    got = {}
    for t, s_ in zip(p["target_logical"].tolist(), p["source_logical"].tolist()):
        got.setdefault(t, []).append(s_)
    assert got == {t: sorted(v) for t, v in exp.items()}
    assert sorted(got) == list(got)                    # targets ascending
    assert len(r["target_off"]) == len(got) + 1


def test_dedupe_by_physical_keeps_smallest_logical():
    # three identical steps of 32 content tokens + delim, phase aligned at 0, 48, 96 (d = 16)
    c = list(range(100, 132))
    pad = list(range(500, 515))
    toks = np.asarray(c + pad + [1] + c + pad + [1] + c + pad + [1], np.int32)
    seg = oracle.segment_steps(toks, [0, toks.size], [0], [1], [1])
    assert seg["step_start"].tolist() == [0, 48, 96]
    nblk = -(-toks.size // 16)
    tab = np.arange(nblk, dtype=np.int32)[None, :].copy()
    tab[0, 3] = tab[0, 0]                              # step 1's block 3 already shares step 0's block 0
    r = oracle.step_candidates(toks, [0, toks.size], seg, [1], tab, 16, 0.8)
    p = r["pairs"]
    rows = list(zip(p["target_logical"].tolist(), p["source_logical"].tolist(), p["source_phys"].tolist()))
    # target 6 (step 2, i = 0): sources logical 0 (phys 0) and 3 (phys 0 too) -> keep logical 0 only
    assert [x for x in rows if x[0] == 6] == [(6, 0, 0)]
    assert [x for x in rows if x[0] == 7] == [(7, 1, 1), (7, 4, 4)]
    # target 3 (step 1, i = 0) pairs with logical 0 whose phys equals its own (kept; D = 0)
    assert [x for x in rows if x[0] == 3] == [(3, 0, 0)]
