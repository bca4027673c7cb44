"""Pins for the oracle's bag-of-words cosine and Stage-1 filter (a2, a3).

PAPER.md:224-234 (Alg. 1 Stage 1), :254 (bag of words), :318 ('exceeding').
"""
import collections
import json
import os

import numpy as np
import pytest

import oracle
from synth import traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EX = json.load(open(os.path.join(GOLD, "spec_examples.json")))


@pytest.mark.parametrize("ex", EX["bag"], ids=lambda e: e["cite"][:30])
def test_bag_worked_examples(ex):
    ids, cnt, n2 = oracle.bag(ex["tokens"])
    assert ids.tolist() == ex["ids"] and cnt.tolist() == ex["counts"] and n2 == ex["n2"]


def test_bag_permutation_invariant_and_delims_excluded():
    a = oracle.bag([9, 5, 5, 1, 1])
    b = oracle.bag([5, 1, 9, 5, 1], delims=[1])
    assert a[0].tolist() == [1, 5, 9] and b[0].tolist() == [5, 9] and b[2] == 5


@pytest.mark.parametrize("ex", EX["cosine"], ids=lambda e: e["cite"][:30])
def test_cosine_worked_examples(ex):
    c = oracle.cosine_of_tokens(ex["a"], ex["b"])
    if "cos" in ex:
        assert c == ex["cos"]                      # exact: 1.0 and 0.0 are exact in IEEE
    else:
        assert c == ex["cos_num"] / ex["cos_den"]  # single correctly rounded quotient


def test_cosine_matches_dense_library_and_is_symmetric():
    rng = np.random.default_rng(1)
    for _ in range(200):
        a = rng.integers(0, 40, rng.integers(1, 80))
        b = rng.integers(0, 40, rng.integers(1, 80))
        va = np.bincount(a, minlength=40).astype(np.float64)
        vb = np.bincount(b, minlength=40).astype(np.float64)
        ref = va @ vb / (np.linalg.norm(va) * np.linalg.norm(vb))
        c = oracle.cosine_of_tokens(a, b)
        assert abs(c - ref) <= 4e-16 * max(1.0, ref)
        assert c == oracle.cosine_of_tokens(b, a)
        assert oracle.cosine_of_tokens(a, a) == 1.0


def _steps_tokens(tokens, steps, s, delims):
    lo, hi = steps["seq_step_off"][s], steps["seq_step_off"][s + 1]
    return [tokens[a:b] for a, b in zip(steps["step_start"][lo:hi], steps["step_end"][lo:hi])]


def _brute_candidates(step_toks, k, tau, delims):
    """Dense-vector brute force with Counter + numpy (independent of the oracle's sparse merge)."""
    def vec(t):
        return collections.Counter(int(x) for x in t if int(x) not in delims)
    vk = vec(step_toks[k])
    if not vk:
        return []
    out = []
    for j in range(k):
        vj = vec(step_toks[j])
        if not vj:
            continue
        keys = sorted(set(vk) | set(vj))
        a = np.array([vk.get(x, 0) for x in keys], np.float64)
        b = np.array([vj.get(x, 0) for x in keys], np.float64)
        c = float(a @ b / np.sqrt(float(a @ a) * float(b @ b)))
        if c > tau:
            out.append((c, j))
    out.sort(key=lambda x: (-x[0], x[1]))
    return out


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("tau", [0.8, 0.9, 0.3])
def test_stage1_brute_force(seed, tau):
    b = traces.make_batch(seed, 2, 2500, 64, 16, vocab=400, len_lo=8, len_hi=40)
    dl = set(b.delim_ids.tolist())
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, tau)
    m = r["matches"]
    for s in range(2):
        st = _steps_tokens(b.seq_tokens(s), seg, s, dl)
        for k in range(len(st)):
            exp = _brute_candidates(st, k, tau, dl)
            sel = (m["seq"] == s) & (m["step"] == k)
            got = list(zip(m["cosine"][sel].tolist(), m["cand_step"][sel].tolist()))
            assert [j for _, j in got] == [j for _, j in exp]
            assert np.allclose([c for c, _ in got], [c for c, _ in exp], rtol=0, atol=1e-15)
            assert m["rank"][sel].tolist() == list(range(len(got)))


def test_strict_threshold_at_exact_tie():
    # steps {a:2,b:1} then {a:2,c:1}: cosine exactly 0.8 (reading R10: strict '>')
    toks = np.asarray([10, 10, 11, 1, 10, 10, 12, 1], np.int32)
    seg = oracle.segment_steps(toks, [0, 8], [0], [1], [1])
    tab = np.arange(1, dtype=np.int32)[None, :]
    for tau, n in [(0.8, 0), (0.79, 1)]:
        r = oracle.step_candidates(toks, [0, 8], seg, [1], tab, 16, tau)
        assert r["matches"]["seq"].size == n
    r = oracle.step_candidates(toks, [0, 8], seg, [1], tab, 16, 0.79)
    assert r["matches"]["cosine"][0] == 0.8


def test_planted_exact_copies_always_candidates_and_modes():
    b = traces.make_batch(3, 1, 6000, 0, 16, m_max=0.0)
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.9)
    m = r["matches"]
    starts = seg["step_start"].tolist()
    for k, src in enumerate(b.copy_of[0]):
        if src < 0 or k >= len(starts):
            continue
        gk = starts.index(int(b.step_starts[0][k]))
        gj = starts.index(int(b.step_starts[0][src]))
        sel = (m["step"] == gk) & (m["cand_step"] == gj)
        assert sel.sum() == 1
    # tau_s = -1 and top_k = 0: every earlier non-void step is a candidate
    r_all = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, -1.0)
    S = seg["step_start"].size
    assert r_all["matches"]["seq"].size == S * (S - 1) // 2
    # LAST mode == the ALL-mode matches of the last step
    r_last = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.5,
                                    cur_mode=oracle.CUR_LAST)
    r_a = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.5)
    sel = r_a["matches"]["step"] == S - 1
    assert r_last["matches"]["cand_step"].tolist() == r_a["matches"]["cand_step"][sel].tolist()
    # RANGE mode == the ALL-mode matches restricted to the range
    r_rng = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.5,
                                   cur_mode=oracle.CUR_RANGE, cur_begin=[5], cur_end=[20])
    sel = (r_a["matches"]["step"] >= 5) & (r_a["matches"]["step"] < 20)
    assert r_rng["matches"]["cand_step"].tolist() == r_a["matches"]["cand_step"][sel].tolist()


def test_monotone_in_tau_and_topk_prefix():
    b = traces.make_batch(11, 1, 8000, 0, 16)
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, _ = traces.identity_table(b, 16)

    def mset(tau, k=0):
        m = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, tau, top_k=k)["matches"]
        return m
    lo, hi = mset(0.5), mset(0.9)
    s_lo = set(zip(lo["step"].tolist(), lo["cand_step"].tolist()))
    s_hi = set(zip(hi["step"].tolist(), hi["cand_step"].tolist()))
    assert s_hi <= s_lo
    capped = mset(0.1, 2)
    full = mset(0.1)
    for k in np.unique(full["step"]):
        f = full["cand_step"][full["step"] == k].tolist()
        c = capped["cand_step"][capped["step"] == k].tolist()
        assert c == f[:2]


def test_similarity_ratio_in_paper_band():
    """20-40 % of steps similar at 0.8, 10-30 % at 0.9 -- the generator's
    calibration target (a property of the INPUT recipe, checked through the oracle)."""
    r8, r9 = [], []
    for seed in range(5):
        b = traces.make_batch(seed, 1, 12406, 128, 16)
        seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
        tab, _ = traces.identity_table(b, 16)
        S = seg["step_start"].size
        for tau, acc in ((0.8, r8), (0.9, r9)):
            m = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, tau)["matches"]
            acc.append(np.unique(m["step"]).size / S)
    assert 0.2 <= np.mean(r8) <= 0.4, r8
    assert 0.1 <= np.mean(r9) <= 0.3, r9
