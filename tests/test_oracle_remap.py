"""Pins for the oracle's zero-copy remap (a7).

PAPER.md:276-278 ('simply updates the block table'), :283-284 (zero-copy)
(share_block examples), :395-401 (audit invariants); readings R23, R26.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import kv, traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dec(rows):
    """rows: (seq, target_logical, source_phys, accepted)"""
    a = np.asarray(rows, np.int64).reshape(-1, 4)
    return {"seq": a[:, 0], "target_logical": a[:, 1], "source_phys": a[:, 2], "accepted": a[:, 3]}


def fresh(nseq, nblk):
    tab = np.arange(nseq * nblk, dtype=np.int32).reshape(nseq, nblk)
    return tab, np.ones(nseq * nblk, np.int32), np.full(nseq * nblk, -1, np.int32)


def audit(tab, rc, fl, fc, num_blocks):
    """SPEC.md:395-397 refcount audit + no dangling + conservation, by brute-force recount."""
    cnt = np.bincount(tab[tab >= 0].ravel(), minlength=num_blocks)
    assert np.array_equal(cnt, rc)
    free = fl[:fc]
    assert len(set(free.tolist())) == fc
    assert np.all(rc[free] == 0)
    assert (rc > 0).sum() + fc == num_blocks


def test_spec_share_one_block():
    tab, rc, fl = fresh(2, 3)                 # two sequences, share 1 block
    st, tab2, rc2, fl2, fc, nf, af = oracle.remap(tab, rc, fl, 0, dec([(1, 0, 0, 1)]), 16)
    assert st == 0 and nf == 1 and fl2[0] == 3 and tab2[1, 0] == 0 and rc2[0] == 2 and af == 16
    assert (rc2 > 0).sum() == 5               # allocated -1
    # the same pair again is an idempotent no-op
    st, tab3, rc3, fl3, fc3, nf3, af3 = oracle.remap(tab2, rc2, fl2, fc, dec([(1, 0, 0, 1)]), 16)
    assert st == 0 and nf3 == 0 and af3 == 0 and np.array_equal(tab3, tab2) and np.array_equal(rc3, rc2)


def test_spec_chain_keeps_audit():
    # chain A->B then B->C stays consistent
    tab, rc, fl = fresh(3, 2)
    st, tab, rc, fl, fc, nf, _ = oracle.remap(tab, rc, fl, 0, dec([(1, 0, 0, 1)]), 16)
    st, tab, rc, fl, fc, nf, _ = oracle.remap(tab, rc, fl, fc, dec([(2, 0, tab[1, 0], 1)]), 16)
    assert st == 0
    audit(tab, rc, fl, fc, 6)
    assert tab[2, 0] == 0 and rc[0] == 3


def test_ten_logical_two_shared_stats():
    # 10 logical blocks, 2 shared -> allocated 8, affected ratio 0.2 at equal fill
    tab, rc, fl = fresh(1, 10)
    st, tab2, rc2, fl2, fc, nf, af = oracle.remap(tab, rc, fl, 0, dec([(0, 5, 0, 1), (0, 6, 1, 1)]), 16)
    assert (rc2 > 0).sum() == 8 and af / (10 * 16) == 0.2 and nf == 2


def test_rejected_decisions_change_nothing():
    tab, rc, fl = fresh(1, 4)
    st, tab2, rc2, fl2, fc, nf, af = oracle.remap(tab, rc, fl, 0, dec([(0, 2, 0, 0), (0, 3, 1, 0)]), 16)
    assert st == 0 and np.array_equal(tab2, tab) and np.array_equal(rc2, rc) and nf == 0 and af == 0


def test_increment_after_decrement_is_not_freed():
    """Reading R26: freed = decremented in this call AND final refcount 0. Target 4 moves to
    block 0 (block 4 decremented to 0), but target 8 then takes block 4 as its source: block 4
    ends at refcount 1 and must not be freed (it is referenced)."""
    tab, rc, fl = fresh(1, 12)
    st, tab2, rc2, fl2, fc, nf, af = oracle.remap(tab, rc, fl, 0, dec([(0, 4, 0, 1), (0, 8, 4, 1)]), 16)
    assert st == 0 and tab2[0, 4] == 0 and tab2[0, 8] == 4
    assert rc2[4] == 1 and rc2[8] == 0 and fl2[:fc].tolist() == [8]
    audit(tab2, rc2, fl2, fc, 12)


def test_free_list_order_is_last_decrement_order():
    tab, rc, fl = fresh(1, 8)
    tab[0, 6] = 5                       # blocks 5 referenced twice (logical 5 and 6)
    rc[5], rc[6] = 2, 0
    fl[0] = 6
    d = dec([(0, 1, 0, 1), (0, 5, 0, 1), (0, 6, 0, 1), (0, 7, 2, 1)])
    st, tab2, rc2, fl2, fc, nf, af = oracle.remap(tab, rc, fl, 1, d, 16)
    # block 1 freed by decision 0, block 5 by its LAST decrement (decision 2), block 7 by decision 3
    assert st == 0 and fl2[:fc].tolist() == [6, 1, 5, 7] and nf == 3 and af == 64
    audit(tab2, rc2, fl2, fc, 8)


def test_invalid_order_and_corruption():
    tab, rc, fl = fresh(1, 4)
    assert oracle.remap(tab, rc, fl, 0, dec([(0, 2, 0, 1), (0, 1, 0, 1)]), 16)[0] == oracle.INVALID
    assert oracle.remap(tab, rc, fl, 0, dec([(0, 2, 0, 1), (0, 2, 1, 1)]), 16)[0] == oracle.INVALID
    assert oracle.remap(tab, rc, fl, 0, dec([(0, 2, 9, 1)]), 16)[0] == oracle.CORRUPTION
    bad = rc.copy()
    bad[2] = 0                                  # table references block 2 but its count is 0
    assert oracle.remap(tab, bad, fl, 0, dec([(0, 2, 0, 1)]), 16)[0] == oracle.CORRUPTION


def test_tiny_t0_final_state_golden():
    g = json.load(open(os.path.join(GOLD, "tiny_t0.json")))
    b = traces.tiny_t0()
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    tab, nbk = traces.identity_table(b, 16)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, g["tau_s"])
    k, v, ls, bs = kv.host_pool(kv.TINY, nbk)
    s_, l_, p_ = kv.table_blocks(b.seq_tok_off, tab, 16)
    kv.fill_blocks_host(k, v, ls, bs, kv.TINY, b.tokens, b.seq_tok_off, s_, l_, p_, 0, 0.0)
    p = r["pairs"]
    D = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, p["target_phys"], p["source_phys"])
    best, acc, _ = oracle.select(D, r["target_off"], p["source_logical"], g["tau_b"])
    d = oracle.decisions(p, r["target_off"], D, best, acc)
    st, tab2, rc2, fl2, fc, nf, af = oracle.remap(tab, np.ones(nbk, np.int32), np.full(nbk, -1, np.int32), 0, d, 16)
    assert st == 0
    for t_, s_phys in g["final_table_changes"].items():
        assert tab2[0, int(t_)] == s_phys
    assert rc2[g["final_refcount_2"]].tolist() == [2] * 8 and rc2[g["final_refcount_0"]].tolist() == [0] * 8
    assert fl2[:fc].tolist() == g["free_list"] and nf == g["num_freed"] and af == g["affected_tokens"]
    assert (rc2 > 0).sum() == g["allocated_after"]


def _t1_chain():
    """T1 chain fixture: 3 steps of 64 tokens, steps 1 and 2 exact copies of
    step 0, eta = 0, tau_s = 0.8, tau_b = 0.5, tiny dims."""
    c = np.arange(63, dtype=np.int32) + 100
    toks = np.concatenate([c, [1], c, [1], c, [1]]).astype(np.int32)
    b = traces.TraceBatch(tokens=toks, seq_tok_off=np.array([0, 192]), gen_start=np.zeros(1, np.int32),
                          final=np.ones(1, np.uint8), delim_ids=np.array([1], np.int32), vocab=1000)
    tab, nbk = traces.identity_table(b, 16)
    k, v, ls, bs = kv.host_pool(kv.TINY, nbk)
    s_, l_, p_ = kv.table_blocks(b.seq_tok_off, tab, 16)
    kv.fill_blocks_host(k, v, ls, bs, kv.TINY, b.tokens, b.seq_tok_off, s_, l_, p_, 0, 0.0)
    return b, tab, nbk, (k, v, ls, bs)


def _round(b, tab, rc, fl, fc, pool, cur_mode, cb=None, ce=None):
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.8, cur_mode=cur_mode,
                               cur_begin=cb, cur_end=ce)
    p = r["pairs"]
    D = oracle.block_distance(*pool, 2, 2, 2, 64, 16, p["target_phys"], p["source_phys"])
    best, acc, _ = oracle.select(D, r["target_off"], p["source_logical"], 0.5)
    d = oracle.decisions(p, r["target_off"], D, best, acc)
    return r, oracle.remap(tab, rc, fl, fc, d, 16)


def test_t1_chain_online_and_offline_agree():
    b, tab, nbk, pool = _t1_chain()
    rc0, fl0 = np.ones(nbk, np.int32), np.full(nbk, -1, np.int32)
    # offline: one call, snapshot -> 4 + 8 pairs, all D = 0, ties -> smaller source logical
    r, (st, tabo, rco, flo, fco, nfo, afo) = _round(b, tab, rc0, fl0, 0, pool, oracle.CUR_ALL)
    assert r["pairs"]["seq"].size == 12 and st == 0
    # online: round 1 evaluates step 1, round 2 evaluates step 2 against the remapped table
    r1, (st, tab1, rc1, fl1, fc1, _, af1) = _round(b, tab, rc0, fl0, 0, pool, oracle.CUR_RANGE, [1], [2])
    r2, (st, tab2, rc2, fl2, fc2, _, af2) = _round(b, tab1, rc1, fl1, fc1, pool, oracle.CUR_RANGE, [2], [3])
    assert r2["matches"]["cand_step"].tolist() == [0, 1]            # both cos 1.0, ranked j ascending
    assert r2["pairs"]["seq"].size == 4                              # step 1's slots resolve to blocks 0..3
    for T_, R_, F_, A_ in ((tabo, rco, flo[:fco], afo), (tab2, rc2, fl2[:fc2], af1 + af2)):
        assert T_[0, 4:12].tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
        assert R_[0:4].tolist() == [3] * 4 and R_[4:12].tolist() == [0] * 8
        assert F_.tolist() == list(range(4, 12)) and A_ == 128


def test_randomized_audit_1e5_decisions():
    """a 10^5-operation randomized store audit."""
    rng = np.random.default_rng(0)
    nseq, nblk = 8, 64
    tab, rc, fl = fresh(nseq, nblk)
    fc, total = 0, 0
    while total < 100_000:
        n = int(rng.integers(1, 400))
        keys = np.unique(rng.integers(0, nseq * nblk, n))
        seqs, tls = keys // nblk, keys % nblk
        # sources: physical ids currently referenced by some table entry (a live block)
        live = tab.ravel()
        sp = live[rng.integers(0, live.size, keys.size)]
        acc = rng.random(keys.size) < 0.7
        st, tab, rc, fl, fc, nf, af = oracle.remap(tab, rc, fl, fc, dec(np.stack([seqs, tls, sp, acc], 1)), 16)
        assert st == 0
        audit(tab, rc, fl, fc, nseq * nblk)
        total += keys.size
