"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): segmentation, candidate sets, block pairs, remaps, refcounts and
free lists bit-exact; cosines bit-exact (one IEEE expression on both sides, reading R12);
distances within 1e-5 relative (exactly 0 for identical blocks); decisions identical except
targets within 1e-4 relative of tau_b or with a near tie, which are reported.
"""
import numpy as np
import pytest

import oracle
from synth import kv, traces, workloads

from _gpu_util import (assert_candidates_equal, assert_steps_equal, compare_decisions, compare_distances,
                       host_pool_from_device, make_path, oracle_candidates, oracle_steps)

pytestmark = pytest.mark.gpu

SMALL = kv.KVShape(8, 4, 64, 16)       # several tiles per slice, quick oracle


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_21433_b200 import build
    build.build()


def full_parity(w, tau_s=None, tau_b=None, top_k=0, pairing=oracle.ALIGNED, cur_mode=oracle.CUR_ALL, cb=None, ce=None,
                fused=False):
    """One round through the four calls (fused=True: a5-a7 through memshare_block_distance_remap)."""
    import torch
    p = make_path(w)
    tau_s = w.tau_s if tau_s is None else tau_s
    tau_b = w.tau_b if tau_b is None else tau_b
    p.autosize(tau_s, top_k, pairing, cur_mode, cb, ce)
    p.segment()
    p.candidates(tau_s, top_k, pairing, cur_mode, cb, ce)
    if fused:
        p.distance_remap(tau_b)
    else:
        p.distance_call(tau_b)
        p.remap()
    torch.cuda.synchronize()
    return check_round(p, w, tau_s, tau_b, top_k, pairing, cur_mode, cb, ce)


def check_round(p, w, tau_s, tau_b, top_k=0, pairing=oracle.ALIGNED, cur_mode=oracle.CUR_ALL, cb=None, ce=None):
    """Every output of one completed round on path `p` (started from w's pristine state) against the oracle."""
    assert p.read_status() == 0
    st = oracle_steps(w)
    assert_steps_equal(p.read_steps(), st)
    oc = oracle_candidates(w, st, tau_s, top_k, pairing, cur_mode, cb, ce)
    gc = p.read_candidates()
    assert_candidates_equal(gc, oc)
    kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
    sh = w.shape
    pr = oc["pairs"]
    D = oracle.block_distance(kh, vh, p.pool.layer_stride, p.pool.block_stride, sh.num_layers, sh.num_kv_heads,
                              sh.num_kv_heads, sh.head_dim, sh.block_size, pr["target_phys"], pr["source_phys"])
    gd = p.read_distance()
    compare_distances(gd["distance"], D)
    assert np.array_equal(gd["under"].astype(bool), gd["distance"] < np.float32(tau_b))
    near = compare_decisions(gd["decisions"], gd["distance"], D, oc["target_off"], pr, tau_b)
    # remap parity on the GPU's own decisions (identical inputs to both sides)
    s = p.read_state()
    st_o, tab, rc, fl, fc, nf, af = oracle.remap(w.table, w.refcount, w.free_list, w.free_count, gd["decisions"],
                                                 sh.block_size)
    assert st_o == 0
    assert np.array_equal(s["table"], tab) and np.array_equal(s["refcount"], rc)
    assert np.array_equal(s["free_list"], fl) and s["free_count"] == fc
    assert s["num_freed"] == nf and s["affected"] == af
    return p, oc, D, near


@pytest.mark.parametrize("eta", [0.0, 0.05])
def test_tiny_t0(eta):
    import json
    import os
    w = workloads.tiny(eta=eta)
    p, oc, D, near = full_parity(w)
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tiny_t0.json")))
    if eta == 0.0:
        s = p.read_state()
        assert s["free_list"][:s["free_count"]].tolist() == g["free_list"]
        assert s["affected"] == g["affected_tokens"]


def _t1_chain_workload(extra_copies=0):
    """SURVEY.md §8(c.3) T1 chain fixture: tiny dims, one sequence of 3 (+ extra_copies) steps of
    64 tokens, every step after the first an exact copy of step 0, eta = 0 (identical blocks: all
    D == 0 exactly), tau_s = 0.8, tau_b = 0.5, identity table."""
    c = np.arange(63, dtype=np.int32) + 100
    n_steps = 3 + extra_copies
    toks = np.concatenate([np.concatenate([c, [1]]) for _ in range(n_steps)]).astype(np.int32)
    b = traces.TraceBatch(tokens=toks, seq_tok_off=np.array([0, toks.size]), gen_start=np.zeros(1, np.int32),
                          final=np.ones(1, np.uint8), delim_ids=np.array([1], np.int32), vocab=1000)
    return workloads._paged("t1_chain", kv.TINY, b, 0, 0.0, 0.8, 0.5, identity=True)


def test_t1_chain_exact_ties_offline_and_online():
    """Exact D == 0 ties (reading R22: ties -> the smaller source logical), asserted exactly.
    Offline (one ALL call, snapshot): 4 + 8 pairs, all D == 0; each target of step 2 has two tied
    sources (blocks of step 0 and step 1) and must take step 0's. Online (two RANGE rounds, the
    second on the remapped table): round 2's two candidate steps resolve to the same physical
    blocks, so the dedupe keeps 4 pairs. Both end in table[4..11] = [0,1,2,3,0,1,2,3],
    rc[0..3] = 3, rc[4..11] = 0, free list [4..11], affected 128 (hand-computed)."""
    import torch
    w = _t1_chain_workload()
    p, oc, D, (near_thr, near_tie) = full_parity(w)
    assert oc["pairs"]["seq"].size == 12 and np.all(D == 0.0)
    gd = p.read_distance()
    assert np.all(gd["distance"] == 0.0)
    assert near_tie == 0 and near_thr == 0
    assert gd["decisions"]["source_logical"].tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
    s = p.read_state()
    assert s["table"][0, 4:12].tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
    assert s["refcount"][0:4].tolist() == [3] * 4 and s["refcount"][4:12].tolist() == [0] * 8
    assert s["free_list"][s["free_count"] - 8:s["free_count"]].tolist() == list(range(4, 12))
    assert s["affected"] == 128
    # online: round 1 = step 1, round 2 = step 2 on the state round 1 left
    q = make_path(w)
    q.autosize(w.tau_s, cur_mode=oracle.CUR_RANGE, cur_begin=[1], cur_end=[3])
    fc0 = q.read_state()["free_count"]
    aff = 0
    for k in (1, 2):
        q.round(w.tau_s, w.tau_b, cur_mode=oracle.CUR_RANGE, cur_begin=[k], cur_end=[k + 1])
        torch.cuda.synchronize()
        assert q.read_status() == 0
        aff += q.read_state()["affected"]
        if k == 2:
            c2 = q.read_candidates()
            assert c2["matches"]["cand_step"].tolist() == [0, 1]      # both cos 1.0, ranked j ascending
            assert c2["pairs"]["seq"].size == 4                       # step 1's slots resolve to blocks 0..3
            assert c2["pairs"]["source_logical"].tolist() == [0, 1, 2, 3]
    s = q.read_state()
    assert s["table"][0, 4:12].tolist() == [0, 1, 2, 3, 0, 1, 2, 3]
    assert s["refcount"][0:4].tolist() == [3] * 4 and s["refcount"][4:12].tolist() == [0] * 8
    assert s["free_list"][fc0:s["free_count"]].tolist() == list(range(4, 12)) and aff == 128


@pytest.mark.parametrize("extra", [2, 40])
def test_exact_ties_many_duplicate_sources(extra):
    """A chain of 5 / 43 identical steps offline: the last step's targets have 4 / 42 exact
    D == 0 sources; every target must pick the smallest source logical (reading R22), checked by
    compare_decisions' exact-zero rule and directly."""
    w = _t1_chain_workload(extra_copies=extra)
    p, oc, D, (near_thr, near_tie) = full_parity(w)
    assert np.all(D == 0.0) and near_tie == 0
    dec = p.read_distance()["decisions"]
    assert np.all(dec["source_logical"] == dec["target_logical"] % 4)
    assert np.diff(oc["target_off"]).max() == 2 + extra


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_small_shape_pipeline(seed):
    w = workloads.small(SMALL, 3, 5000 + 777 * seed, seed=seed)
    full_parity(w)


@pytest.mark.parametrize("tau_s,top_k,pairing", [(0.9, 0, oracle.ALIGNED), (0.5, 2, oracle.ALIGNED),
                                                 (0.8, 0, oracle.CROSS), (-1.0, 0, oracle.ALIGNED),
                                                 (0.3, 3, oracle.CROSS)])
def test_stage1_and_pair_variants(tau_s, top_k, pairing):
    w = workloads.small(SMALL, 2, 2500, seed=7)
    full_parity(w, tau_s=tau_s, top_k=top_k, pairing=pairing)


@pytest.mark.parametrize("seed", range(24))
def test_randomized_configurations(seed):
    """Seeded fuzz over the parameter space: KV shapes (incl. 10 heads, block sizes 8 / 32),
    pairing, tau_s, top_k and call granularity, each through the full parity check."""
    rng = np.random.default_rng(1000 + seed)
    shape = [kv.KVShape(2, 2, 64, 16), kv.KVShape(3, 10, 128, 16), kv.KVShape(4, 8, 128, 8),
             kv.KVShape(2, 4, 64, 32)][seed % 4]
    num_seqs = int(rng.integers(1, 4))
    length = int(rng.integers(700, 2600))
    w = workloads.small(shape, num_seqs, length, seed=seed, gen_start=int(rng.integers(0, 200)))
    pairing = [oracle.ALIGNED, oracle.CROSS][int(rng.integers(0, 2))]
    tau_s = float(rng.choice([0.3, 0.6, 0.8, 0.95]))
    top_k = int(rng.choice([0, 0, 1, 3]))
    mode = int(rng.integers(0, 3))
    if mode == 2:
        cb = [int(x) for x in rng.integers(0, 6, num_seqs)]
        ce = [b + int(x) for b, x in zip(cb, rng.integers(1, 12, num_seqs))]
        full_parity(w, tau_s=tau_s, top_k=top_k, pairing=pairing, cur_mode=oracle.CUR_RANGE, cb=cb, ce=ce,
                    fused=seed % 2 == 1)
    else:
        full_parity(w, tau_s=tau_s, top_k=top_k, pairing=pairing, cur_mode=[oracle.CUR_ALL, oracle.CUR_LAST][mode],
                    fused=seed % 2 == 1)


@pytest.mark.parametrize("shape", [kv.KVShape(2, 3, 64, 16), kv.KVShape(2, 12, 128, 16), kv.KVShape(2, 20, 128, 16),
                                   kv.KVShape(3, 1, 8, 16), kv.KVShape(2, 9, 128, 16)])
def test_stage_geometries(shape):
    """Slice sizes off the configs' grid: 6 KiB and 256 B (not 4 KiB multiples: generic kernel),
    48 KiB (two 24 KiB stages), 80 KiB (two 40 KiB stages), 36 KiB (one 36 KiB stage)."""
    w = workloads.small(shape, 2, 1800, seed=shape.num_kv_heads)
    full_parity(w, tau_s=0.6, pairing=oracle.CROSS)
    full_parity(w)


@pytest.mark.parametrize("case", ["empty", "clamped", "all_steps", "mixed"])
def test_range_round_work_items(case):
    """RANGE rounds take the current steps as work items (a dense list built by the encode kernel;
    zeros published for every other step): all-empty ranges (no item: the totals are written
    directly), ranges beyond the step counts and negative begins (clamped as the oracle does),
    ranges covering every step (= the offline round), and a mix -- each the full oracle check,
    with the 8-CTA clusters of few sequences and one CTA per item for many."""
    w = workloads.small(SMALL, 3, 2600, seed=9)
    S = np.diff(oracle_steps(w)["seq_step_off"])
    if case == "empty":
        cb, ce = [3, 0, 7], [3, 0, 7]
    elif case == "clamped":
        cb, ce = [-5, int(S[1]) - 2, int(S[2]) + 3], [2, int(S[1]) + 40, int(S[2]) + 9]
    elif case == "all_steps":
        cb, ce = [0, 0, 0], [int(x) for x in S]
    else:
        cb, ce = [1, 0, 5], [2, 0, int(S[2])]
    p, oc, D, near = full_parity(w, tau_s=0.5, cur_mode=oracle.CUR_RANGE, cb=cb, ce=ce)
    if case == "empty":
        assert p.counts()["matches"] == 0 and p.counts()["pairs"] == 0
    if case == "all_steps":
        ref = oracle_candidates(w, oracle_steps(w), 0.5)             # the offline (ALL) round
        assert_candidates_equal(p.read_candidates(), ref)
    w2 = workloads.small(SMALL, 100, 300, seed=10)                     # many sequences: one CTA per item
    S2 = np.diff(oracle_steps(w2)["seq_step_off"])
    full_parity(w2, tau_s=0.5, cur_mode=oracle.CUR_RANGE, cb=[0] * 100, ce=[int(min(x, 2)) for x in S2])


def test_online_modes():
    """LAST with 3 sequences runs Stage 1 as 8-CTA clusters per current step (DSMEM sum of the
    ranks' partial dots); RANGE runs one CTA per step."""
    w = workloads.small(SMALL, 3, 3000, seed=3)
    full_parity(w, cur_mode=oracle.CUR_LAST)
    full_parity(w, cur_mode=oracle.CUR_RANGE, cb=[0, 5, 10], ce=[4, 30, 11])


@pytest.mark.parametrize("num_seqs", [20, 40, 100])
def test_online_last_cluster_sizes(num_seqs):
    """LAST rounds over many sequences: Stage-1 clusters of 4, 2 and 1 CTAs per current step."""
    w = workloads.small(SMALL, num_seqs, 900, seed=num_seqs, gen_start=16)
    full_parity(w, tau_s=0.5, cur_mode=oracle.CUR_LAST)


def test_qwen32b_shape_two_sequences():
    w = workloads.small(kv.QWEN32B, 2, 3100, seed=11, gen_start=128)
    full_parity(w)


def test_phi4_shape_ten_consumer_warps():
    """Phi-4's 40 KiB slice is one stage for ten consumer warps (8 chunks each); a 10-head slice of
    head_dim 64 (20 KiB) and an 80 KiB slice (two 40 KiB stages, eight warps) around it."""
    w = workloads.small(kv.PHI4, 1, 3300, seed=5, gen_start=128, vocab=traces.PHI4_VOCAB)
    full_parity(w)
    full_parity(w, tau_s=0.5, pairing=oracle.CROSS)
    for shape in (kv.KVShape(2, 10, 64, 16), kv.KVShape(2, 10, 128, 32)):
        full_parity(workloads.small(shape, 2, 1800, seed=6))


@pytest.mark.parametrize("cur_mode", [oracle.CUR_ALL, oracle.CUR_LAST])
def test_bit_reproducible_rounds(cur_mode):
    """memshare.h: outputs are bit-reproducible run to run -- the same round twice (dynamic work
    tickets, look-back, cluster reductions and atomics notwithstanding) gives identical matches,
    pairs, distances, decisions and table state."""
    import torch
    w = workloads.small(kv.QWEN32B, 2, 2600, seed=8, gen_start=64)
    outs = []
    for _ in range(2):
        p = make_path(w)
        p.autosize(0.6, pairing=oracle.CROSS, cur_mode=cur_mode)
        p.round(0.6, w.tau_b, pairing=oracle.CROSS, cur_mode=cur_mode)
        torch.cuda.synchronize()
        assert p.read_status() == 0
        c, d, st = p.read_candidates(), p.read_distance(), p.read_state()
        outs.append((c, d, st))
        del p
    (c0, d0, s0), (c1, d1, s1) = outs
    assert c0["pairs"]["seq"].size > 0
    for k in c0["matches"]:
        assert np.array_equal(c0["matches"][k], c1["matches"][k]), k
    for k in c0["pairs"]:
        assert np.array_equal(c0["pairs"][k], c1["pairs"][k]), k
    assert np.array_equal(d0["distance"].view(np.uint32), d1["distance"].view(np.uint32))
    for k in d0["decisions"]:
        assert np.array_equal(d0["decisions"][k], d1["decisions"][k]), k
    for k in ("table", "refcount", "free_list"):
        assert np.array_equal(s0[k], s1[k]), k


def _round_outputs(p):
    c, d, st = p.read_candidates(), p.read_distance(), p.read_state()
    return c, d, st


@pytest.mark.parametrize("case", ["tiny0", "tiny5", "chain", "small", "cross", "phi4", "geom", "two_rounds"])
def test_fused_distance_remap_matches_separate_calls(case):
    """memshare_block_distance_remap (a5-a7 in one call: the remap run by the finalisation kernel's
    last CTA) against
    memshare_block_distance + memshare_remap on the same round: distances, under flags, decisions,
    table, refcounts, free list and counters bit-identical, and the fused round passes the full
    oracle check."""
    import torch
    tau_s, pairing, rounds = None, oracle.ALIGNED, 1
    if case in ("tiny0", "tiny5"):
        w = workloads.tiny(eta=0.0 if case == "tiny0" else 0.05)
    elif case == "chain":
        w = _t1_chain_workload(extra_copies=5)
    elif case == "small":
        w = workloads.small(SMALL, 3, 2500, seed=3)
    elif case == "cross":
        w, tau_s, pairing = workloads.small(SMALL, 2, 2500, seed=7), 0.3, oracle.CROSS
    elif case == "phi4":
        w = workloads.small(kv.PHI4, 1, 3300, seed=5, gen_start=128, vocab=traces.PHI4_VOCAB)
    elif case == "geom":
        w, tau_s, pairing = workloads.small(kv.KVShape(2, 3, 64, 16), 2, 1800, seed=3), 0.6, oracle.CROSS
    else:
        w, rounds = workloads.small(SMALL, 2, 2500, seed=11, eta=0.0), 2
    tau_s = w.tau_s if tau_s is None else tau_s
    tau_b = 1e-3 if case == "two_rounds" else w.tau_b
    outs = []
    for fused in (False, True):
        p = make_path(w)
        p.autosize(tau_s, pairing=pairing)
        for _ in range(rounds):
            p.segment()
            p.candidates(tau_s, pairing=pairing)
            if fused:
                p.distance_remap(tau_b)
            else:
                p.distance_call(tau_b)
                p.remap()
        torch.cuda.synchronize()
        assert p.read_status() == 0
        outs.append(_round_outputs(p))
        if fused and rounds == 1:
            check_round(p, w, tau_s, tau_b, pairing=pairing)
        del p
    (c0, d0, s0), (c1, d1, s1) = outs
    assert c0["pairs"]["seq"].size > 0
    assert np.array_equal(d0["distance"].view(np.uint32), d1["distance"].view(np.uint32))
    assert np.array_equal(d0["under"], d1["under"])
    for k in d0["decisions"]:
        assert np.array_equal(d0["decisions"][k], d1["decisions"][k]), k
    for k in ("table", "refcount", "free_list", "free_count", "num_freed", "affected"):
        assert np.array_equal(s0[k], s1[k]), k


def test_fused_distance_remap_rejects_bad_decisions_like_remap():
    """A remap validation failure in the fused call changes nothing (as memshare_remap): a
    corrupted block table entry makes the fused call report CORRUPTION and leave the state."""
    import torch
    w = workloads.small(SMALL, 2, 2500, seed=3)
    p = make_path(w)
    p.autosize(w.tau_s)
    p.segment()
    p.candidates(w.tau_s)
    torch.cuda.synchronize()
    d = p.read_candidates()
    tgt = d["pairs"]
    assert tgt["seq"].size > 0
    s, tl = int(tgt["seq"][0]), int(tgt["target_logical"][0])
    p.table.view(p.num_seqs, p.table_stride)[s, tl] = p.num_blocks + 5     # out of range: CORRUPTION
    before = p.read_state()
    p.distance_remap(1e9)                                                   # every decision accepted
    torch.cuda.synchronize()
    assert p.read_status() == 3
    after = p.read_state()
    for k in ("table", "refcount", "free_list"):
        assert np.array_equal(before[k], after[k]), k


@pytest.mark.parametrize("pairing,tau_s", [(oracle.ALIGNED, 0.5), (oracle.CROSS, 0.3)])
def test_second_round_on_shared_blocks(pairing, tau_s):
    """A round on the state a previous round left: after the zero-copy remap
    several logical blocks share one physical block, so a target's source slots repeat physical
    blocks and only the first slot of each is kept (the dedup; R25, oracle_step_candidates). Round 2 is compared in
    full with the oracle run on round 1's table, refcounts and free list; CROSS at a low tau_s gives
    targets with more than 32 source slots (the dedup across 32-slot windows)."""
    import torch
    w = workloads.small(SMALL, 2, 2500, seed=11, eta=0.0)
    p = make_path(w)
    tau_b = 1e-3                                 # eta = 0: planted copies are exact (D = 0), all accepted
    p.autosize(tau_s, pairing=pairing, slack=1.0)
    p.round(tau_s, tau_b, pairing=pairing)
    torch.cuda.synchronize()
    assert p.read_status() == 0
    s1 = p.read_state()
    assert s1["num_freed"] > 0 and (s1["refcount"] > 1).any()
    p.round(tau_s, tau_b, pairing=pairing)      # round 2 on the remapped state
    torch.cuda.synchronize()
    assert p.read_status() == 0
    st = oracle_steps(w)
    assert_steps_equal(p.read_steps(), st)
    oc = oracle_candidates(w, st, tau_s, 0, pairing, table=s1["table"])
    assert_candidates_equal(p.read_candidates(), oc)
    # the dedup did drop slots: the same matches on a table without shared blocks give more pairs
    uniq = np.arange(s1["table"].size, dtype=np.int32).reshape(s1["table"].shape)
    ou = oracle_candidates(w, st, tau_s, 0, pairing, table=uniq)
    assert ou["pairs"]["seq"].size > oc["pairs"]["seq"].size
    if pairing == oracle.CROSS:                  # targets with more than 32 source slots
        assert np.diff(ou["target_off"]).max() > 32
    kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
    sh = w.shape
    pr = oc["pairs"]
    D = oracle.block_distance(kh, vh, p.pool.layer_stride, p.pool.block_stride, sh.num_layers, sh.num_kv_heads,
                              sh.num_kv_heads, sh.head_dim, sh.block_size, pr["target_phys"], pr["source_phys"])
    gd = p.read_distance()
    compare_distances(gd["distance"], D)
    compare_decisions(gd["decisions"], gd["distance"], D, oc["target_off"], pr, tau_b)
    s2 = p.read_state()
    st_o, tab, rc, fl, fc, nf, af = oracle.remap(s1["table"], s1["refcount"], s1["free_list"], s1["free_count"],
                                                 gd["decisions"], sh.block_size)
    assert st_o == 0
    assert np.array_equal(s2["table"], tab) and np.array_equal(s2["refcount"], rc)
    assert np.array_equal(s2["free_list"], fl) and s2["free_count"] == fc and s2["num_freed"] == nf


def test_degenerate_rounds():
    """Rounds with nothing to share: tau_s = 1.0 (strict 'exceeding' can never hold) gives no
    match, no pair, no target -- the distance call and the remap are no-ops and the table,
    refcounts and free list come back unchanged; a trace without any delimiter has no finished
    step unless it is final."""
    import torch
    w = workloads.small(SMALL, 2, 2000, seed=3)
    p = make_path(w)
    s0 = p.read_state()
    p.round(1.0, w.tau_b)
    torch.cuda.synchronize()
    assert p.read_status() == 0
    assert p.counts()["pairs"] == 0 and p.counts()["targets"] == 0 and p.counts()["matches"] == 0
    s1 = p.read_state()
    for k in ("table", "refcount", "free_list"):
        assert np.array_equal(s0[k], s1[k]), k
    assert s1["num_freed"] == 0 and s1["affected"] == 0 and s1["free_count"] == s0["free_count"]
    # no delimiter at all: one step per FINAL sequence, none for an open one
    b = w.batch
    toks = np.full(3000, 7, np.int32)
    off = np.asarray([0, 1500, 3000], np.int64)
    for fin in ([1, 0], [0, 0]):
        exp = oracle.segment_steps(toks, off, np.zeros(2, np.int32), np.asarray(fin, np.uint8), b.delim_ids)
        assert exp["seq_step_off"][-1] == sum(fin)
        pp = MemSharePathFor(toks, off, fin, b.delim_ids, w)
        pp.segment()
        pp.candidates(-1.0)
        torch.cuda.synchronize()
        assert pp.read_status() == 0 and pp.counts()["steps"] == sum(fin) and pp.counts()["pairs"] == 0


def MemSharePathFor(toks, off, fin, delims, w):
    from paper_2507_21433_b200.pipeline import MemSharePath
    S = off.size - 1
    nb = int(sum(-(-(off[i + 1] - off[i]) // 16) for i in range(S)))
    table = np.arange(nb, dtype=np.int32).reshape(S, -1) if nb % S == 0 else None
    assert table is not None
    rc = np.ones(nb, np.int32)
    fl = np.full(nb, -1, np.int32)
    return MemSharePath(toks, off, np.zeros(S, np.int32), np.asarray(fin, np.uint8), delims, table, rc, fl, 0, None,
                        None, 0, 0, nb, SMALL.num_layers, SMALL.num_kv_heads, SMALL.num_kv_heads, SMALL.head_dim,
                        SMALL.block_size)


def test_segment_edge_cases():
    """Ragged, empty, non-final, prompt-only, delimiter-only, multi-delimiter and multi-tile
    sequences, against the oracle."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    rng = np.random.default_rng(0)
    seqs = [np.zeros(0, np.int32), np.asarray([5], np.int32), np.asarray([1, 1, 1], np.int32),
            rng.choice([1, 2, 3, 4, 9], 20000, p=[0.05, 0.02, 0.31, 0.31, 0.31]).astype(np.int32),
            rng.choice([1, 3, 4], 4097, p=[0.3, 0.35, 0.35]).astype(np.int32),
            np.asarray([3, 3, 1, 4, 1], np.int32)]
    toks = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum([s.size for s in seqs])]).astype(np.int64)
    gs = np.asarray([0, 0, 1, 100, 0, 9], np.int32)
    fin = np.asarray([1, 0, 1, 1, 0, 0], np.uint8)
    delims = np.asarray([1, 2], np.int32)
    exp = oracle.segment_steps(toks, off, gs, fin, delims)
    dev = torch.device("cuda")
    S = len(seqs)
    cap = toks.size
    out = [torch.full((cap,), -7, dtype=torch.int32, device=dev) for _ in range(3)]
    sso = torch.zeros(S + 1, dtype=torch.int64, device=dev)
    ws = torch.empty(L.segment_steps_workspace_size(toks.size, S, cap), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    t = lambda a, dt: torch.as_tensor(a, dtype=dt, device=dev)
    rc = L.segment_steps(t(toks, torch.int32), toks.size, t(off, torch.int64), t(gs, torch.int32), t(fin, torch.uint8), S,
                         delims, out[0], out[1], out[2], sso, cap, ws, status)
    assert rc == 0
    torch.cuda.synchronize()
    n = int(sso[-1])
    assert status.item() == 0
    got = {"step_start": out[0][:n].cpu().numpy(), "step_end": out[1][:n].cpu().numpy(),
           "step_nbag": out[2][:n].cpu().numpy(), "seq_step_off": sso.cpu().numpy()}
    assert_steps_equal(got, exp)
    # capacity: count-then-fill semantics
    status.zero_()
    rc = L.segment_steps(t(toks, torch.int32), toks.size, t(off, torch.int64), t(gs, torch.int32), t(fin, torch.uint8), S,
                         delims, out[0], out[1], out[2], sso, 10, ws, status)
    torch.cuda.synchronize()
    assert rc == 0 and status.item() == L.CAPACITY and int(sso[-1]) == n


def _edge_trace():
    """Ragged, empty, one-token, delimiter-only, prompt-only, long multi-delimiter and ragged-tail
    sequences (test_segment_edge_cases' traces)."""
    rng = np.random.default_rng(0)
    seqs = [np.zeros(0, np.int32), np.asarray([5], np.int32), np.asarray([1, 1, 1], np.int32),
            rng.choice([1, 2, 3, 4, 9], 20000, p=[0.05, 0.02, 0.31, 0.31, 0.31]).astype(np.int32),
            rng.choice([1, 3, 4], 4097, p=[0.3, 0.35, 0.35]).astype(np.int32),
            np.asarray([3, 3, 1, 4, 1], np.int32), rng.choice([1, 3, 4, 5, 6], 3000).astype(np.int32)]
    toks = np.concatenate(seqs)
    off = np.concatenate([[0], np.cumsum([q.size for q in seqs])]).astype(np.int64)
    gs = np.asarray([0, 0, 1, 100, 0, 9, 40], np.int32)
    fin = np.asarray([1, 0, 1, 1, 0, 0, 1], np.uint8)
    return toks, off, gs, fin, np.asarray([1, 2], np.int32)


@pytest.mark.parametrize("tau_s,top_k,pairing,step_cap", [(-1.0, 7, oracle.ALIGNED, None), (0.3, 5, oracle.CROSS, None),
                                                          (0.5, 0, oracle.ALIGNED, 40)])
def test_online_round_edge_cases(tau_s, top_k, pairing, step_cap):
    """An online round (cur_mode LAST: 8-CTA Stage-1 clusters) on the segmentation edge cases --
    empty, one-token, prompt-only, delimiter-only, non-final, multi-delimiter and 20k-token
    sequences -- against the oracle's segmentation and Stage 1; with a step capacity below the step
    count: CAPACITY, the required size in seq_step_off, the steps below the capacity written, and
    no Stage-1 output for the sequences whose last step is beyond it."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    from paper_2507_21433_b200.pipeline import Caps, MemSharePath
    toks, off, gs, fin, delims = _edge_trace()
    S = off.size - 1
    bs = SMALL.block_size
    nbl = [-(-(int(off[i + 1] - off[i])) // bs) for i in range(S)]
    perm = np.random.default_rng(5).permutation(sum(nbl)).astype(np.int32)
    table = np.zeros((S, max(nbl)), np.int32)
    o = 0
    for i in range(S):
        table[i, :nbl[i]] = perm[o:o + nbl[i]]
        o += nbl[i]
    nb = int(sum(nbl))
    p = MemSharePath(toks, off, gs, fin, delims, table, np.ones(nb, np.int32), np.full(nb, -1, np.int32), 0,
                     None, None, 0, 0, nb, SMALL.num_layers, SMALL.num_kv_heads, SMALL.num_kv_heads, SMALL.head_dim, bs)
    if step_cap is not None:
        p.set_caps(Caps(step=step_cap, match=p.caps.match, pair=p.caps.pair, target=p.caps.target))
    p.segment()
    p.candidates(tau_s, top_k, pairing, oracle.CUR_LAST)
    torch.cuda.synchronize()
    st, steps, cand = p.read_status(), p.read_steps(), p.read_candidates()
    exp = oracle.segment_steps(toks, off, gs, fin, delims)
    if step_cap is None:
        assert st == 0
        assert_steps_equal(steps, exp)
        oc = oracle.step_candidates(toks, off, exp, delims, table, bs, tau_s, top_k, pairing, oracle.CUR_LAST)
        assert_candidates_equal(cand, oc)
        assert oc["matches"]["seq"].size > 0
    else:
        assert st == L.CAPACITY and steps["seq_step_off"][-1] == exp["seq_step_off"][-1] > step_cap
        assert np.array_equal(steps["seq_step_off"], exp["seq_step_off"])
        for k in ("step_start", "step_end", "step_nbag"):
            assert np.array_equal(steps[k], exp[k][:step_cap]), k
        # Stage 1 only for the sequences whose last step lies below the capacity
        below = [q for q in range(S) if exp["seq_step_off"][q + 1] <= step_cap]
        got_seqs = set(np.unique(cand["matches"]["seq"]).tolist())
        assert got_seqs <= set(below)


def test_long_step_uses_global_table():
    """A 6000-token step (> 2048 content tokens) takes the global-memory hash table path."""
    rng = np.random.default_rng(4)
    long_step = rng.integers(10, 900, 6000).astype(np.int32)
    toks = np.concatenate([long_step, [1], long_step[:5000], [1], rng.integers(10, 900, 3000), [1],
                           long_step, [1]]).astype(np.int32)
    b = traces.TraceBatch(tokens=toks, seq_tok_off=np.array([0, toks.size]), gen_start=np.zeros(1, np.int32),
                          final=np.ones(1, np.uint8), delim_ids=np.array([1], np.int32), vocab=1000)
    w = workloads._paged("long", SMALL, b, 1, 0.05, 0.5)
    full_parity(w)


def test_distance_properties_on_gpu():
    """D(B,B) = 0 exactly, D(a,b) == D(b,a) bit for bit, and the constant-offset closed form."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    from paper_2507_21433_b200.pipeline import MemSharePath
    sh = kv.QWEN32B
    nb = 6
    slice_e = sh.slice_elems
    rng = np.random.default_rng(0)
    base = (rng.integers(-64, 64, (sh.num_layers, 1, slice_e)) * 0.125).astype(np.float32)
    vals = np.concatenate([base, base + np.float32(0.5), base[:, :, ::-1], base - np.float32(0.5),
                           base * np.float32(2.0), base + np.float32(0.5)], axis=1)
    bits = (vals.view(np.uint32) >> 16).astype(np.uint16)
    k = torch.as_tensor(bits.view(np.int16).ravel(), device="cuda").view(torch.bfloat16)
    vbits = ((-vals).view(np.uint32) >> 16).astype(np.uint16)      # V = -K: same squared differences
    v = torch.as_tensor(vbits.view(np.int16).ravel(), device="cuda").view(torch.bfloat16)
    pairs_np = np.zeros(7, L.PAIR_DTYPE)
    tp = [1, 0, 0, 2, 0, 1, 5]
    sp = [0, 1, 0, 0, 2, 5, 1]
    for i in range(7):
        pairs_np[i] = (0, i, i, 10 + i, tp[i], sp[i])
    dims = L.Dims(sh.num_layers, sh.num_kv_heads, sh.num_kv_heads, sh.head_dim, sh.block_size)
    pool = L.KVPool(k.data_ptr(), v.data_ptr(), nb * slice_e, slice_e, nb, 0)
    dev = torch.device("cuda")
    pairs = torch.as_tensor(pairs_np.view(np.uint8), device=dev)
    toff = torch.arange(8, dtype=torch.int64, device=dev)
    npairs = torch.tensor([7], dtype=torch.int64, device=dev)
    ntg = torch.tensor([7], dtype=torch.int64, device=dev)
    dist = torch.empty(7, dtype=torch.float32, device=dev)
    under = torch.empty(7, dtype=torch.uint8, device=dev)
    dec = torch.empty(7 * 32, dtype=torch.uint8, device=dev)
    ws = torch.empty(L.block_distance_workspace_size(dims, nb, 7, 7), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    assert L.block_distance(pool, dims, pairs, toff, npairs, ntg, 7, 7, L.DIST_FULL, None, 0.3, dist, under, dec, ws,
                            status) == 0
    torch.cuda.synchronize()
    D = dist.cpu().numpy()
    assert status.item() == 0
    assert D[2] == 0.0                                   # D(B, B) = 0
    assert D[0] == D[1]                                  # symmetric, bit for bit
    assert abs(D[0] - 0.5) <= 1e-6 * 0.5                 # constant offset 0.5 -> D = 0.5 (32B shape)
    assert D[5] == 0.0 and D[6] == 0.0                   # blocks 1 and 5 are identical
    kh = bits.ravel()
    vh = vbits.ravel()
    Do = oracle.block_distance(kh, vh, nb * slice_e, slice_e, sh.num_layers, sh.num_kv_heads, sh.num_kv_heads,
                               sh.head_dim, sh.block_size, tp, sp)
    compare_distances(D, Do)


def test_head_sharded_two_shards_on_one_gpu():
    """KV-head sharding (bench.py --mode headshard) with both shards on this
    GPU: each shard holds 4 of the 8 KV heads, runs a1-a4 (identical pair lists) and PARTIAL;
    memshare_block_distance_finalize_peers reads both partials through a pointer array (the fused
    peer-memory reduction) and must equal, bit for bit, the device-side sum + FINALIZE (the NCCL
    all-reduce stand-in); both must match the fp64 oracle on the full 8-head pool."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    shape = kv.KVShape(4, 8, 128, 16)
    w = workloads.small(shape, 2, 4000, seed=11)
    shards = [make_path(w, h_local=4, head_offset=h0) for h0 in (0, 4)]
    for p in shards:
        p.autosize(w.tau_s)
        p.segment()
        p.candidates(w.tau_s)
        p.alloc_partial()
        p.distance_call(w.tau_b, L.DIST_PARTIAL)
    torch.cuda.synchronize()
    c0, c1 = (p.read_candidates() for p in shards)
    for k_ in c0["pairs"]:
        assert np.array_equal(c0["pairs"][k_], c1["pairs"][k_]), k_
    p = shards[0]
    # fused reduction: FINALIZE loads both shards' partial sums through a device pointer array
    # (on a multi-GPU node these are symmetric-memory peer mappings over NVLink)
    ptrs = torch.tensor([q.partial_sq.data_ptr() for q in shards], dtype=torch.int64, device="cuda")
    p.finalize_peers(w.tau_b, ptrs, 2)
    torch.cuda.synchronize()
    assert p.read_status() == 0
    gp = p.read_distance()
    p.partial_sq += shards[1].partial_sq                   # the all-reduce (sum over head shards)
    p.distance_call(w.tau_b, L.DIST_FINALIZE)
    torch.cuda.synchronize()
    assert p.read_status() == 0 and shards[1].read_status() == 0
    gd = p.read_distance()
    assert np.array_equal(gp["distance"], gd["distance"])   # same rank-order fp32 sum -> bit-identical
    for k_ in gd["decisions"]:
        assert np.array_equal(gp["decisions"][k_], gd["decisions"][k_]), k_
    pr = c0["pairs"]
    kh, vh, ls, bs = w.host_pool()
    D = oracle.block_distance(kh, vh, ls, bs, shape.num_layers, shape.num_kv_heads, shape.num_kv_heads,
                              shape.head_dim, shape.block_size, pr["target_phys"], pr["source_phys"])
    assert pr["seq"].size > 0
    compare_distances(gd["distance"], D)
    compare_decisions(gd["decisions"], gd["distance"], D, c0["target_off"], pr, w.tau_b)


def test_partial_then_finalize_equals_full():
    import torch
    from paper_2507_21433_b200 import _lib as L
    w = workloads.small(SMALL, 2, 4000, seed=9)
    p = make_path(w)
    p.autosize(w.tau_s)
    p.segment()
    p.candidates(w.tau_s)
    p.alloc_partial()
    p.distance_call(w.tau_b, L.DIST_FULL)
    torch.cuda.synchronize()
    full = p.read_distance()
    ps_full = p.partial_sq.clone()
    p.distance_call(w.tau_b, L.DIST_PARTIAL)
    torch.cuda.synchronize()
    assert torch.equal(p.partial_sq, ps_full)
    p.distance.zero_()
    p.distance_call(w.tau_b, L.DIST_FINALIZE)
    torch.cuda.synchronize()
    fin = p.read_distance()
    assert np.array_equal(full["distance"], fin["distance"])
    for k_ in full["decisions"]:
        assert np.array_equal(full["decisions"][k_], fin["decisions"][k_])
    # partial squares against the oracle's per-layer sums
    oc = p.read_candidates()["pairs"]
    kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
    sk, sv = oracle.partial_sq(kh, vh, p.pool.layer_stride, p.pool.block_stride, SMALL.num_layers,
                               SMALL.num_kv_heads, SMALL.head_dim, SMALL.block_size, oc["target_phys"],
                               oc["source_phys"])
    got = p.partial_sq.cpu().numpy()[:sk.size * 2].reshape(-1, SMALL.num_layers, 2)
    ref = np.stack([sk, sv], -1)
    nz = ref > 0
    assert np.all(got[~nz] == 0)
    assert np.max(np.abs(got[nz] - ref[nz]) / ref[nz]) < 1e-5


def test_remap_random_decisions_vs_oracle():
    """Remap is bit-exact with the oracle on identical (random) decisions, including chains,
    rejected entries, increments after decrements and repeated old blocks."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    rng = np.random.default_rng(1)
    dev = torch.device("cuda")
    for trial in range(20):
        nseq, nblk = 4, 50
        tab = rng.permutation(nseq * nblk).astype(np.int32).reshape(nseq, nblk)
        tab[rng.random(tab.shape) < 0.1] = tab[0, 0]
        rc = np.bincount(tab.ravel(), minlength=nseq * nblk).astype(np.int32)
        fl = np.full(nseq * nblk, -1, np.int32)
        free = np.flatnonzero(rc == 0).astype(np.int32)
        fl[:free.size] = free
        keys = np.unique(rng.integers(0, nseq * nblk, 60))
        dec = np.zeros(keys.size, L.DECISION_DTYPE)
        dec["seq"], dec["target_logical"] = keys // nblk, keys % nblk
        dec["source_phys"] = tab.ravel()[rng.integers(0, tab.size, keys.size)]
        dec["accepted"] = rng.random(keys.size) < 0.8
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=dev)
        dtab, drc, dfl = t(tab, torch.int32), t(rc, torch.int32), t(fl, torch.int32)
        fc = t([free.size], torch.int64)
        nf, af = t([0], torch.int64), t([0], torch.int64)
        ddec = t(dec.view(np.uint8), torch.uint8)
        nt = t([keys.size], torch.int64)
        ws = torch.empty(L.remap_workspace_size(nseq * nblk, keys.size), dtype=torch.uint8, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        assert L.remap(dtab, nblk, nseq, drc, nseq * nblk, dfl, fc, ddec, nt, keys.size, 16, nf, af, ws, status) == 0
        torch.cuda.synchronize()
        st, tab2, rc2, fl2, fc2, nf2, af2 = oracle.remap(tab, rc, fl, free.size,
                                                         {k_: dec[k_] for k_ in dec.dtype.names}, 16)
        assert st == 0 and status.item() == 0
        assert np.array_equal(dtab.cpu().numpy(), tab2) and np.array_equal(drc.cpu().numpy(), rc2)
        assert np.array_equal(dfl.cpu().numpy(), fl2) and int(fc) == fc2 and int(nf) == nf2 and int(af) == af2


def test_device_errors():
    import torch
    from paper_2507_21433_b200 import _lib as L
    from paper_2507_21433_b200.pipeline import Caps
    w = workloads.small(SMALL, 2, 3000, seed=2)
    p = make_path(w, caps=Caps(step=w.num_tokens, match=3, pair=5, target=2))
    p.segment()
    p.candidates(w.tau_s)
    torch.cuda.synchronize()
    assert p.read_status() == L.CAPACITY
    c = p.counts()
    exp = oracle_candidates(w, oracle_steps(w))
    assert c["matches"] == exp["matches"]["seq"].size and c["pairs"] == exp["pairs"]["seq"].size
    # a corrupt physical id in the block table is reported
    w2 = workloads.small(SMALL, 1, 3000, seed=2)
    w2.table = w2.table.copy()
    w2.table[0, 40:] = w2.num_blocks + 5
    p2 = make_path(w2, with_pool=False)
    p2.segment()
    p2.candidates(-1.0)
    torch.cuda.synchronize()
    assert p2.read_status() == L.CORRUPTION


def test_state_snapshot_round_trip():
    """SURVEY.md §5 JSON state snapshot: the path state after a round survives a JSON
    round trip; restored into a fresh path on the pristine trace, the next round gives the same
    decisions and state as the original path's next round; the T0 round's snapshot holds the
    golden free list and affected tokens (tests/golden/tiny_t0.json)."""
    import json
    import os
    import torch
    w = workloads.small(SMALL, 2, 2500, seed=11, eta=0.0)
    p = make_path(w)
    p.autosize(0.5)
    p.round(0.5, 1e-3)
    snap = json.loads(json.dumps(p.snapshot()))
    assert snap["status"] == 0 and snap["counters"]["freed"] > 0
    assert len(snap["free_list"]) == snap["free_count"]
    q = make_path(w, caps=p.caps)
    q.restore_snapshot(snap)
    for path in (p, q):
        path.round(0.5, 1e-3)
    torch.cuda.synchronize()
    a, b = p.read_distance(), q.read_distance()
    for k in a["decisions"]:
        assert np.array_equal(a["decisions"][k], b["decisions"][k]), k
    sa, sb = p.read_state(), q.read_state()
    for k in ("table", "refcount", "free_list", "free_count", "num_freed", "affected"):
        assert np.array_equal(sa[k], sb[k]), k
    # golden T0
    t0 = workloads.tiny(eta=0.0)
    pt = make_path(t0)
    pt.autosize(t0.tau_s)
    pt.round(t0.tau_s, t0.tau_b)
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tiny_t0.json")))
    st = pt.snapshot()
    assert st["free_list"] == g["free_list"] and st["counters"]["affected_tokens"] == g["affected_tokens"]
    with pytest.raises(ValueError):
        make_path(w, caps=p.caps).restore_snapshot(st)       # another geometry


def test_fault_injection_refcount_and_free_list():
    """SURVEY.md §5 fault injection (SPEC.md:607 'corrupted bound'): a refcount corrupted to drive
    a block below zero, and a free list without room for the freed blocks, are reported as
    CORRUPTION by the remap (and a corrupted source id in the pair list by the distance call)."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    w = workloads.small(SMALL, 2, 2500, seed=11, eta=0.0)
    # (1) a refcount of 0 on a block the remap decrements: final count -1
    p = make_path(w)
    p.autosize(0.5)
    p.segment()
    p.candidates(0.5)
    p.distance_call(1e-3)
    torch.cuda.synchronize()
    dec = p.read_distance()["decisions"]
    acc = np.nonzero(dec["accepted"])[0]
    tab = p.table.view(p.num_seqs, p.table_stride).cpu().numpy()
    olds = [int(tab[dec["seq"][i], dec["target_logical"][i]]) for i in acc]
    srcs = set(dec["source_phys"][acc].tolist())
    cand = [o for o, i in zip(olds, acc) if o not in srcs and o != dec["source_phys"][i]]
    assert cand, "no accepted decision whose old block is nobody's source"
    p.refcount[cand[0]] = 0
    p.remap()
    torch.cuda.synchronize()
    assert p.read_status() == L.CORRUPTION
    # (2) the free list already full: no room for the freed blocks
    p2 = make_path(w)
    p2.autosize(0.5)
    p2.free_count.fill_(w.num_blocks)
    p2.round(0.5, 1e-3)
    torch.cuda.synchronize()
    assert p2.read_status() == L.CORRUPTION
    # (3) a source physical id out of range in the pair list
    p3 = make_path(w)
    p3.autosize(0.5)
    p3.segment()
    p3.candidates(0.5)
    torch.cuda.synchronize()
    pr = p3.pairs.view(torch.int32).view(-1, 6)
    pr[0, 5] = w.num_blocks + 3
    p3.distance_call(1e-3)
    torch.cuda.synchronize()
    assert p3.read_status() == L.CORRUPTION


def test_generator_twins_bit_identical():
    w = workloads.small(SMALL, 2, 1500, seed=3)
    p = make_path(w)
    kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
    k2, v2, _, _ = w.host_pool()
    assert np.array_equal(kh, k2) and np.array_equal(vh, v2)


def test_c2_full_size_parity():
    """configs[1] at full size, in the launch configuration bench.py times: segmentation,
    candidates, pairs and remap bit-exact; every pair's distance against the oracle."""
    w = workloads.c2(seed=0)
    p, oc, D, (near_thr, near_tie) = full_parity(w)
    assert oc["pairs"]["seq"].size > 150
    print(f"c2: pairs={oc['pairs']['seq'].size} targets={oc['target_off'].size - 1} near_thresh={near_thr} "
          f"near_tie={near_tie}")


@pytest.mark.parametrize("length", [40000, 100000])
def test_single_cot_more_steps_than_sms(length):
    """The fused single-CoT Stage-1 shape with more finished steps than CTAs (a 40k / 100k-token
    trace: ~400 / ~1,000 steps on 148 CTAs, each CTA taking several steps in ascending order):
    every step's output offsets come from its predecessors' published counts, so the matches,
    pairs and target offsets must still be bit-exact, and the history staging takes several
    passes for the late steps."""
    w = workloads.small(SMALL, 1, length, seed=21)
    st = oracle_steps(w)
    assert st["seq_step_off"][-1] > 2 * 148
    p, oc, D, _ = full_parity(w)
    assert oc["pairs"]["seq"].size > 0


@pytest.mark.parametrize("empty_seq", [0, 2])
def test_online_rounds_with_a_stepless_sequence(empty_seq):
    """Online rounds (LAST and RANGE, fused fill) when one sequence has no finished step (no
    delimiter, not final): its work item publishes zero counts -- as the first key, or as the
    last key that also writes the totals -- and the other sequences' outputs are unchanged."""
    import dataclasses
    w = workloads.small(SMALL, 3, 2000, seed=13)
    b = w.batch
    toks = b.tokens.copy()
    lo, hi = int(b.seq_tok_off[empty_seq]), int(b.seq_tok_off[empty_seq + 1])
    seg = toks[lo:hi]
    seg[np.isin(seg, b.delim_ids)] = 7                    # no delimiter left in that sequence
    fin = np.asarray(b.final, np.uint8).copy()
    fin[empty_seq] = 0                                    # and it is not final: no finished step
    w2 = dataclasses.replace(w, batch=dataclasses.replace(b, tokens=toks, final=fin))
    st = oracle_steps(w2)
    assert st["seq_step_off"][empty_seq + 1] == st["seq_step_off"][empty_seq]
    full_parity(w2, tau_s=0.5, cur_mode=oracle.CUR_LAST)
    full_parity(w2, tau_s=0.5, cur_mode=oracle.CUR_RANGE, cb=[0, 1, 2], ce=[4, 6, 9])


def test_c2_full_size_online_round():
    """configs[1] online: only the last finished step is current; Stage 1 runs as an
    8-CTA cluster over its 12k-token history; everything bit-exact / within tolerance."""
    w = workloads.c2(seed=1)
    full_parity(w, cur_mode=oracle.CUR_LAST)


@pytest.mark.parametrize("shape,eta", [(SMALL, 0.05), (kv.QWEN32B, 0.02), (kv.PHI4, 0.02)])
def test_cosine_metric_vs_oracle(shape, eta):
    """f2 (reading R34): cosine block distance D = mean_l (1 - cos_K + 1 - cos_V)/2,
    GPU vs the fp64 oracle on the same candidate pairs, held to the north star's 1e-5 RELATIVE bar
    (the GPU forms 1 - cos from |t-s|^2 and the norms, without the cancellation of 1 - dot/(|t||s|):
    near-duplicates at eta = 0.02 have D_cos ~ 4e-4); decisions by the same rule as the Euclidean
    metric (tie set, smaller-source-logical tie break, strict threshold)."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    w = workloads.small(shape, 2, 3100, seed=21, eta=eta, **({"vocab": traces.PHI4_VOCAB} if shape is kv.PHI4 else {}))
    p = make_path(w)
    p.autosize(w.tau_s)
    p.segment()
    p.candidates(w.tau_s)
    tau_b = 1.6 * eta * eta      # duplicate pair: both blocks carry independent noise -> D ~ eta^2
    p.distance_call(tau_b, L.DIST_FULL, metric=L.METRIC_COSINE)
    torch.cuda.synchronize()
    assert p.status.item() == 0
    got = p.read_distance()
    c = p.read_candidates()
    oc = c["pairs"]
    assert oc["target_phys"].size > 50
    kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
    Do = oracle.block_cosine(kh, vh, p.pool.layer_stride, p.pool.block_stride, shape.num_layers,
                             shape.num_kv_heads, shape.head_dim, shape.block_size, oc["target_phys"],
                             oc["source_phys"])
    same = oc["target_phys"] == oc["source_phys"]
    assert np.all(got["distance"][same] == 0.0)
    compare_distances(got["distance"], Do)                    # 1e-5 relative, exact 0 where the oracle is 0
    assert (Do < 4 * eta * eta).sum() > 10                    # the near-duplicate regime is exercised
    near = compare_decisions(got["decisions"], got["distance"], Do, c["target_off"], oc, tau_b)
    acc = got["decisions"]["accepted"].astype(bool)
    assert acc.any() and not acc.all()
    print(f"cosine {shape}: near_thresh/tie={near}")


def test_cosine_metric_rejects_partial_modes():
    import torch
    from paper_2507_21433_b200 import _lib as L
    w = workloads.small(SMALL, 2, 2000, seed=4)
    p = make_path(w)
    p.autosize(w.tau_s)
    p.alloc_partial()
    with pytest.raises(RuntimeError):
        p.distance_call(0.01, L.DIST_PARTIAL, metric=L.METRIC_COSINE)
    torch.cuda.synchronize()


@pytest.mark.parametrize("seed", [0, 1])
def test_segment_many_tiles(seed):
    """> 32 tiles (several look-back windows of the single-pass scan), empty and one-token
    sequences between long ones, mixed final flags and prompt lengths, steps crossing tiles."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    rng = np.random.default_rng(100 + seed)
    lens = rng.choice([0, 1, 7, 3000, 40000, 90000], 24, p=[0.15, 0.1, 0.15, 0.3, 0.2, 0.1])
    seqs = [rng.choice([1, 2, 5, 6, 7, 8], n, p=[0.03, 0.01, 0.24, 0.24, 0.24, 0.24]).astype(np.int32) for n in lens]
    toks = np.concatenate(seqs).astype(np.int32)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    gs = np.minimum(rng.integers(0, 300, lens.size), np.maximum(lens, 0) + 2).astype(np.int32)
    fin = rng.integers(0, 2, lens.size).astype(np.uint8)
    delims = np.asarray([1, 2], np.int32)
    exp = oracle.segment_steps(toks, off, gs, fin, delims)
    assert toks.size > 33 * 4096
    dev = torch.device("cuda")
    S, cap = lens.size, int(exp["seq_step_off"][-1]) + 5
    out = [torch.full((cap,), -7, dtype=torch.int32, device=dev) for _ in range(3)]
    sso = torch.full((S + 1,), -9, dtype=torch.int64, device=dev)
    ws = torch.full((L.segment_steps_workspace_size(toks.size, S, cap),), 0xAB, dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    t = lambda a, dt: torch.as_tensor(a, dtype=dt, device=dev)
    for _ in range(2):                                   # the second call reuses the dirty workspace
        assert L.segment_steps(t(toks, torch.int32), toks.size, t(off, torch.int64), t(gs, torch.int32),
                               t(fin, torch.uint8), S, delims, out[0], out[1], out[2], sso, cap, ws, status) == 0
        torch.cuda.synchronize()
        n = int(sso[-1])
        assert status.item() == 0
        got = {"step_start": out[0][:n].cpu().numpy(), "step_end": out[1][:n].cpu().numpy(),
               "step_nbag": out[2][:n].cpu().numpy(), "seq_step_off": sso.cpu().numpy()}
        assert_steps_equal(got, exp)
