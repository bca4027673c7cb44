"""GPU parity of the grouped distance schedule (MEMSHARE_DIST_GROUPED: runs of targets whose
source lists are nested prefixes share every staged source slice -- CROSS pairing, PAPER.md:319
"pairwise"; the all-pairs matrix).

Each case scores the same list with the hint off and on: the grouped schedule must match the
oracle (distances within 1e-5 relative, decisions, remap) and the single-anchor kernel to fp32
summation-order rounding (it forms the same per-thread chains; only the fixed cross-warp order over
16 KiB sub-slices differs), with exact zeros kept exact."""
import os

import numpy as np
import pytest

import oracle
from synth import kv, traces, workloads

from _gpu_util import compare_distances, host_pool_from_device, make_path
from test_gpu_path import check_round

pytestmark = pytest.mark.gpu

SMALL = kv.KVShape(8, 4, 64, 16)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_21433_b200 import build
    build.build()


def _with_hint(on):
    old = os.environ.get("MEMSHARE_GROUPED")
    os.environ["MEMSHARE_GROUPED"] = "1" if on else "0"
    return old


def _restore(old):
    if old is None:
        os.environ.pop("MEMSHARE_GROUPED", None)
    else:
        os.environ["MEMSHARE_GROUPED"] = old


def _cross_round(w, tau_s, top_k, grouped, force_hint=False, pairing=oracle.CROSS):
    import torch
    old = _with_hint(grouped)
    try:
        p = make_path(w)
        p.autosize(tau_s, top_k, pairing)
        p.segment()
        p.candidates(tau_s, top_k, pairing)
        if force_hint:
            p.grouped_hint = True
        p.distance_call(w.tau_b)
        p.remap()
        torch.cuda.synchronize()
    finally:
        _restore(old)
    assert p.read_status() == 0
    return p


def _assert_close_to_single(d_grp, d_one):
    d_grp = np.asarray(d_grp, np.float64)
    d_one = np.asarray(d_one, np.float64)
    assert d_grp.shape == d_one.shape
    z = d_one == 0.0
    assert np.array_equal(d_grp[z], d_one[z])            # identical blocks: exact zero on both
    rel = np.abs(d_grp[~z] - d_one[~z]) / np.abs(d_one[~z])
    assert rel.size == 0 or rel.max() <= 2e-6, rel.max()


CASES = {
    # name: (workload factory, tau_s, top_k)
    "cross_small": (lambda: workloads.small(SMALL, 2, 2500, seed=7), 0.3, 0),
    "cross_geom": (lambda: workloads.small(kv.KVShape(2, 3, 64, 16), 2, 1800, seed=3), 0.6, 0),      # 6 KiB slices
    "cross_phi4": (lambda: workloads.small(kv.PHI4, 1, 3300, seed=5, gen_start=128, vocab=traces.PHI4_VOCAB),
                   0.3, 0),                                                                          # 40 KiB: partial stage
    "cross_long_lists": (lambda: workloads.small(SMALL, 1, 6000, seed=2), -1.0, 8),                  # > 64 sources
    "cross_tiny": (lambda: workloads.tiny(eta=0.0), -1.0, 3),                                         # 4 KiB slices, D == 0
}


@pytest.mark.parametrize("case", list(CASES))
def test_grouped_cross_parity(case):
    make, tau_s, top_k = CASES[case]
    w = make()
    p1 = _cross_round(w, tau_s, top_k, grouped=True)
    check_round(p1, w, tau_s, w.tau_b, top_k, oracle.CROSS)
    d1 = p1.read_distance()["distance"]
    tl = np.diff(p1.read_candidates()["target_off"])
    assert d1.size > 0
    if case == "cross_long_lists":
        assert tl.max() > 64                               # the producer's 64-source chunks
    del p1
    p0 = _cross_round(w, tau_s, top_k, grouped=False)
    _assert_close_to_single(d1, p0.read_distance()["distance"])


@pytest.mark.parametrize("seed", [3, 11])
def test_grouped_hint_on_aligned_lists(seed):
    """ALIGNED lists rarely nest: the hint must find the (few) prefix runs and leave the rest as
    one-anchor groups, with the full oracle check passing."""
    w = workloads.small(SMALL, 3, 2500, seed=seed)
    p = _cross_round(w, w.tau_s, 0, grouped=True, force_hint=True, pairing=oracle.ALIGNED)
    check_round(p, w, w.tau_s, w.tau_b, 0, oracle.ALIGNED)


@pytest.mark.parametrize("shape,window", [(SMALL, 40), (kv.PHI4, 24), (kv.KVShape(2, 2, 64, 16), 32)])
def test_grouped_all_pairs(shape, window):
    """f3: every pair of a block window (target j against blocks lo..j-1: nested prefixes)."""
    import torch
    from paper_2507_21433_b200.pipeline import Caps
    w = workloads.small(shape, 1, max(2000, 16 * (window + 40)), seed=9)
    npairs = window * (window - 1) // 2
    outs = []
    for grouped in (True, False):
        old = _with_hint(grouped)
        try:
            p = make_path(w, caps=Caps(step=4096, match=64, pair=npairs, target=window))
            p.all_pairs([8], [8 + window])
            p.distance_call(0.5)
            torch.cuda.synchronize()
        finally:
            _restore(old)
        assert p.read_status() == 0
        outs.append(p.read_distance()["distance"].copy())
        if grouped:
            r = oracle.all_pairs(w.batch.seq_tok_off, [8], [8 + window], w.table, shape.block_size)
            kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
            D = oracle.block_distance(kh, vh, p.pool.layer_stride, p.pool.block_stride, shape.num_layers,
                                      shape.num_kv_heads, shape.num_kv_heads, shape.head_dim, shape.block_size,
                                      r["pairs"]["target_phys"], r["pairs"]["source_phys"])
            assert D.size == npairs
            compare_distances(outs[0], D)
        del p
    _assert_close_to_single(outs[0], outs[1])


def test_grouped_partial_mode():
    """PARTIAL (KV-head-sharded) mode under the hint: the per-(pair, layer, K|V) squared sums
    match the single-anchor kernel's to summation-order rounding."""
    import torch
    from paper_2507_21433_b200 import _lib as L
    w = workloads.small(SMALL, 2, 2500, seed=7)
    outs = []
    for grouped in (True, False):
        old = _with_hint(grouped)
        try:
            p = make_path(w)
            p.autosize(0.3, 0, oracle.CROSS)
            p.segment()
            p.candidates(0.3, 0, oracle.CROSS)
            ps = p.alloc_partial()
            p.distance_call(w.tau_b, mode=L.DIST_PARTIAL, partial_sq=ps)
            torch.cuda.synchronize()
        finally:
            _restore(old)
        assert p.read_status() == 0
        n = int(p.read_candidates()["target_off"][-1])
        outs.append(ps.reshape(-1)[: n * SMALL.num_layers * 2].cpu().numpy().astype(np.float64))
        del p
    assert outs[0].size > 0
    _assert_close_to_single(outs[0], outs[1])
