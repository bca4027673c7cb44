"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py uses.

c3 (QwQ-32B shape, the 64-sequence batch as bench.py's two N = 1 waves), c4 (Phi-4-reasoning-
plus shape, all 128 AIME-length traces in bench.py's waves) and a c5 wave: segmentation, Stage-1
matches and block pairs are compared in full (bit-exact); distances and decisions on a seeded
sample of whole targets the oracle computes one by one (only their blocks are copied to the
host); the remap in full on the GPU's own decisions.
"""
import numpy as np
import pytest

import oracle
from synth import workloads

from _gpu_util import (assert_candidates_equal, assert_steps_equal, compare_decisions, compare_distances, make_path,
                       oracle_candidates, oracle_steps)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_21433_b200 import build
    build.build()


def sampled_parity(w, n_targets=24, seed=0):
    import torch
    p = make_path(w)
    p.autosize(w.tau_s)
    p.round(w.tau_s, w.tau_b)
    torch.cuda.synchronize()
    assert p.read_status() == 0
    st = oracle_steps(w)
    assert_steps_equal(p.read_steps(), st)
    oc = oracle_candidates(w, st)
    gc = p.read_candidates()
    assert_candidates_equal(gc, oc)
    gd = p.read_distance()
    toff, pr = oc["target_off"], oc["pairs"]
    T = toff.size - 1
    rng = np.random.default_rng(seed)
    tsel = np.sort(rng.choice(T, size=min(n_targets, T), replace=False))
    psel = np.concatenate([np.arange(toff[t], toff[t + 1]) for t in tsel])
    # copy only the blocks these pairs touch into a compact host pool
    blocks = np.unique(np.concatenate([pr["target_phys"][psel], pr["source_phys"][psel]]))
    sh = w.shape
    slice_e = sh.block_size * sh.num_kv_heads * sh.head_dim
    idx = torch.as_tensor(blocks, device=p.dev, dtype=torch.long)
    kc = p.k_pool.view(sh.num_layers, w.num_blocks, slice_e).index_select(1, idx)
    vc = p.v_pool.view(sh.num_layers, w.num_blocks, slice_e).index_select(1, idx)
    kh = kc.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).ravel()
    vh = vc.contiguous().view(torch.int16).cpu().numpy().view(np.uint16).ravel()
    remap = {int(b): i for i, b in enumerate(blocks)}
    tp = np.array([remap[int(x)] for x in pr["target_phys"][psel]], np.int32)
    sp = np.array([remap[int(x)] for x in pr["source_phys"][psel]], np.int32)
    D = oracle.block_distance(kh, vh, blocks.size * slice_e, slice_e, sh.num_layers, sh.num_kv_heads,
                              sh.num_kv_heads, sh.head_dim, sh.block_size, tp, sp)
    compare_distances(gd["distance"][psel], D)
    sub_off = np.concatenate([[0], np.cumsum([toff[t + 1] - toff[t] for t in tsel])])
    sub_dec = {k: v[tsel] for k, v in gd["decisions"].items()}
    near = compare_decisions(sub_dec, gd["distance"][psel], D, sub_off, {k: v[psel] for k, v in pr.items()}, w.tau_b)
    s = p.read_state()
    st_o, tab, rc, fl, fc, nf, af = oracle.remap(w.table, w.refcount, w.free_list, w.free_count, gd["decisions"],
                                                 sh.block_size)
    assert st_o == 0
    assert np.array_equal(s["table"], tab) and np.array_equal(s["refcount"], rc)
    assert np.array_equal(s["free_list"], fl) and s["free_count"] == fc and s["num_freed"] == nf and s["affected"] == af
    print(f"{w.name}: steps={st['step_start'].size} pairs={pr['seq'].size} targets={T} sampled_pairs={psel.size} "
          f"near_thresh/tie={near} freed={nf} affected={af}")
    del p
    torch.cuda.empty_cache()


def _plan(cfg, n):
    import torch

    import bench
    bins, W, _ = bench.plan_waves(cfg, n, 1, 0, torch.device("cuda", 0))
    return bins


def test_c3_bench_waves_64_targets():
    """configs[2]: the 64-sequence QwQ-32B batch, both waves of bench.py's N = 1 plan (LPT on
    Stage-1 pair counts, ~32 sequences / 103 GB of KV each), 64 sampled targets per wave."""
    for wi, idx in enumerate(_plan("c3", 64)):
        sampled_parity(workloads.batch("c3", idx, 0), n_targets=64, seed=wi)


def test_c4_phi4_all_128_traces():
    """configs[3]: all 128 Phi-4-reasoning-plus AIME-length traces (~430 GB of KV) as bench.py's
    waves, 48 sampled targets per wave."""
    bins = _plan("c4", 128)
    assert sorted(i for b in bins for i in b) == list(range(128))
    for wi, idx in enumerate(bins):
        sampled_parity(workloads.batch("c4", idx, 0), n_targets=48, seed=wi)


def test_c5_one_wave_32_sequences():
    """configs[4]: 32 x 16,384-token CoTs at the 32B shape (one per-GPU wave, 137 GB pool), 64
    sampled targets."""
    sampled_parity(workloads.batch("c5", list(range(32)), 0), n_targets=64)
