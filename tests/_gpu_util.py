"""Helpers for the -m gpu parity tests: run the CUDA path and the oracle on the same inputs."""
from __future__ import annotations

import numpy as np

import oracle

DIST_RTOL = 1e-5          # north_star: distances within 1e-5 relative (fp32 accumulation)
NEAR_THRESH = 1e-4        # decisions may differ only within 1e-4 relative of tau_b ...
NEAR_TIE = 1e-5           # ... or when the best two oracle distances are within 1e-5 relative


def make_path(w, h_local=None, head_offset=0, caps=None, with_pool=True):
    import torch
    from paper_2507_21433_b200.pipeline import MemSharePath
    if with_pool:
        k, v, ls, bs = w.device_pool("cuda", h_local=h_local, head_offset=head_offset)
    else:
        k = v = None
        ls = bs = 0
    b = w.batch
    sh = w.shape
    p = MemSharePath(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids, w.table, w.refcount, w.free_list,
                     w.free_count, k, v, ls, bs, w.num_blocks, sh.num_layers, h_local or sh.num_kv_heads,
                     sh.num_kv_heads, sh.head_dim, sh.block_size, caps=caps)
    torch.cuda.synchronize()
    return p


def oracle_steps(w):
    b = w.batch
    return oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)


def oracle_candidates(w, steps, tau_s=None, top_k=0, pairing=oracle.ALIGNED, cur_mode=oracle.CUR_ALL, cur_begin=None,
                      cur_end=None, table=None):
    b = w.batch
    return oracle.step_candidates(b.tokens, b.seq_tok_off, steps, b.delim_ids, w.table if table is None else table,
                                  w.shape.block_size, w.tau_s if tau_s is None else tau_s, top_k, pairing, cur_mode,
                                  cur_begin, cur_end)


def assert_steps_equal(got, exp):
    for k in ("step_start", "step_end", "step_nbag", "seq_step_off"):
        assert np.array_equal(np.asarray(got[k]), np.asarray(exp[k])), k


def assert_candidates_equal(got, exp):
    for k in ("seq", "step", "cand_step", "rank"):
        assert np.array_equal(got["matches"][k], exp["matches"][k]), f"matches.{k}"
    # the cosine is one IEEE expression on both sides: bit-exact
    assert np.array_equal(got["matches"]["cosine"].view(np.uint64), exp["matches"]["cosine"].view(np.uint64))
    for k in ("seq", "target_idx", "target_logical", "source_logical", "target_phys", "source_phys"):
        assert np.array_equal(got["pairs"][k], exp["pairs"][k]), f"pairs.{k}"
    assert np.array_equal(got["target_off"], exp["target_off"])


def compare_distances(gpu_D, ora_D):
    """Relative error within DIST_RTOL; exact zero where the oracle is exactly zero."""
    gpu_D = np.asarray(gpu_D, np.float64)
    zero = ora_D == 0.0
    assert np.all(gpu_D[zero] == 0.0), "identical blocks must give D == 0 exactly"
    nz = ~zero
    rel = np.abs(gpu_D[nz] - ora_D[nz]) / np.abs(ora_D[nz])
    assert rel.size == 0 or rel.max() <= DIST_RTOL, f"max rel err {rel.max():.3e}"
    return float(rel.max()) if rel.size else 0.0


def compare_decisions(gpu_dec, ora_D, target_off, src_logical, tau_b):
    """Decisions equal except near-threshold / near-tie targets, which are counted and returned."""
    best, acc, _ = oracle.select(ora_D, target_off, src_logical, tau_b)
    near_thresh = near_tie = 0
    tb = float(np.float32(tau_b))
    for t in range(target_off.size - 1):
        p0, p1 = target_off[t], target_off[t + 1]
        Ds = np.sort(ora_D[p0:p1])
        tie = Ds.size > 1 and (Ds[1] - Ds[0]) <= NEAR_TIE * max(Ds[1], 1e-30)
        thr = abs(ora_D[best[t]] - tb) <= NEAR_THRESH * tb
        src_ok = gpu_dec["source_logical"][t] == src_logical[best[t]]
        acc_ok = bool(gpu_dec["accepted"][t]) == bool(acc[t])
        if not src_ok:
            assert tie, f"target {t}: source differs without a near tie"
            near_tie += 1
        if not acc_ok:
            assert thr, f"target {t}: accept differs away from the threshold"
            near_thresh += 1
    return near_thresh, near_tie


def host_pool_from_device(k, v):
    import torch
    return (k.view(torch.int16).cpu().numpy().view(np.uint16), v.view(torch.int16).cpu().numpy().view(np.uint16))
