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


def compare_decisions(gpu_dec, gpu_D, ora_D, target_off, pairs, tau_b):
    """Per-target decisions ("selecting those with minimal distances", reading R22;
    accept iff D < tau_b, R21) against the oracle on the same pairs.

    `pairs` holds the oracle's pair records (seq, target_logical, target_phys, source_logical,
    source_phys) aligned with `ora_D` / `gpu_D`, grouped by `target_off`. Checked per target:
      * the target identity (seq, target_logical, target_phys) and num_candidates: exact;
      * the GPU's pick is one of the target's pairs (source_logical AND source_phys), its recorded
        distance is bit-equal to the GPU's per-pair distance and within DIST_RTOL of the oracle's;
      * the pick is the argmin of the GPU's own distances with exact ties -> smaller source
        logical (the rule, enforced exactly on the GPU's values);
      * the pick lies in the oracle's tie set: D_oracle[pick] <= D_min (1 + NEAR_TIE); where the
        oracle minimum is exactly 0 (bit-identical blocks: both sides compute 0 exactly) the pick
        must BE the oracle's (the smallest source logical among the zeros);
      * accepted == (GPU distance < fp32 tau_b) exactly, and equals the oracle's decision unless
        the oracle's best distance is within NEAR_THRESH of tau_b.
    Returns (near_threshold, near_tie) counts (reported, not failed)."""
    src_logical = np.asarray(pairs["source_logical"])
    gpu_D = np.asarray(gpu_D, np.float32)
    best, acc, _ = oracle.select(ora_D, target_off, src_logical, tau_b)
    near_thresh = near_tie = 0
    tb32 = np.float32(tau_b)
    tb = float(tb32)
    for t in range(target_off.size - 1):
        p0, p1 = int(target_off[t]), int(target_off[t + 1])
        ob = int(best[t])
        for k in ("seq", "target_logical", "target_phys"):
            assert gpu_dec[k][t] == pairs[k][ob], f"target {t}: {k} {gpu_dec[k][t]} != {pairs[k][ob]}"
        assert gpu_dec["num_candidates"][t] == p1 - p0, f"target {t}: num_candidates"
        hit = np.nonzero(src_logical[p0:p1] == gpu_dec["source_logical"][t])[0]
        assert hit.size == 1, f"target {t}: GPU source logical {gpu_dec['source_logical'][t]} is not a candidate"
        g = p0 + int(hit[0])
        assert gpu_dec["source_phys"][t] == pairs["source_phys"][g], f"target {t}: source_phys"
        gdist = np.float32(gpu_dec["distance"][t])
        assert gdist.view(np.uint32) == gpu_D[g].view(np.uint32), f"target {t}: decision distance != pair distance"
        if ora_D[g] == 0.0:
            assert gdist == 0.0, f"target {t}: identical blocks must give 0"
        else:
            assert abs(float(gdist) - ora_D[g]) <= DIST_RTOL * ora_D[g], f"target {t}: decision distance"
        # the GPU's own argmin with the smaller-logical tie rule, exactly
        seg = gpu_D[p0:p1]
        m = seg.min()
        cand = np.nonzero(seg == m)[0]
        exp_g = p0 + int(cand[np.argmin(src_logical[p0:p1][cand])])
        assert g == exp_g, f"target {t}: GPU pick {g} is not its own argmin / smallest-logical tie {exp_g}"
        # the oracle's tie set
        dmin = float(ora_D[p0:p1].min())
        if dmin == 0.0:
            assert g == ob, f"target {t}: exact D == 0 tie must go to the smaller source logical"
        else:
            assert ora_D[g] <= dmin * (1.0 + NEAR_TIE), f"target {t}: GPU pick D={ora_D[g]!r} outside the tie set of {dmin!r}"
        if g != ob:
            near_tie += 1
        assert bool(gpu_dec["accepted"][t]) == bool(gdist < tb32), f"target {t}: accepted != (D < tau_b)"
        if bool(gpu_dec["accepted"][t]) != bool(acc[t]):
            assert abs(ora_D[ob] - tb) <= NEAR_THRESH * tb, f"target {t}: accept differs away from the threshold"
            near_thresh += 1
    return near_thresh, near_tie


def host_pool_from_device(k, v):
    import torch
    return (k.view(torch.int16).cpu().numpy().view(np.uint16), v.view(torch.int16).cpu().numpy().view(np.uint16))
