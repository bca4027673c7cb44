"""CPU oracle for MemShare's KV-block reuse path -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

ctypes + numpy marshalling around ``memshare_oracle.c`` (plain single-threaded C99,
fp64), which follows PAPER.md Algorithm 1 and the block-table sharing mechanism line by
line; see that file's header for the citations and DESIGN.md for the readings taken.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. It shares no code with
``paper_2507_21433_b200`` and never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(_HERE, "memshare_oracle.c")
SO = os.path.join(_HERE, "libmemshare_oracle.so")

ALIGNED, CROSS = 0, 1
CUR_ALL, CUR_LAST, CUR_RANGE = 0, 1, 2
OK, INVALID, CAPACITY, CORRUPTION = 0, 1, 2, 3


def build() -> str:
    """Compile the oracle (plain -O2, no fast-math, no FMA contraction, no OpenMP)."""
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-ffp-contract=off",
                               "-fno-fast-math", "-o", SO, SRC, "-lm"])
    return SO


_lib = None
P = ctypes.c_void_p
I32, I64, F64, F32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_float


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_segment_steps.argtypes = [P, P, P, P, I32, P, I32, P, P, P, P, I64]
        L.oracle_segment_steps.restype = I64
        L.oracle_cosine.argtypes = [I64, I64, I64]
        L.oracle_cosine.restype = F64
        L.oracle_bag.argtypes = [P, I64, P, I32, P, P, P]
        L.oracle_bag.restype = I32
        L.oracle_step_candidates.argtypes = ([P, P, I32, P, P, P, P, I32, I32, P, P, P, I32, I32, F64, I32, I32]
                                             + [P] * 5 + [I64, P] + [P] * 6 + [I64, P, P, I64, P])
        L.oracle_step_candidates.restype = ctypes.c_int
        L.oracle_partial_sq.argtypes = [P, P, I64, I64, I32, I32, I32, I32, P, P, I64, P, P]
        L.oracle_partial_sq.restype = None
        L.oracle_finalize.argtypes = [P, P, I64, I32, I32, I32, P]
        L.oracle_finalize.restype = None
        L.oracle_block_distance.argtypes = [P, P, I64, I64, I32, I32, I32, I32, I32, P, P, I64, P]
        L.oracle_block_distance.restype = None
        L.oracle_select.argtypes = [P, I64, P, I64, P, F32, P, P, P]
        L.oracle_select.restype = None
        L.oracle_remap.argtypes = [P, I32, P, I32, P, P, P, P, P, P, I64, I32, P, P]
        L.oracle_remap.restype = ctypes.c_int
        L.oracle_block_cosine.argtypes = [P, P, I64, I64, I32, I32, I32, I32, P, P, I64, P]
        L.oracle_block_cosine.restype = None
        L.oracle_kv_append.argtypes = [P, P, I64, I64, I32, I32, I32, I32, P, I32, I32, P, P, P, I32, P, P, P, P]
        L.oracle_kv_append.restype = ctypes.c_int
        L.oracle_paged_attention.argtypes = [P, P, I64, I64, I32, I32, I32, I32, P, I32, P, I32, P, I32, F64, P]
        L.oracle_paged_attention.restype = ctypes.c_int
        L.oracle_admit.argtypes = [P, I32, I32, I32, I64, P]
        L.oracle_admit.restype = I32
        L.oracle_similarity_ratio.argtypes = [P, P, I64, I32, P]
        L.oracle_similarity_ratio.restype = None
        L.oracle_all_pairs.argtypes = [P, I32, P, P, P, I32, I32] + [P] * 6 + [I64, P, I64, P]
        L.oracle_all_pairs.restype = I64
        _lib = L
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def _p(a):
    return a.ctypes.data


# ---------------------------------------------------------------- a1 segmentation
def segment_steps(tokens, seq_tok_off, gen_start, final, delims):
    tokens, off = _c(tokens, np.int32), _c(seq_tok_off, np.int64)
    gs, fin, dl = _c(gen_start, np.int32), _c(final, np.uint8), _c(delims, np.int32)
    S = gs.size
    cap = max(1, tokens.size)
    st, en, nb = (np.zeros(cap, np.int32) for _ in range(3))
    sso = np.zeros(S + 1, np.int64)
    n = lib().oracle_segment_steps(_p(tokens), _p(off), _p(gs), _p(fin), S, _p(dl), dl.size,
                                   _p(st), _p(en), _p(nb), _p(sso), cap)
    return {"step_start": st[:n].copy(), "step_end": en[:n].copy(), "step_nbag": nb[:n].copy(),
            "seq_step_off": sso}


# ---------------------------------------------------------------- a2/a3 helpers (pins)
def bag(tokens, delims=()):
    t, dl = _c(tokens, np.int32), _c(list(delims) or [-1], np.int32)
    ids, cnt, n2 = np.zeros(max(1, t.size), np.int32), np.zeros(max(1, t.size), np.int64), np.zeros(1, np.int64)
    n = lib().oracle_bag(_p(t), t.size, _p(dl), dl.size, _p(ids), _p(cnt), _p(n2))
    return ids[:n].copy(), cnt[:n].copy(), int(n2[0])


def cosine(dot, n2a, n2b):
    return lib().oracle_cosine(int(dot), int(n2a), int(n2b))


def cosine_of_tokens(a, b, delims=()):
    ia, ca, na = bag(a, delims)
    ib, cb, nb = bag(b, delims)
    common, xa, xb = np.intersect1d(ia, ib, return_indices=True)
    dot = int((ca[xa] * cb[xb]).sum())
    return cosine(dot, na, nb)


# ---------------------------------------------------------------- a3/a4 candidates + pairs
def step_candidates(tokens, seq_tok_off, steps, delims, table, block_size, tau_s, top_k=0, pairing=ALIGNED,
                    cur_mode=CUR_ALL, cur_begin=None, cur_end=None):
    tokens, off = _c(tokens, np.int32), _c(seq_tok_off, np.int64)
    sso, st, en = _c(steps["seq_step_off"], np.int64), _c(steps["step_start"], np.int32), _c(steps["step_end"], np.int32)
    dl, tab = _c(delims, np.int32), _c(table, np.int32)
    S = sso.size - 1
    cb = _c(cur_begin if cur_begin is not None else np.zeros(max(S, 1)), np.int32)
    ce = _c(cur_end if cur_end is not None else np.zeros(max(S, 1)), np.int32)
    counts = np.zeros(3, np.int64)
    mcap, pcap, tcap = 1024, 4096, 2048
    while True:
        m = [np.zeros(mcap, np.int32) for _ in range(4)] + [np.zeros(mcap, np.float64)]
        p = [np.zeros(pcap, np.int32) for _ in range(6)]
        toff = np.zeros(tcap + 1, np.int64)
        nm, np_, nt = (np.zeros(1, np.int64) for _ in range(3))
        rc = lib().oracle_step_candidates(
            _p(tokens), _p(off), S, _p(sso), _p(st), _p(en), _p(dl), dl.size, cur_mode, _p(cb), _p(ce),
            _p(tab), tab.shape[1], block_size, float(tau_s), int(top_k), int(pairing),
            *[_p(a) for a in m], mcap, _p(nm), *[_p(a) for a in p], pcap, _p(np_), _p(toff), tcap, _p(nt))
        if rc == OK:
            break
        assert rc == CAPACITY, rc
        mcap, pcap, tcap = max(mcap, int(nm[0])), max(pcap, int(np_[0])), max(tcap, int(nt[0]))
    M, Pn, T = int(nm[0]), int(np_[0]), int(nt[0])
    names_m = ["seq", "step", "cand_step", "rank", "cosine"]
    names_p = ["seq", "target_idx", "target_logical", "source_logical", "target_phys", "source_phys"]
    return {"matches": {k: a[:M].copy() for k, a in zip(names_m, m)},
            "pairs": {k: a[:Pn].copy() for k, a in zip(names_p, p)},
            "target_off": toff[:T + 1].copy()}


# ---------------------------------------------------------------- a5/a6 distance + selection
def partial_sq(k, v, layer_stride, block_stride, num_layers, h_local, head_dim, block_size, tphys, sphys):
    k, v = _c(k, np.uint16), _c(v, np.uint16)
    tp, sp = _c(tphys, np.int32), _c(sphys, np.int32)
    sk = np.zeros((tp.size, num_layers), np.float64)
    sv = np.zeros_like(sk)
    lib().oracle_partial_sq(_p(k), _p(v), layer_stride, block_stride, num_layers, h_local, head_dim, block_size,
                            _p(tp), _p(sp), tp.size, _p(sk), _p(sv))
    return sk, sv


def finalize(sk, sv, num_layers, block_size, h_global):
    sk, sv = _c(sk, np.float64), _c(sv, np.float64)
    Pn = sk.shape[0]
    D = np.zeros(Pn, np.float64)
    lib().oracle_finalize(_p(sk), _p(sv), Pn, num_layers, block_size, h_global, _p(D))
    return D


def block_distance(k, v, layer_stride, block_stride, num_layers, h_local, h_global, head_dim, block_size,
                   tphys, sphys):
    k, v = _c(k, np.uint16), _c(v, np.uint16)
    tp, sp = _c(tphys, np.int32), _c(sphys, np.int32)
    D = np.zeros(tp.size, np.float64)
    lib().oracle_block_distance(_p(k), _p(v), layer_stride, block_stride, num_layers, h_local, h_global, head_dim,
                                block_size, _p(tp), _p(sp), tp.size, _p(D))
    return D


def select(D, target_off, src_logical, tau_b):
    D, toff, sl = _c(D, np.float64), _c(target_off, np.int64), _c(src_logical, np.int32)
    T = toff.size - 1
    best = np.zeros(max(T, 1), np.int64)
    acc = np.zeros(max(T, 1), np.uint8)
    under = np.zeros(max(D.size, 1), np.uint8)
    lib().oracle_select(_p(D), D.size, _p(toff), T, _p(sl), float(np.float32(tau_b)), _p(best), _p(acc), _p(under))
    return best[:T].copy(), acc[:T].copy(), under[:D.size].copy()


def decisions(pairs, target_off, D, best, accepted):
    """Per-target decision records (SoA) from the selection."""
    T = target_off.size - 1
    b = best[:T]
    return {"seq": pairs["seq"][b].copy(), "target_logical": pairs["target_logical"][b].copy(),
            "target_phys": pairs["target_phys"][b].copy(), "source_logical": pairs["source_logical"][b].copy(),
            "source_phys": pairs["source_phys"][b].copy(), "accepted": accepted[:T].astype(np.uint8),
            "distance": D[b].copy(), "num_candidates": np.diff(target_off).astype(np.int32)}


# ---------------------------------------------------------------- a7 remap
def remap(table, refcount, free_list, free_count, dec, block_size):
    """Returns (status, table, refcount, free_list, free_count, num_freed, affected) on copies."""
    tab, rc, fl = _c(table, np.int32).copy(), _c(refcount, np.int32).copy(), _c(free_list, np.int32).copy()
    fc = np.asarray([free_count], np.int64)
    nf, af = np.zeros(1, np.int64), np.zeros(1, np.int64)
    ds, dt, dp = _c(dec["seq"], np.int32), _c(dec["target_logical"], np.int32), _c(dec["source_phys"], np.int32)
    da = _c(dec["accepted"], np.uint8)
    st = lib().oracle_remap(_p(tab), tab.shape[1], _p(rc), rc.size, _p(fl), _p(fc), _p(ds), _p(dt), _p(dp), _p(da),
                            ds.size, block_size, _p(nf), _p(af))
    return st, tab, rc, fl, int(fc[0]), int(nf[0]), int(af[0])


# ---------------------------------------------------------------- f4 similarity ratio
def similarity_ratio_counts(matches, num_seqs):
    """Per-sequence number of steps with a Stage-1 survivor (numerator of PAPER.md:121-126)."""
    ms, mr = _c(matches["seq"], np.int32), _c(matches["rank"], np.int32)
    out = np.zeros(max(num_seqs, 1), np.int64)
    lib().oracle_similarity_ratio(_p(ms), _p(mr), ms.size, num_seqs, _p(out))
    return out[:num_seqs]


# ---------------------------------------------------------------- f3 all pairs
def all_pairs(seq_tok_off, blk_begin, blk_end, table, block_size):
    off, bb, be, tab = _c(seq_tok_off, np.int64), _c(blk_begin, np.int32), _c(blk_end, np.int32), _c(table, np.int32)
    S = bb.size
    cap = 16
    while True:
        p = [np.zeros(cap, np.int32) for _ in range(6)]
        toff = np.zeros(cap + 1, np.int64)
        nt = np.zeros(1, np.int64)
        n = lib().oracle_all_pairs(_p(off), S, _p(bb), _p(be), _p(tab), tab.shape[1], block_size, *[_p(a) for a in p],
                                   cap, _p(toff), cap, _p(nt))
        if n <= cap and nt[0] <= cap:
            break
        cap = max(n, int(nt[0])) + 1
    names_p = ["seq", "target_idx", "target_logical", "source_logical", "target_phys", "source_phys"]
    return {"pairs": {k: a[:n].copy() for k, a in zip(names_p, p)}, "target_off": toff[:int(nt[0]) + 1].copy()}


# ---------------------------------------------------------------- f2 cosine block metric
def block_cosine(k, v, layer_stride, block_stride, num_layers, h_local, head_dim, block_size, tphys, sphys):
    """D_cos = 1 - mean over layers of (cos_K + cos_V)/2 (reading R34)."""
    k, v = _c(k, np.uint16), _c(v, np.uint16)
    tp, sp = _c(tphys, np.int32), _c(sphys, np.int32)
    D = np.zeros(tp.size, np.float64)
    lib().oracle_block_cosine(_p(k), _p(v), layer_stride, block_stride, num_layers, h_local, head_dim, block_size,
                              _p(tp), _p(sp), tp.size, _p(D))
    return D


# ---------------------------------------------------------------- f1 decode-loop integration
def kv_append(k, v, layer_stride, block_stride, num_layers, h, head_dim, block_size, table, seq_len, active,
              refcount, free_list, free_count, new_k, new_v):
    """Paged KV append (reading R35) on copies. Returns (status, k, v, table, seq_len, refcount,
    free_list, free_count)."""
    k, v = _c(k, np.uint16).copy(), _c(v, np.uint16).copy()
    tab, sl = _c(table, np.int32).copy(), _c(seq_len, np.int32).copy()
    rc, fl = _c(refcount, np.int32).copy(), _c(free_list, np.int32).copy()
    fc = np.asarray([free_count], np.int64)
    act = None if active is None else _c(active, np.uint8)
    nk, nv = _c(new_k, np.uint16), _c(new_v, np.uint16)
    st = lib().oracle_kv_append(_p(k), _p(v), layer_stride, block_stride, num_layers, h, head_dim, block_size,
                                _p(tab), tab.shape[1], tab.shape[0], _p(sl), None if act is None else _p(act),
                                _p(rc), rc.size, _p(fl), _p(fc), _p(nk), _p(nv))
    return st, k, v, tab, sl, rc, fl, int(fc[0])


def paged_attention(k, v, layer_stride, block_stride, layer, h, head_dim, block_size, q, num_q_heads, table,
                    seq_len, scale):
    """fp64 decode attention through the block table (reading R36): out [S][hq][d_h]."""
    k, v, q = _c(k, np.uint16), _c(v, np.uint16), _c(q, np.uint16)
    tab, sl = _c(table, np.int32), _c(seq_len, np.int32)
    out = np.zeros((sl.size, num_q_heads, head_dim), np.float64)
    st = lib().oracle_paged_attention(_p(k), _p(v), layer_stride, block_stride, layer, h, head_dim, block_size,
                                      _p(q), num_q_heads, _p(tab), tab.shape[1], _p(sl), sl.size, scale, _p(out))
    if st != 0:
        raise ValueError("paged_attention: invalid arguments")
    return out


def admit(prompt_len, reserve, block_size, free_blocks):
    """FCFS block-budget admission (reading R37): (admitted, blocks_used)."""
    pl = _c(prompt_len, np.int32)
    used = np.zeros(1, np.int64)
    n = lib().oracle_admit(_p(pl), pl.size, reserve, block_size, free_blocks, _p(used))
    return int(n), int(used[0])
