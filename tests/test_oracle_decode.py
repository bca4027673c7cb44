"""Pins for the oracle's f1 decode-loop functions: paged KV append (R35), decode attention
through the block table (R36) and block-budget admission (R37).

PAPER.md:276-284 (shared blocks are read through the block table by paged attention),
PAPER.md:177-193 (Theorem 1: replacing v_j by v_j' with ||v_j - v_j'|| < delta moves the output
by at most delta).
"""
import math

import numpy as np
import pytest

import oracle


def bf(x):
    a = np.asarray(x, np.float32)
    u = a.view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "value not bf16-exact"
    return (u >> 16).astype(np.uint16)


def unbf(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


N, H, DH, D = 2, 2, 8, 4          # layers, kv heads, head dim, block size
ROW = H * DH
SLICE = D * ROW


def empty_pool(nb):
    return np.zeros(N * nb * SLICE, np.uint16), np.zeros(N * nb * SLICE, np.uint16), nb * SLICE, SLICE


def new_tokens(S, seed):
    rng = np.random.default_rng(seed)
    return (bf((rng.integers(-16, 16, (N, S, H, DH)) * 0.25).astype(np.float32)),
            bf((rng.integers(-16, 16, (N, S, H, DH)) * 0.25).astype(np.float32)))


def test_kv_append_worked_example():
    """seq 0 (len 3) appends at offset 3 of its private tail block 2; seq 1 (len 4 = d) takes a
    fresh block from the END of the free list (9), LIFO; seq 2 is inactive."""
    nb = 10
    k, v, ls, bs = empty_pool(nb)
    table = np.full((3, 4), -1, np.int32)
    table[0, 0] = 2
    table[1, 0] = 5
    table[2, 0] = 6
    refcount = np.zeros(nb, np.int32)
    refcount[[2, 5, 6]] = 1
    free_list = np.asarray([7, 9, 0, 0], np.int32)
    nk, nv = new_tokens(3, 0)
    st, k2, v2, t2, sl2, rc2, fl2, fc2 = oracle.kv_append(k, v, ls, bs, N, H, DH, D, table, [3, 4, 1], [1, 1, 0],
                                                          refcount, free_list, 2, nk, nv)
    assert st == 0
    assert sl2.tolist() == [4, 5, 1]
    assert t2[1, 1] == 9 and rc2[9] == 1 and fc2 == 1 and t2[0, 1] == -1
    assert (t2 != table).sum() == 1 and (rc2 != refcount).sum() == 1
    for l in range(N):
        o0 = l * ls + 2 * bs + 3 * ROW
        o1 = l * ls + 9 * bs + 0 * ROW
        assert np.array_equal(k2[o0:o0 + ROW], nk[l, 0].ravel()) and np.array_equal(v2[o0:o0 + ROW], nv[l, 0].ravel())
        assert np.array_equal(k2[o1:o1 + ROW], nk[l, 1].ravel()) and np.array_equal(v2[o1:o1 + ROW], nv[l, 1].ravel())
    changed = np.flatnonzero(k2 != k)
    assert changed.size <= 2 * N * ROW                   # nothing else written


def test_kv_append_fills_blocks_in_order():
    """d appends to an empty sequence fill one block, the (d+1)-th takes the next free block."""
    nb = 6
    k, v, ls, bs = empty_pool(nb)
    table = np.full((1, 3), -1, np.int32)
    rc = np.zeros(nb, np.int32)
    fl = np.asarray([1, 4, 3], np.int32)
    fc, sl = 3, np.zeros(1, np.int32)
    for step in range(D + 1):
        nk, nv = new_tokens(1, step)
        st, k, v, table, sl, rc, fl, fc = oracle.kv_append(k, v, ls, bs, N, H, DH, D, table, sl, None, rc, fl, fc,
                                                           nk, nv)
        assert st == 0
    assert sl[0] == D + 1 and table[0, :2].tolist() == [3, 4] and fc == 1 and rc.tolist() == [0, 0, 0, 1, 1, 0]


@pytest.mark.parametrize("case,expect", [("no_free", 2), ("table_full", 2), ("shared_tail", 3), ("busy_free", 3)])
def test_kv_append_errors_change_nothing(case, expect):
    nb = 6
    k, v, ls, bs = empty_pool(nb)
    table = np.asarray([[1, -1], [2, -1]], np.int32)
    rc = np.asarray([0, 1, 1, 0, 0, 0], np.int32)
    fl = np.asarray([3, 4], np.int32)
    fc, sl = 2, np.asarray([4, 2], np.int32)
    if case == "no_free":
        fc = 0
    elif case == "table_full":
        sl = np.asarray([8, 2], np.int32)
    elif case == "shared_tail":
        rc[2] = 2
    elif case == "busy_free":
        rc[4] = 1
    nk, nv = new_tokens(2, 1)
    st, k2, v2, t2, sl2, rc2, fl2, fc2 = oracle.kv_append(k, v, ls, bs, N, H, DH, D, table, sl, None, rc, fl, fc, nk, nv)
    assert st == expect
    assert np.array_equal(k2, k) and np.array_equal(t2, table) and np.array_equal(sl2, sl)
    assert np.array_equal(rc2, rc) and fc2 == fc


# ------------------------------------------------------------------------------- attention
def att_pool(rng, nb, scale_k=0.25, scale_v=0.25):
    k = bf((rng.integers(-8, 8, N * nb * SLICE) * scale_k).astype(np.float32))
    v = bf((rng.integers(-8, 8, N * nb * SLICE) * scale_v).astype(np.float32))
    return k, v, nb * SLICE, SLICE


def rows(pool, ls, bs, layer, table_row, n, g):
    """[n][DH] rows of KV head g of a sequence, as float64 (test-side gather)."""
    out = np.zeros((n, DH))
    for j in range(n):
        b = table_row[j // D]
        o = layer * ls + b * bs + ((j % D) * H + g) * DH
        out[j] = unbf(pool[o:o + DH])
    return out


def test_attention_single_token_returns_v():
    rng = np.random.default_rng(0)
    k, v, ls, bs = att_pool(rng, 4)
    q = bf((rng.integers(-8, 8, (1, 4, DH)) * 0.5).astype(np.float32))
    tab = np.asarray([[3, 0]], np.int32)
    out = oracle.paged_attention(k, v, ls, bs, 1, H, DH, D, q, 4, tab, [1], 0.3)
    for qh in range(4):
        assert np.array_equal(out[0, qh], rows(v, ls, bs, 1, tab[0], 1, qh // 2)[0])


def test_attention_zero_query_and_identical_keys_give_mean():
    rng = np.random.default_rng(1)
    k, v, ls, bs = att_pool(rng, 4)
    tab = np.asarray([[2, 0, 3]], np.int32)
    n = 10
    mean = [rows(v, ls, bs, 0, tab[0], n, g).mean(0) for g in range(H)]
    q0 = np.zeros((1, 2, DH), np.uint16)
    out = oracle.paged_attention(k, v, ls, bs, 0, H, DH, D, q0, 2, tab, [n], 1.0)
    for g in range(H):
        assert np.allclose(out[0, g], mean[g], rtol=0, atol=1e-15)
    kc = k.copy()                                      # every key row of layer 0 equal
    r0 = kc[0:DH].copy()
    for j in range(0, ls, DH):
        kc[j:j + DH] = r0
    q = bf((rng.integers(-8, 8, (1, 2, DH)) * 0.5).astype(np.float32))
    out = oracle.paged_attention(kc, v, ls, bs, 0, H, DH, D, q, 2, tab, [n], 1.0)
    for g in range(H):
        assert np.allclose(out[0, g], mean[g], rtol=0, atol=1e-15)


def test_attention_two_tokens_closed_form():
    """scores 0 and 1 (q.k1 = 0, q.k2 = 1, scale 1): out = v1/(1+e) + v2 e/(1+e)."""
    nb = 1
    k = np.zeros(N * nb * SLICE, np.uint16)
    v = bf((np.random.default_rng(2).integers(-8, 8, N * nb * SLICE) * 0.25).astype(np.float32))
    ls, bs = nb * SLICE, SLICE
    one = bf(np.float32(1.0))
    k[(1 * H + 0) * DH + 0] = one                      # layer 0, token 1, head 0: k2 = e_0
    q = np.zeros((1, H, DH), np.uint16)
    q[0, 0, 0] = one
    out = oracle.paged_attention(k, v, ls, bs, 0, H, DH, D, q, H, np.zeros((1, 1), np.int32), [2], 1.0)
    v1, v2 = rows(v, ls, bs, 0, [0], 2, 0)
    e = math.e
    assert np.allclose(out[0, 0], v1 / (1 + e) + v2 * e / (1 + e), rtol=0, atol=1e-15)


def test_attention_dominant_key_and_gqa_mapping():
    rng = np.random.default_rng(3)
    k, v, ls, bs = att_pool(rng, 3)
    tab = np.asarray([[1, 2]], np.int32)
    q = np.zeros((1, 4, DH), np.uint16)
    # query heads 0,1 -> kv head 0; 2,3 -> kv head 1. Plant a key aligned with q at j = 5 (head 0)
    kk = k.copy()
    o = 0 * ls + 2 * bs + ((5 % D) * H + 0) * DH
    kk[o:o + DH] = bf(np.full(DH, 4.0, np.float32))
    q[0, :, :] = bf(np.full((4, DH), 4.0, np.float32))
    out = oracle.paged_attention(kk, v, ls, bs, 0, H, DH, D, q, 4, tab, [8], 1.0)
    v5 = rows(v, ls, bs, 0, tab[0], 8, 0)[5]
    assert np.allclose(out[0, 0], v5, atol=1e-12) and np.allclose(out[0, 1], v5, atol=1e-12)
    assert not np.allclose(out[0, 2], v5, atol=1e-3)   # kv head 1 does not see the planted key


def test_attention_physical_placement_invariance():
    """The same logical KV stored in other physical blocks gives a bit-identical output."""
    rng = np.random.default_rng(4)
    k, v, ls, bs = att_pool(rng, 4)
    q = bf((rng.integers(-8, 8, (1, 2, DH)) * 0.5).astype(np.float32))
    tab = np.asarray([[0, 1, 2]], np.int32)
    perm = np.asarray([3, 2, 0, 1])                    # logical block i moves to physical perm[i]
    k2, v2 = k.copy(), v.copy()
    for l in range(N):
        for i in range(4):
            k2[l * ls + perm[i] * bs:l * ls + perm[i] * bs + bs] = k[l * ls + i * bs:l * ls + i * bs + bs]
            v2[l * ls + perm[i] * bs:l * ls + perm[i] * bs + bs] = v[l * ls + i * bs:l * ls + i * bs + bs]
    a = oracle.paged_attention(k, v, ls, bs, 1, H, DH, D, q, 2, tab, [11], 0.5)
    b = oracle.paged_attention(k2, v2, ls, bs, 1, H, DH, D, q, 2, perm[tab], [11], 0.5)
    assert np.array_equal(a, b)


def test_theorem1_value_replacement_bound():
    """replacing v_j by v_j' (keys unchanged) moves o by at most max_j ||dv_j||."""
    rng = np.random.default_rng(5)
    k, v, ls, bs = att_pool(rng, 4)
    q = bf((rng.integers(-8, 8, (2, 2, DH)) * 0.5).astype(np.float32))
    tab = np.asarray([[0, 1, 2, 3], [3, 2, 1, 0]], np.int32)
    v2 = bf((unbf(v) + rng.integers(-2, 3, v.size) * 0.125).astype(np.float32))
    n = [13, 16]
    a = oracle.paged_attention(k, v, ls, bs, 0, H, DH, D, q, 2, tab, n, 0.35)
    b = oracle.paged_attention(k, v2, ls, bs, 0, H, DH, D, q, 2, tab, n, 0.35)
    for s in range(2):
        for g in range(H):
            dv = rows(v2, ls, bs, 0, tab[s], n[s], g) - rows(v, ls, bs, 0, tab[s], n[s], g)
            delta = np.linalg.norm(dv, axis=1).max()
            assert np.linalg.norm(a[s, g] - b[s, g]) <= delta + 1e-12


def test_attention_empty_sequence_is_zero():
    rng = np.random.default_rng(6)
    k, v, ls, bs = att_pool(rng, 2)
    q = bf((rng.integers(-8, 8, (1, 2, DH)) * 0.5).astype(np.float32))
    out = oracle.paged_attention(k, v, ls, bs, 0, H, DH, D, q, 2, np.zeros((1, 1), np.int32), [0], 1.0)
    assert np.all(out == 0.0)


# ------------------------------------------------------------------------------- admission
def test_admit_worked_examples():
    # needs: ceil(32/16)=2, ceil(12/16)=1, ceil(52/16)=4 -> with 5 free: 2 admitted, 3 used
    assert oracle.admit([30, 10, 50], 2, 16, 5) == (2, 3)
    assert oracle.admit([30, 10, 50], 2, 16, 7) == (3, 7)
    assert oracle.admit([100, 1], 0, 16, 3) == (0, 0)      # FCFS: no skipping past a request that does not fit
    assert oracle.admit([], 0, 16, 3) == (0, 0)
    assert oracle.admit([16, 16], 0, 16, 2) == (2, 2)      # exact fit
