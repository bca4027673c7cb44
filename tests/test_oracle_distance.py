"""Pins for the oracle's Stage-2 block distance and selection (a5, a6).

PAPER.md:237-248 (Alg. 1 Stage 2): D = (1/N) sum_l (||K_l[B1]-K_l[B2]|| + ||V_l[B1]-V_l[B2]||)/(2dh).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from synth import kv, traces

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bf16_bits(x):
    """float -> bf16 bits (values used here are exactly representable)."""
    a = np.asarray(x, np.float32)
    u = a.view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "value not bf16-exact"
    return (u >> 16).astype(np.uint16)


def pool_from_values(vals_k, vals_v):
    """vals: float32 [N, num_blocks, slice] -> layer-major bf16 pools + strides."""
    N, nb, sl = vals_k.shape
    return bf16_bits(vals_k).ravel(), bf16_bits(vals_v).ravel(), nb * sl, sl


def test_spec_worked_example():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["distance"][0]
    N, d, h, dh = ex["N"], ex["d"], ex["h"], ex["d_h"]
    sl = d * h * dh
    a = np.zeros((N, 2, sl), np.float32)
    a[:, 1, :] = ex["offset"]
    k, v, ls, bs = pool_from_values(a, a)
    D = oracle.block_distance(k, v, ls, bs, N, h, h, dh, d, [0], [1])
    assert D[0] == ex["D"]
    sk, sv = oracle.partial_sq(k, v, ls, bs, N, h, dh, d, [0], [1])
    assert sk[0, 0] == 4.0 and sv[0, 0] == 4.0           # Delta_K = Delta_V = 2


@pytest.mark.parametrize("shape,c,expected", [
    (kv.TINY, 1.0, math.sqrt(2.0)),                # sqrt(64/(16*2)) = sqrt(2)
    (kv.QWEN32B, 0.5, 0.5),                        # 0.5 * sqrt(128/(16*8)) = 0.5
    (kv.PHI4, 1.0, math.sqrt(128 / 160)),          # sqrt(128/(16*10)) = 0.894427191
])
def test_constant_offset_closed_form(shape, c, expected):
    """If every element of B1 differs from B2 by c in every layer, ||.||_F = |c| sqrt(d h d_h) and
    D = (1/N) sum_l 2|c| sqrt(d h d_h) / (2 d h) = |c| sqrt(d_h / (d h))."""
    rng = np.random.default_rng(0)
    N, sl = shape.num_layers, shape.slice_elems
    base = (rng.integers(-8, 8, size=(N, 1, sl)) * 0.25).astype(np.float32)
    vals = np.concatenate([base, base + np.float32(c)], axis=1)
    k, v, ls, bs = pool_from_values(vals, vals[:, :, ::-1].copy())
    D = oracle.block_distance(k, v, ls, bs, N, shape.num_kv_heads, shape.num_kv_heads, shape.head_dim,
                              shape.block_size, [1], [0])
    assert abs(D[0] - expected) <= 1e-12 * expected


def test_layer_mean_closed_form():
    """c_l = l + 1 in layer l -> D = (N+1)/2 * sqrt(d_h/(d h)) (tests the 1/N mean)."""
    sh = kv.TINY
    N, sl = sh.num_layers, sh.slice_elems
    vals = np.zeros((N, 2, sl), np.float32)
    for l in range(N):
        vals[l, 1, :] = l + 1
    k, v, ls, bs = pool_from_values(vals, vals)
    D = oracle.block_distance(k, v, ls, bs, N, 2, 2, 64, 16, [0], [1])
    assert abs(D[0] - (N + 1) / 2 * math.sqrt(64 / 32)) < 1e-12


def _tiny_pool(eta=0.05, seed=0):
    b = traces.tiny_t0()
    tab, nbk = traces.identity_table(b, 16)
    k, v, ls, bs = kv.host_pool(kv.TINY, nbk)
    s_, l_, p_ = kv.table_blocks(b.seq_tok_off, tab, 16)
    kv.fill_blocks_host(k, v, ls, bs, kv.TINY, b.tokens, b.seq_tok_off, s_, l_, p_, seed=seed, eta=eta)
    return k, v, ls, bs, nbk


def test_all_pairs_tiny_vs_numpy_norm():
    """all 32*31/2 = 496 block pairs against numpy.linalg.norm in float64."""
    k, v, ls, bs, nbk = _tiny_pool()
    i, j = np.triu_indices(nbk, 1)
    D = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, i, j)
    assert D.size == 496
    f = lambda a: (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    K = f(k).reshape(2, nbk, -1)
    V = f(v).reshape(2, nbk, -1)
    ref = np.zeros(496)
    for l in range(2):
        ref += (np.linalg.norm(K[l, i] - K[l, j], axis=1) + np.linalg.norm(V[l, i] - V[l, j], axis=1)) / (2 * 16 * 2)
    ref /= 2
    assert np.allclose(D, ref, rtol=1e-13, atol=0)


def test_pseudometric_properties():
    k, v, ls, bs, nbk = _tiny_pool()
    rng = np.random.default_rng(3)
    a, b, c = (rng.integers(0, nbk, 300) for _ in range(3))
    dab = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, a, b)
    dba = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, b, a)
    dbc = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, b, c)
    dac = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, a, c)
    daa = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, a, a)
    assert np.all(daa == 0.0)
    assert np.array_equal(dab, dba)
    assert np.all(dac <= dab + dbc + 1e-12)


def test_scaling_by_two_doubles_distance_exactly():
    k, v, ls, bs, nbk = _tiny_pool()
    f = lambda a: (a.astype(np.uint32) << 16).view(np.float32)
    k2 = bf16_bits(f(k) * 2)
    v2 = bf16_bits(f(v) * 2)
    a, b = np.arange(0, 16), np.arange(16, 32)
    d1 = oracle.block_distance(k, v, ls, bs, 2, 2, 2, 64, 16, a, b)
    d2 = oracle.block_distance(k2, v2, ls, bs, 2, 2, 2, 64, 16, a, b)
    assert np.array_equal(d2, 2 * d1)


def test_head_sharded_partials_sum_to_unsharded():
    """sum over heads decomposes: partial squares of head shards add up to the full ones
    (the basis of the head-sharded mode)."""
    sh = kv.KVShape(3, 4, 16, 8)
    b = traces.make_batch(2, 1, 200, 0, 8, vocab=500)
    tab, nbk = traces.identity_table(b, 8)
    s_, l_, p_ = kv.table_blocks(b.seq_tok_off, tab, 8)
    full = kv.host_pool(sh, nbk)
    kv.fill_blocks_host(full[0], full[1], full[2], full[3], sh, b.tokens, b.seq_tok_off, s_, l_, p_, 9, 0.05)
    a, c = np.arange(0, 12), np.arange(12, 24)
    skf, svf = oracle.partial_sq(full[0], full[1], full[2], full[3], 3, 4, 16, 8, a, c)
    sk_sum, sv_sum = 0, 0
    for h0 in (0, 2):
        sh_ = kv.host_pool(sh, nbk, h_local=2)
        kv.fill_blocks_host(sh_[0], sh_[1], sh_[2], sh_[3], sh, b.tokens, b.seq_tok_off, s_, l_, p_, 9, 0.05,
                            h_local=2, head_offset=h0)
        sk, sv = oracle.partial_sq(sh_[0], sh_[1], sh_[2], sh_[3], 3, 2, 16, 8, a, c)
        sk_sum, sv_sum = sk_sum + sk, sv_sum + sv
    assert np.allclose(sk_sum, skf, rtol=1e-14) and np.allclose(sv_sum, svf, rtol=1e-14)
    D = oracle.finalize(sk_sum, sv_sum, 3, 8, 4)
    Df = oracle.block_distance(full[0], full[1], full[2], full[3], 3, 4, 4, 16, 8, a, c)
    assert np.allclose(D, Df, rtol=1e-14)


def test_doubling_head_dim_raises_distance():
    """d_h is not in the denominator, so the same per-element difference gives a
    larger D at larger d_h (by sqrt(2))."""
    out = []
    for dh in (8, 16):
        sl = 2 * 1 * dh
        vals = np.zeros((1, 2, sl), np.float32)
        vals[:, 1] = 1.0
        k, v, ls, bs = pool_from_values(vals, vals)
        out.append(oracle.block_distance(k, v, ls, bs, 1, 1, 1, dh, 2, [0], [1])[0])
    assert out[1] > out[0] and abs(out[1] / out[0] - math.sqrt(2)) < 1e-12


def test_generator_statistical_closed_forms():
    """E[D_dup] ~ eta*sqrt(2 d_h/(d h)); E[D_random] ~ sqrt(1+eta^2)*sqrt(2 d_h/(d h))
    (derived for unit-variance base/noise)."""
    sh = kv.KVShape(4, 2, 64, 16)
    eta = 0.05
    b = traces.make_batch(1, 1, 4096, 0, 16, m_max=0.0)
    tab, nbk = traces.identity_table(b, 16)
    s_, l_, p_ = kv.table_blocks(b.seq_tok_off, tab, 16)
    k, v, ls, bs = kv.host_pool(sh, nbk)
    kv.fill_blocks_host(k, v, ls, bs, sh, b.tokens, b.seq_tok_off, s_, l_, p_, 4, eta)
    seg = oracle.segment_steps(b.tokens, b.seq_tok_off, b.gen_start, b.final, b.delim_ids)
    r = oracle.step_candidates(b.tokens, b.seq_tok_off, seg, b.delim_ids, tab, 16, 0.99)
    p = r["pairs"]
    assert p["seq"].size > 20
    D = oracle.block_distance(k, v, ls, bs, 4, 2, 2, 64, 16, p["target_phys"], p["source_phys"])
    scale = math.sqrt(2 * 64 / (16 * 2))
    # exact copies (m = 0): every aligned block pair is identical tokens -> pure noise distance
    assert abs(np.median(D) / (eta * scale) - 1) < 0.03
    rng = np.random.default_rng(0)
    a, c = rng.integers(0, nbk - 1, 200), rng.integers(0, nbk - 1, 200)
    keep = a != c
    Dr = oracle.block_distance(k, v, ls, bs, 4, 2, 2, 64, 16, a[keep], c[keep])
    assert abs(np.median(Dr) / (math.sqrt(1 + eta ** 2) * scale) - 1) < 0.03


def test_select_argmin_ties_and_strict_threshold():
    D = np.array([0.3, 0.1, 0.1, 0.5, 0.25, 0.25], np.float64)
    toff = np.array([0, 3, 4, 6])
    sl = np.array([9, 7, 4, 1, 3, 2], np.int32)
    best, acc, under = oracle.select(D, toff, sl, 0.25)
    assert best.tolist() == [2, 3, 5]            # tie 0.1/0.1 -> smaller source logical 4; tie 0.25 -> logical 2
    assert acc.tolist() == [1, 0, 0]             # 0.25 is not < 0.25 (strict, reading R21)
    assert under.tolist() == [0, 1, 1, 0, 0, 0]


# ------------------------------------------------------------------- f2: cosine block metric
def test_cosine_metric_pins():
    """cosine measures only angular alignment. Identical -> 0; a scaled copy
    (x2, bf16-exact) -> 0 (magnitude ignored, unlike Alg. 1's D); negated -> 2; orthogonal -> 1."""
    rng = np.random.default_rng(5)
    sl = 2 * 2 * 8
    base = (rng.integers(-8, 8, (1, 1, sl)) * 0.25).astype(np.float32)
    orth = np.zeros_like(base)
    half = sl // 2
    b1 = base.copy(); b1[..., half:] = 0
    orth[..., half:] = 1.0                                  # disjoint supports -> dot 0
    vals = np.concatenate([b1, b1, 2 * b1, -b1, orth], axis=1)
    k, v, ls, bs = pool_from_values(vals, vals)
    D = oracle.block_cosine(k, v, ls, bs, 1, 2, 8, 2, [0, 0, 0, 0], [1, 2, 3, 4])
    assert D[0] == 0.0 and abs(D[1]) < 1e-15 and abs(D[2] - 2.0) < 1e-15 and D[3] == 1.0
    # against numpy on random blocks
    k2, v2, ls2, bs2, nbk = _tiny_pool()
    f = lambda a: (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    K = f(k2).reshape(2, nbk, -1)
    V = f(v2).reshape(2, nbk, -1)
    i, j = np.arange(0, 10), np.arange(10, 20)
    cos = lambda A, B: (A * B).sum(-1) / np.sqrt((A * A).sum(-1) * (B * B).sum(-1))
    ref = 1 - np.mean([(cos(K[l, i], K[l, j]) + cos(V[l, i], V[l, j])) / 2 for l in range(2)], axis=0)
    got = oracle.block_cosine(k2, v2, ls2, bs2, 2, 2, 64, 16, i, j)
    assert np.allclose(got, ref, rtol=0, atol=1e-13)
    assert np.array_equal(got, oracle.block_cosine(k2, v2, ls2, bs2, 2, 2, 64, 16, j, i))
