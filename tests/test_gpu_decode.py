"""f1 decode-loop integration on the GPU: paged KV append and decode attention through the
(remapped) block table against the oracle; Theorem-1 drift bound; admission with freed blocks.
PAPER.md:276-284, :322, :177-193; R35-R37."""
import math

import numpy as np
import pytest

import oracle
from synth import decode as sd
from synth import kv, workloads

pytestmark = pytest.mark.gpu

ATT_ATOL = 1e-4      # |o_gpu - o_oracle| <= ATT_ATOL * max|v|: fp32 sums of <= 4k terms + ex2.approx


def _torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def unbf(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def dev_u16(t, a):
    return t.as_tensor(np.ascontiguousarray(a, np.uint16).view(np.int16), device="cuda")


def host_u16(x):
    return x.view(_torch().int16).cpu().numpy().view(np.uint16)


def run_attention(L, pool_k, pool_v, ls, bs, nb, shape, layer, q_bits, hq, table, seq_len, scale):
    torch = _torch()
    S = len(seq_len)
    dims = L.Dims(shape.num_layers, shape.num_kv_heads, shape.num_kv_heads, shape.head_dim, shape.block_size)
    pool = L.KVPool(pool_k.data_ptr(), pool_v.data_ptr(), ls, bs, nb, 0)
    max_len = int(max(1, np.max(seq_len)))
    q = dev_u16(torch, q_bits)
    tab = torch.as_tensor(np.ascontiguousarray(table, np.int32), device="cuda")
    sl = torch.as_tensor(np.ascontiguousarray(seq_len, np.int32), device="cuda")
    out = torch.full((S, hq, shape.head_dim), float("nan"), dtype=torch.float32, device="cuda")
    ws = torch.empty(L.paged_attention_workspace_size(dims, S, hq, max_len), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    assert L.paged_attention_decode(pool, dims, layer, q, hq, tab, table.shape[1], sl, S, max_len, scale, out, ws,
                                    st) == 0
    torch.cuda.synchronize()
    assert st.item() == 0
    return out.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("shape,hq,S,maxlen", [(kv.KVShape(3, 8, 128, 16), 40, 12, 3000),
                                                (kv.KVShape(2, 2, 64, 16), 8, 12, 3000),
                                                (kv.KVShape(2, 10, 128, 16), 40, 12, 3000),
                                                # enough split CTAs for 32-block (512-token) and
                                                # 64-block (1,024-token) work items
                                                (kv.KVShape(2, 8, 128, 16), 40, 20, 3000),
                                                (kv.KVShape(2, 8, 128, 16), 40, 24, 6000)])
def test_attention_vs_oracle_ragged(shape, hq, S, maxlen):
    """Ragged lengths (0, 1, d-1, d, d+1, 255-257 chunk edges, work-item edges 511-513 / 1023-1025 /
    2047-2049, random up to maxlen) through a shuffled block table; GQA groups of 5, 4 and 4. The
    host picks the work item (16 / 32 / 64 blocks) from the grid size: the last two cases take 32
    and 64."""
    torch = _torch()
    from paper_2507_21433_b200 import _lib as L
    rng = np.random.default_rng(hq + S + maxlen)
    seq_len = sd.ragged_lengths(rng, S, maxlen)
    edges = [511, 512, 513, 1023, 1024, 1025, 2047, 2048, 2049]
    if S >= 8 + len(edges):                      # after ragged_lengths' own 8 edge lengths
        seq_len[8:8 + len(edges)] = edges
    stride = int(math.ceil(maxlen / 16)) + 1
    need = [int(math.ceil(n / 16)) for n in seq_len]
    nb = sum(need) + 5
    perm = rng.permutation(nb)
    table = np.full((S, stride), -1, np.int32)
    c = 0
    for s in range(S):
        table[s, :need[s]] = perm[c:c + need[s]]
        c += need[s]
    sl_ = shape.block_size * shape.num_kv_heads * shape.head_dim
    kb = sd.gaussian_bf16(rng, shape.num_layers * nb * sl_)
    vb = sd.gaussian_bf16(rng, shape.num_layers * nb * sl_)
    qb = sd.gaussian_bf16(rng, (S, hq, shape.head_dim))
    k, v = dev_u16(torch, kb), dev_u16(torch, vb)
    scale = 1.0 / math.sqrt(shape.head_dim)
    for layer in range(shape.num_layers):
        got = run_attention(L, k, v, nb * sl_, sl_, nb, shape, layer, qb, hq, table, seq_len, scale)
        exp = oracle.paged_attention(kb, vb, nb * sl_, sl_, layer, shape.num_kv_heads, shape.head_dim,
                                     shape.block_size, qb, hq, table, seq_len, scale)
        vmax = np.abs(unbf(vb)).max()
        err = np.abs(got - exp).max()
        assert err <= ATT_ATOL * vmax, f"layer {layer}: max abs err {err:.3e}"
        assert np.all(got[seq_len == 0] == 0.0)


def _kv_state(rng, shape, S, nb, stride):
    lens = rng.integers(0, 4 * shape.block_size, S).astype(np.int32)
    lens[:3] = [0, 16, 31]
    table = np.full((S, stride), -1, np.int32)
    rc = np.zeros(nb, np.int32)
    free = list(rng.permutation(nb))
    for s in range(S):
        for lb in range(int(math.ceil(lens[s] / shape.block_size))):
            b = free.pop()
            table[s, lb] = b
            rc[b] = 1
    fl = np.zeros(nb, np.int32)
    fl[:len(free)] = free
    return lens, table, rc, fl, len(free)


def test_kv_append_vs_oracle_many_steps():
    torch = _torch()
    from paper_2507_21433_b200 import _lib as L
    shape = kv.KVShape(3, 8, 128, 16)
    rng = np.random.default_rng(7)
    S, nb, stride = 37, 400, 12
    lens, table, rc, fl, fc = _kv_state(rng, shape, S, nb, stride)
    sl_ = shape.slice_elems
    kb = sd.gaussian_bf16(rng, shape.num_layers * nb * sl_)
    vb = sd.gaussian_bf16(rng, shape.num_layers * nb * sl_)
    dims = L.Dims(shape.num_layers, shape.num_kv_heads, shape.num_kv_heads, shape.head_dim, shape.block_size)
    k, v = dev_u16(torch, kb), dev_u16(torch, vb)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")
    d_tab, d_len, d_rc, d_fl = t(table, torch.int32), t(lens, torch.int32), t(rc, torch.int32), t(fl, torch.int32)
    d_fc = torch.tensor([fc], dtype=torch.int64, device="cuda")
    ws = torch.empty(L.kv_append_workspace_size(S), dtype=torch.uint8, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    o = (kb, vb, table, lens, rc, fl, fc)
    for step in range(20):
        active = (rng.random(S) < 0.8).astype(np.uint8)
        nk = sd.gaussian_bf16(rng, (shape.num_layers, S, shape.num_kv_heads, shape.head_dim))
        nv = sd.gaussian_bf16(rng, (shape.num_layers, S, shape.num_kv_heads, shape.head_dim))
        assert L.kv_append(k, v, nb * sl_, sl_, nb, dims, d_tab, stride, S, d_len, t(active, torch.uint8), d_rc, d_fl,
                           d_fc, dev_u16(torch, nk), dev_u16(torch, nv), ws, st) == 0
        r = oracle.kv_append(o[0], o[1], nb * sl_, sl_, shape.num_layers, shape.num_kv_heads, shape.head_dim,
                             shape.block_size, o[2], o[3], active, o[4], o[5], o[6], nk, nv)
        assert r[0] == 0
        o = r[1:]
        torch.cuda.synchronize()
        assert st.item() == 0
        assert np.array_equal(d_tab.cpu().numpy(), o[2]) and np.array_equal(d_len.cpu().numpy(), o[3])
        assert np.array_equal(d_rc.cpu().numpy(), o[4]) and int(d_fc.item()) == o[6]
        assert np.array_equal(d_fl.cpu().numpy()[:o[6]], o[5][:o[6]])
    assert np.array_equal(host_u16(k), o[0]) and np.array_equal(host_u16(v), o[1])
    # capacity: more fresh blocks needed than free -> status CAPACITY, state untouched
    d_fc.fill_(0)
    d_len.copy_(t(np.full(S, 32, np.int32), torch.int32))
    before = (d_tab.clone(), d_rc.clone(), host_u16(k))
    nk = sd.gaussian_bf16(rng, (shape.num_layers, S, shape.num_kv_heads, shape.head_dim))
    assert L.kv_append(k, v, nb * sl_, sl_, nb, dims, d_tab, stride, S, d_len, None, d_rc, d_fl, d_fc,
                       dev_u16(torch, nk), dev_u16(torch, nk), ws, st) == 0
    torch.cuda.synchronize()
    assert st.item() == L.CAPACITY
    assert torch.equal(d_tab, before[0]) and torch.equal(d_rc, before[1]) and np.array_equal(host_u16(k), before[2])
    assert np.all(d_len.cpu().numpy() == 32)


def test_remap_then_decode_attention_and_theorem1_drift():
    """A MemShare round remaps target blocks onto sources; decode attention through the remapped
    table equals the oracle on that table, and its drift from the unshared output obeys the
    Theorem-1 bound ||do|| <= (exp(2 eta) - 1) max||v|| + delta, eta = scale ||q|| max||dk||,
    delta = max||dv|| over the replaced token rows (PAPER.md:179-191 with softmax's ratio bound)."""
    torch = _torch()
    from paper_2507_21433_b200 import _lib as L
    from _gpu_util import make_path
    shape = kv.KVShape(4, 8, 128, 16)
    w = workloads.small(shape, 3, 3000, seed=5, eta=0.05)
    p = make_path(w)
    p.autosize(w.tau_s)
    table0 = p.table.cpu().numpy().copy()
    p.round(w.tau_s, w.tau_b)
    torch.cuda.synchronize()
    st = p.read_state()
    assert st["num_freed"] > 0
    table1 = st["table"]
    assert (table1 != table0).sum() > 0
    lens = np.diff(w.batch.seq_tok_off).astype(np.int32)
    rng = np.random.default_rng(1)
    hq = 40
    qb = sd.gaussian_bf16(rng, (len(lens), hq, shape.head_dim))
    scale = 1.0 / math.sqrt(shape.head_dim)
    kb, vb = host_u16(p.k_pool), host_u16(p.v_pool)
    ls, bs = p.pool.layer_stride, p.pool.block_stride
    for layer in (0, shape.num_layers - 1):
        o0 = run_attention(L, p.k_pool, p.v_pool, ls, bs, w.num_blocks, shape, layer, qb, hq, table0, lens, scale)
        o1 = run_attention(L, p.k_pool, p.v_pool, ls, bs, w.num_blocks, shape, layer, qb, hq, table1, lens, scale)
        e1 = oracle.paged_attention(kb, vb, ls, bs, layer, shape.num_kv_heads, shape.head_dim, shape.block_size, qb,
                                    hq, table1, lens, scale)
        vmax_all = np.abs(unbf(vb)).max()
        assert np.abs(o1 - e1).max() <= ATT_ATOL * vmax_all
        G = hq // shape.num_kv_heads
        K = unbf(kb).reshape(shape.num_layers, -1, 16, shape.num_kv_heads, shape.head_dim)[layer]
        V = unbf(vb).reshape(shape.num_layers, -1, 16, shape.num_kv_heads, shape.head_dim)[layer]
        for s in range(len(lens)):
            changed = np.flatnonzero(table1[s] != table0[s])
            if changed.size == 0:
                assert np.array_equal(o0[s], o1[s])
                continue
            j = np.arange(lens[s])
            Ka, Kb = K[table0[s, j // 16], j % 16], K[table1[s, j // 16], j % 16]      # [len, h, d_h]
            Va, Vb = V[table0[s, j // 16], j % 16], V[table1[s, j // 16], j % 16]
            dk = np.linalg.norm(Ka - Kb, axis=2).max(axis=0)                          # [h]
            dv = np.linalg.norm(Va - Vb, axis=2).max(axis=0)
            vmax = np.linalg.norm(Va, axis=2).max(axis=0)
            for qh in range(hq):
                g = qh // G
                eta = scale * np.linalg.norm(unbf(qb[s, qh])) * dk[g]
                bound = (math.exp(2 * eta) - 1) * vmax[g] + dv[g]
                drift = np.linalg.norm(o1[s, qh] - o0[s, qh])
                assert drift <= bound + 2 * ATT_ATOL * vmax_all, (s, qh, drift, bound)


def test_freed_blocks_admit_more_and_feed_kv_append():
    """Blocks freed by remap raise the admission budget (memshare_admit) and are the blocks the
    next appends take (LIFO from the free list)."""
    torch = _torch()
    from paper_2507_21433_b200 import _lib as L
    from _gpu_util import make_path
    shape = kv.KVShape(2, 8, 128, 16)
    w = workloads.small(shape, 3, 3000, seed=8, eta=0.05)
    p = make_path(w)
    p.autosize(w.tau_s)
    fc0 = int(p.free_count.item())
    p.round(w.tau_s, w.tau_b)
    st = p.read_state()
    freed = st["num_freed"]
    assert freed > 0 and st["free_count"] == fc0 + freed
    queue = [40] * 200
    n0, _ = L.admit(queue, 16, 16, fc0)
    n1, _ = L.admit(queue, 16, 16, st["free_count"])
    assert n1 > n0 and (n1 - n0) * 4 <= freed + 4
    # every sequence appends until it needs a fresh block: those come from the END of the free
    # list, in sequence order (a wider table gives the rows room to grow)
    S = w.batch.num_seqs
    wide = torch.full((S, p.table_stride + 2), -1, dtype=torch.int32, device="cuda")
    wide[:, :p.table_stride] = p.table
    lens = p.seq_tok_off.diff().to(torch.int32)
    to_boundary = int(((16 - lens % 16) % 16).max().item()) + 1
    dims = L.Dims(shape.num_layers, shape.num_kv_heads, shape.num_kv_heads, shape.head_dim, shape.block_size)
    ws = torch.empty(L.kv_append_workspace_size(S), dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(0)
    fl = st["free_list"]
    fc1 = st["free_count"]
    for _ in range(to_boundary):
        nk = dev_u16(torch, sd.gaussian_bf16(rng, (shape.num_layers, S, shape.num_kv_heads, shape.head_dim)))
        assert L.kv_append(p.k_pool, p.v_pool, p.pool.layer_stride, p.pool.block_stride, w.num_blocks, dims, wide,
                           p.table_stride + 2, S, lens, None, p.refcount, p.free_list, p.free_count, nk, nk, ws,
                           p.status) == 0
    torch.cuda.synchronize()
    assert p.status.item() == 0
    assert int(p.free_count.item()) == fc1 - S
    tab = wide.cpu().numpy()
    ln = lens.cpu().numpy()
    got = sorted(int(tab[s, (ln[s] - 1) // 16]) for s in range(S))
    assert got == sorted(int(b) for b in fl[fc1 - S:fc1])     # the top S entries of the free list
