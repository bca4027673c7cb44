"""Child process of tests/test_gpu_sanitizer.py: every ABI call of the library on small inputs,
run under compute-sanitizer (memcheck / racecheck / synccheck / initcheck). Device status must be
OK after each phase; prints "ok". Kept small: the sanitizer serialises and instruments every
access (~100x slower)."""
import math
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from synth import kv, workloads  # noqa: E402


def main():
    from _gpu_util import make_path
    from paper_2507_21433_b200 import _lib as L
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    small = kv.KVShape(2, 2, 64, 16)
    # the path: offline ALL (fused fill), CROSS, online LAST (8-CTA clusters, global count table
    # off), RANGE, both metrics, PARTIAL -> FINALIZE, the remap
    w = workloads.small(small, 2, 2200, seed=5)
    p = make_path(w)
    for cur_mode, pairing in ((oracle.CUR_ALL, L.PAIR_ALIGNED), (oracle.CUR_ALL, L.PAIR_CROSS),
                              (oracle.CUR_LAST, L.PAIR_ALIGNED)):
        p.autosize(0.5, pairing=pairing, cur_mode=cur_mode)
        p.round(0.5, w.tau_b, pairing=pairing, cur_mode=cur_mode)
        torch.cuda.synchronize()
        assert p.read_status() == 0, (cur_mode, pairing, p.read_status())
    p.autosize(0.5, cur_mode=oracle.CUR_RANGE, cur_begin=[1, 2], cur_end=[6, 9])
    p.round(0.5, w.tau_b, cur_mode=oracle.CUR_RANGE, cur_begin=[1, 2], cur_end=[6, 9])
    p.distance_call(w.tau_b, L.DIST_FULL, metric=L.METRIC_COSINE)
    p.alloc_partial()
    p.distance_call(w.tau_b, L.DIST_PARTIAL)
    p.distance_call(w.tau_b, L.DIST_FINALIZE)
    torch.cuda.synchronize()
    assert p.read_status() == 0, p.read_status()
    # f4 / f3 analysis calls
    p.similarity_ratio()
    p.set_caps(p.caps.__class__(step=p.caps.step, match=p.caps.match, pair=4096, target=512))
    p.all_pairs([0, 3], [20, 30])
    p.distance_call(w.tau_b)
    torch.cuda.synchronize()
    assert p.read_status() == 0, p.read_status()
    # f1: KV append (with a block allocation) and decode attention through the table
    S, N, h, dh, d, hq = 3, 2, 2, 64, 16, 4
    nbs = 4
    nb = S * nbs + 4
    sl = d * h * dh
    k = torch.randn(N * nb * sl, dtype=torch.bfloat16, device=dev)
    v = torch.randn(N * nb * sl, dtype=torch.bfloat16, device=dev)
    table = torch.full((S, nbs), -1, dtype=torch.int32, device=dev)
    table[:, :2] = torch.arange(2 * S, dtype=torch.int32, device=dev).view(S, 2)
    seq_len = torch.tensor([32, 20, 31], dtype=torch.int32, device=dev)
    rc = torch.zeros(nb, dtype=torch.int32, device=dev)
    rc[:2 * S] = 1
    fl = torch.arange(2 * S, nb, dtype=torch.int32, device=dev)
    fc = torch.tensor([nb - 2 * S], dtype=torch.int64, device=dev)
    dims = L.Dims(N, h, h, dh, d)
    nk = torch.randn(N * S * h * dh, dtype=torch.bfloat16, device=dev)
    nv = torch.randn_like(nk)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(max(1, L.kv_append_workspace_size(S)), dtype=torch.uint8, device=dev)
    L.check(L.kv_append(k, v, nb * sl, sl, nb, dims, table, nbs, S, seq_len, None, rc, fl, fc, nk, nv, ws, st))
    torch.cuda.synchronize()
    assert st.item() == 0, st.item()
    q = torch.randn(S * hq * dh, dtype=torch.bfloat16, device=dev)
    out = torch.empty(S * hq * dh, dtype=torch.float32, device=dev)
    pool = L.KVPool(k.data_ptr(), v.data_ptr(), nb * sl, sl, nb, 0)
    ws2 = torch.empty(L.paged_attention_workspace_size(dims, S, hq, 64), dtype=torch.uint8, device=dev)
    L.check(L.paged_attention_decode(pool, dims, 1, q, hq, table, nbs, seq_len, S, 64, 1 / math.sqrt(dh), out, ws2,
                                     st))
    torch.cuda.synchronize()
    assert st.item() == 0, st.item()
    assert np.isfinite(out.cpu().numpy()).all()
    print("ok", flush=True)


if __name__ == "__main__":
    main()
