"""Host logic: the one-buffer input layout a serving loop uploads per round (pipeline.pack_inputs).

Every part must come back bit-identical from its slice, the int64 parts must sit at even int32
offsets (8-byte aligned views), and the serving state (free count, block table, refcounts, free
list) must be one contiguous range so a single copy snapshots or restores it.
"""
import numpy as np

from paper_2507_21433_b200.pipeline import pack_inputs
from synth import kv, workloads


def test_pack_inputs_round_trip():
    w = workloads.small(kv.KVShape(2, 2, 64, 16), 3, 1500, seed=5)
    b = w.batch
    host, lay = pack_inputs(b.tokens, b.seq_tok_off, b.gen_start, b.final, w.table, w.refcount, w.free_list,
                            w.free_count)
    assert host.dtype == np.int32
    assert lay["seq_tok_off"] % 2 == 0 and lay["state"] % 2 == 0
    ns, nt = len(b.gen_start), len(b.tokens)
    assert np.array_equal(host[lay["seq_tok_off"]:lay["state"]].view(np.int64), b.seq_tok_off)
    st = host[lay["state"]:lay["tokens"]]
    assert int(st[:2].view(np.int64)[0]) == w.free_count
    t = w.table.size
    assert np.array_equal(st[2:2 + t].reshape(w.table.shape), w.table)
    assert np.array_equal(st[2 + t:2 + t + w.refcount.size], w.refcount)
    assert np.array_equal(st[2 + t + w.refcount.size:], w.free_list)
    assert np.array_equal(host[lay["tokens"]:lay["tokens"] + nt], b.tokens)
    assert np.array_equal(host[lay["gen_start"]:lay["gen_start"] + ns], b.gen_start)
    assert np.array_equal(host[lay["final"]:].view(np.uint8)[:ns], np.asarray(b.final, np.uint8))
    assert host.size == lay["final"] + (ns + 3) // 4
