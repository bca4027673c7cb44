"""GPU check of the symmetric-memory plumbing bench.py --mode headshard --collective p2p uses at
N > 1, exercised with a one-rank NCCL group on this GPU: symm.empty + rendezvous give the peer
pointer list, the device barrier runs on the stream, and memshare_block_distance_finalize_peers
reading [symmetric buffer, ordinary buffer] equals the device-side sum + FINALIZE bit for bit."""
import os
import socket

import numpy as np
import pytest

from synth import kv, workloads

from _gpu_util import make_path

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_symmetric_memory_finalize_peers_one_rank():
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed._symmetric_memory as symm
    from paper_2507_21433_b200 import _lib as L
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        shape = kv.KVShape(4, 8, 128, 16)
        w = workloads.small(shape, 2, 3000, seed=17)
        shards = [make_path(w, h_local=4, head_offset=h0) for h0 in (0, 4)]
        for p in shards:
            p.autosize(w.tau_s)
            p.segment()
            p.candidates(w.tau_s)
            p.alloc_partial()
        buf = symm.empty(shards[0].partial_sq.numel(), dtype=torch.float32, device=dev)
        hdl = symm.rendezvous(buf, dist.group.WORLD.group_name)
        assert len(list(hdl.buffer_ptrs)) == 1
        shards[0].partial_sq = buf
        for p in shards:
            p.distance_call(w.tau_b, L.DIST_PARTIAL)
        hdl.barrier(channel=0)
        ptrs = torch.tensor([int(hdl.buffer_ptrs[0]), shards[1].partial_sq.data_ptr()], dtype=torch.int64, device=dev)
        p = shards[0]
        p.finalize_peers(w.tau_b, ptrs, 2)
        hdl.barrier(channel=1)
        torch.cuda.synchronize()
        assert p.read_status() == 0
        gp = p.read_distance()
        p.partial_sq += shards[1].partial_sq
        p.distance_call(w.tau_b, L.DIST_FINALIZE)
        torch.cuda.synchronize()
        gd = p.read_distance()
        assert gd["distance"].size > 0
        assert np.array_equal(gp["distance"], gd["distance"])
        for k in gd["decisions"]:
            assert np.array_equal(gp["decisions"][k], gd["decisions"][k]), k
    finally:
        dist.destroy_process_group()
