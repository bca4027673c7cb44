"""GPU parity of the f3/f4 analysis calls (memshare_all_pairs, memshare_similarity_ratio)."""
import numpy as np
import pytest

import oracle
from synth import kv, workloads

from _gpu_util import compare_distances, host_pool_from_device, make_path, oracle_candidates, oracle_steps

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_21433_b200 import build
    build.build()


@pytest.mark.parametrize("tau", [0.8, 0.9])
def test_similarity_ratio_parity(tau):
    import torch
    w = workloads.small(kv.KVShape(8, 4, 64, 16), 3, 6000, seed=4)
    p = make_path(w, with_pool=False)
    p.autosize(tau, top_k=1)
    p.segment()
    p.candidates(tau, top_k=1)
    red = p.similarity_ratio().cpu().numpy()
    torch.cuda.synchronize()
    assert p.read_status() == 0
    oc = oracle_candidates(w, oracle_steps(w), tau_s=tau, top_k=1)
    assert np.array_equal(red, oracle.similarity_ratio_counts(oc["matches"], 3))


def test_all_pairs_tiny_matrix():
    """All 496 block pairs of T0 through memshare_all_pairs + memshare_block_distance vs the oracle."""
    import torch
    from paper_2507_21433_b200.pipeline import Caps
    w = workloads.tiny(eta=0.05)
    p = make_path(w, caps=Caps(step=512, match=64, pair=496, target=31))
    p.all_pairs([0], [32])
    p.distance_call(0.5)
    torch.cuda.synchronize()
    assert p.read_status() == 0
    g = p.read_candidates()
    r = oracle.all_pairs(w.batch.seq_tok_off, [0], [32], w.table, 16)
    for k in r["pairs"]:
        assert np.array_equal(g["pairs"][k], r["pairs"][k]), k
    assert np.array_equal(g["target_off"], r["target_off"])
    kh, vh = host_pool_from_device(p.k_pool, p.v_pool)
    D = oracle.block_distance(kh, vh, p.pool.layer_stride, p.pool.block_stride, 2, 2, 2, 64, 16,
                              r["pairs"]["target_phys"], r["pairs"]["source_phys"])
    compare_distances(p.read_distance()["distance"], D)
