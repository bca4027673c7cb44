"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol that
include/memshare.h declares, and rejects host-detectable bad arguments without touching CUDA."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "memshare.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2507_21433_b200 import build
    build.build()
    from paper_2507_21433_b200 import _lib
    return _lib


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(memshare_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_four_calls():
    fns = declared_functions()
    for f in ("memshare_segment_steps", "memshare_step_candidates", "memshare_block_distance", "memshare_remap"):
        assert f in fns


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (memshare_\w+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    for f in declared_functions():
        assert hasattr(lib.lib, f)


def test_sass_is_sm100a_with_bulk_copy(lib):
    sass = subprocess.check_output(["cuobjdump", "-sass", lib.LIB_PATH]).decode()
    assert "sm_100a" in subprocess.check_output(["cuobjdump", "-lelf", lib.LIB_PATH]).decode() or "SM100" in sass.upper()
    assert "UBLKCP" in sass          # TMA 1-D bulk copies in the block-distance kernel
    assert "FFMA2" in sass           # packed fp32x2 FMA


def test_status_strings_and_version(lib):
    assert lib.status_string(0) == "MEMSHARE_OK"
    assert lib.status_string(2) == "MEMSHARE_ERR_CAPACITY"
    assert lib.abi_version() == 1


def test_workspace_sizes_are_host_only(lib):
    assert lib.segment_steps_workspace_size(1000, 10, 100) > 0
    assert lib.step_candidates_workspace_size(1000, 2, 100, 50) > lib.step_candidates_workspace_size(10, 2, 100, 50)
    d = lib.Dims(64, 8, 8, 128, 16)
    assert lib.block_distance_workspace_size(d, 50, 100, 10) >= 100 * 64 * 2 * 8 * 4
    assert lib.remap_workspace_size(100, 10) > 0


def test_invalid_arguments_rejected_before_any_launch(lib):
    L = lib.lib
    nul = None
    # null pointers / bad counts -> INVALID_ARGUMENT (1), nothing enqueued
    d = (ctypes.c_int32 * 1)(5)
    assert L.memshare_segment_steps(nul, 0, nul, nul, nul, 1, d, 1, nul, nul, nul, nul, 0, nul, 0, nul, nul) == 1
    assert L.memshare_segment_steps(nul, 0, nul, nul, nul, 1, d, 0, nul, nul, nul, nul, 0, nul, 0, nul, nul) == 1
    dims = lib.Dims(64, 8, 8, 12, 16)        # head_dim % 8 != 0
    assert L.memshare_block_distance(nul, ctypes.byref(dims), nul, nul, nul, nul, 0, 0, 0, 0, nul, 0.1, nul, nul,
                                     nul, nul, 0, nul, nul) == 1
    assert L.memshare_remap(nul, 0, 0, nul, 0, nul, nul, nul, nul, 0, 16, nul, nul, nul, 0, nul, nul) == 1
    good = lib.Dims(64, 1, 8, 128, 16)
    buf = (ctypes.c_char * 64)()
    # finalize over peers: no peers / too many peers / null outputs -> INVALID_ARGUMENT
    for npeers in (0, 65):
        assert L.memshare_block_distance_finalize_peers(buf, npeers, ctypes.byref(good), buf, buf, buf, buf, 1, 1,
                                                        0.1, buf, buf, buf, buf, 64, buf, nul) == 1
    assert L.memshare_block_distance_finalize_peers(buf, 2, ctypes.byref(good), buf, buf, buf, buf, 1, 1, 0.1, nul,
                                                    buf, buf, buf, 64, buf, nul) == 1


def test_f1_host_checks_and_admission(lib):
    L = lib.lib
    nul = None
    dims = lib.Dims(64, 8, 8, 128, 16)
    # kv_append: null workspace / bad dims -> INVALID_ARGUMENT
    assert L.memshare_kv_append(nul, nul, 0, 0, 0, ctypes.byref(dims), nul, 0, 1, nul, nul, nul, nul, nul, nul, nul,
                                nul, 0, nul, nul) == 1
    # attention: block_size must be 16, head_dim 64/128, G <= 8
    bad = lib.Dims(64, 8, 8, 96, 16)
    pool = lib.KVPool(None, None, 0, 0, 0, 0)
    ws = (ctypes.c_char * 64)()
    st = (ctypes.c_int32 * 1)()
    assert L.memshare_paged_attention_decode(ctypes.byref(pool), ctypes.byref(bad), 0, nul, 40, nul, 1, nul, 1, 16,
                                             0.1, nul, ws, 64, st, nul) == 1
    assert L.memshare_paged_attention_decode(ctypes.byref(pool), ctypes.byref(dims), 0, nul, 72, nul, 1, nul, 1, 16,
                                             0.1, nul, ws, 64, st, nul) == 1
    assert lib.paged_attention_workspace_size(dims, 4, 40, 12406) >= 4 * 40 * 49 * 130 * 4
    assert lib.kv_append_workspace_size(8) > 0
    # the native admission scheduler against the oracle's definition on random queues
    import numpy as np
    import oracle
    rng = np.random.default_rng(0)
    for _ in range(200):
        pl = rng.integers(0, 400, rng.integers(0, 12))
        r, bsz, fb = int(rng.integers(0, 64)), int(rng.choice([1, 16, 32])), int(rng.integers(0, 80))
        assert lib.admit(pl, r, bsz, fb) == oracle.admit(pl, r, bsz, fb)
    assert L.memshare_admit(nul, 2, 0, 16, 10, nul) == -1
