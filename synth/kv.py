"""Counter-hash KV generator: Python side of the host (C) and device (CUDA) twins.

Formula and bit-exactness argument: ``csrc/msgen_hash.h``. Shapes follow
BASELINE.json's KV layouts; the pool layout is the product's (layer-major
``K[l][block][tau][head][x]``), but nothing here reads or computes distances.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "csrc")
HOST_SO = os.path.join(_HERE, "libmsgen_host.so")
DEV_SO = os.path.join(_HERE, "libmsgen_dev.so")


@dataclass(frozen=True)
class KVShape:
    num_layers: int
    num_kv_heads: int
    head_dim: int
    block_size: int

    @property
    def slice_elems(self) -> int:          # one (layer, K|V, block) slice
        return self.block_size * self.num_kv_heads * self.head_dim

    @property
    def block_bytes(self) -> int:          # B_blk = N * 2 * d * h * d_h * 2 B
        return self.num_layers * 2 * self.slice_elems * 2


TINY = KVShape(2, 2, 64, 16)
QWEN32B = KVShape(64, 8, 128, 16)      # DeepSeek-R1-Distill-Qwen-32B / QwQ-32B (GQA, 8 KV heads)
PHI4 = KVShape(40, 10, 128, 16)        # Phi-4-reasoning-plus


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_host():
    srcs = [os.path.join(_CSRC, "msgen_host.c"), os.path.join(_CSRC, "msgen_hash.h")]
    if _stale(HOST_SO, srcs):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-fopenmp",
                               "-ffp-contract=off", "-o", HOST_SO, srcs[0]])
    return HOST_SO


def build_dev():
    srcs = [os.path.join(_CSRC, "msgen_dev.cu"), os.path.join(_CSRC, "msgen_hash.h")]
    if _stale(DEV_SO, srcs):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-Xcompiler", "-fPIC", "-shared", "-fmad=false", "-o", DEV_SO, srcs[0]])
    return DEV_SO


_host_lib = None
_dev_lib = None

_ARGT = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float]


def _host():
    global _host_lib
    if _host_lib is None:
        _host_lib = ctypes.CDLL(build_host())
        _host_lib.msgen_fill_blocks_host.argtypes = _ARGT
        _host_lib.msgen_fill_blocks_host.restype = None
    return _host_lib


def _dev():
    global _dev_lib
    if _dev_lib is None:
        _dev_lib = ctypes.CDLL(build_dev())
        _dev_lib.msgen_fill_blocks_dev.argtypes = _ARGT + [ctypes.c_void_p]
        _dev_lib.msgen_fill_blocks_dev.restype = ctypes.c_int
    return _dev_lib


def table_blocks(seq_tok_off: np.ndarray, table: np.ndarray, block_size: int):
    """(seq, logical, physical) of every block the table maps within each sequence's length."""
    seqs, logs, phys = [], [], []
    for s in range(table.shape[0]):
        n = int(seq_tok_off[s + 1] - seq_tok_off[s])
        nb = -(-n // block_size)
        seqs.append(np.full(nb, s, np.int32))
        logs.append(np.arange(nb, dtype=np.int32))
        phys.append(table[s, :nb].astype(np.int32))
    cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int32))
    return cat(seqs), cat(logs), cat(phys)


def fill_blocks_host(k: np.ndarray, v: np.ndarray, layer_stride: int, block_stride: int, shape: KVShape,
                     tokens, seq_tok_off, blk_seq, blk_logical, blk_dst, seed: int, eta: float,
                     h_local: int | None = None, head_offset: int = 0):
    """Fill uint16 (bf16 bits) numpy pools on the host."""
    assert k.dtype == np.uint16 and v.dtype == np.uint16 and k.flags.c_contiguous and v.flags.c_contiguous
    tokens = np.ascontiguousarray(tokens, np.int32)
    seq_tok_off = np.ascontiguousarray(seq_tok_off, np.int64)
    bs, bl, bd = (np.ascontiguousarray(a, np.int32) for a in (blk_seq, blk_logical, blk_dst))
    _host().msgen_fill_blocks_host(k.ctypes.data, v.ctypes.data, layer_stride, block_stride, shape.num_layers,
                                   h_local or shape.num_kv_heads, head_offset, shape.head_dim, shape.block_size,
                                   tokens.ctypes.data, seq_tok_off.ctypes.data, bs.ctypes.data, bl.ctypes.data,
                                   bd.ctypes.data, bs.size, seed & (2**64 - 1), eta)


def fill_blocks_dev(k, v, layer_stride: int, block_stride: int, shape: KVShape, tokens_d, seq_tok_off_d,
                    blk_seq_d, blk_logical_d, blk_dst_d, seed: int, eta: float, h_local: int | None = None,
                    head_offset: int = 0, stream=None):
    """Fill bf16/int16 torch CUDA pools on the device (torch tensors for every array)."""
    import torch
    st = stream if stream is not None else torch.cuda.current_stream()
    rc = _dev().msgen_fill_blocks_dev(k.data_ptr(), v.data_ptr(), layer_stride, block_stride, shape.num_layers,
                                      h_local or shape.num_kv_heads, head_offset, shape.head_dim,
                                      shape.block_size, tokens_d.data_ptr(), seq_tok_off_d.data_ptr(),
                                      blk_seq_d.data_ptr(), blk_logical_d.data_ptr(), blk_dst_d.data_ptr(),
                                      blk_seq_d.numel(), seed & (2**64 - 1), eta, ctypes.c_void_p(st.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"msgen_fill_blocks_dev failed: cuda error {rc}")


def host_pool(shape: KVShape, num_blocks: int, h_local: int | None = None):
    """Zeroed layer-major host pool; returns (k, v, layer_stride, block_stride) in elements."""
    hl = h_local or shape.num_kv_heads
    slice_elems = shape.block_size * hl * shape.head_dim
    k = np.zeros(shape.num_layers * num_blocks * slice_elems, np.uint16)
    v = np.zeros_like(k)
    return k, v, num_blocks * slice_elems, slice_elems
