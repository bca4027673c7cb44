"""ctypes binding of libmemshare.so (include/memshare.h): argument marshalling only.

Every function has the C name without the ``memshare_`` prefix and takes torch CUDA tensors
(device pointers via ``data_ptr()``) plus plain Python scalars; it returns the status code.
There is no fallback: if the CUDA library is missing or fails to load, importing this module
raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MEMSHARE_LIB") or os.path.join(_HERE, "libmemshare.so")   # override: tuning variants only
HEADER = os.path.join(os.path.dirname(_HERE), "include", "memshare.h")

OK, INVALID_ARGUMENT, CAPACITY, CORRUPTION, CUDA_ERROR = 0, 1, 2, 3, 4
CUR_ALL, CUR_LAST, CUR_RANGE = 0, 1, 2
PAIR_ALIGNED, PAIR_CROSS = 0, 1
DIST_FULL, DIST_PARTIAL, DIST_FINALIZE = 0, 1, 2
DIST_GROUPED = 0x100       # schedule hint OR'ed into the mode (CROSS / all-pairs lists)
METRIC_EUCLIDEAN, METRIC_COSINE = 0, 1

MATCH_DTYPE = np.dtype([("seq", "<i4"), ("step", "<i4"), ("cand_step", "<i4"), ("rank", "<i4"), ("cosine", "<f8")])
PAIR_DTYPE = np.dtype([("seq", "<i4"), ("target_idx", "<i4"), ("target_logical", "<i4"), ("source_logical", "<i4"),
                       ("target_phys", "<i4"), ("source_phys", "<i4")])
DECISION_DTYPE = np.dtype([("seq", "<i4"), ("target_logical", "<i4"), ("target_phys", "<i4"),
                           ("source_logical", "<i4"), ("source_phys", "<i4"), ("accepted", "<i4"),
                           ("distance", "<f4"), ("num_candidates", "<i4")])
assert MATCH_DTYPE.itemsize == 24 and PAIR_DTYPE.itemsize == 24 and DECISION_DTYPE.itemsize == 32


class Dims(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_kv_heads_local", ctypes.c_int32),
                ("num_kv_heads_global", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("block_size", ctypes.c_int32)]


class KVPool(ctypes.Structure):
    _fields_ = [("k", ctypes.c_void_p), ("v", ctypes.c_void_p), ("layer_stride", ctypes.c_int64),
                ("block_stride", ctypes.c_int64), ("num_blocks", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class MemShareError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U64, F32, F64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_float,
                                  ctypes.c_double)
    L.memshare_segment_steps.argtypes = [P, I64, P, P, P, I32, P, I32, P, P, P, P, I64, P, U64, P, P]
    L.memshare_segment_steps.restype = I32
    L.memshare_segment_steps_workspace_size.argtypes = [I64, I32, I64]
    L.memshare_segment_steps_workspace_size.restype = U64
    L.memshare_step_candidates.argtypes = ([P, I64, P, I32, P, P, P, P, I64, P, I32, I32, P, P, P, I32, I32, I32, F64,
                                            I32, I32, P, I64, P, P, I64, P, P, I64, P, P, U64, P, P])
    L.memshare_step_candidates.restype = I32
    L.memshare_step_candidates_workspace_size.argtypes = [I64, I32, I64, I64]
    L.memshare_step_candidates_workspace_size.restype = U64
    L.memshare_block_distance.argtypes = [P, P, P, P, P, P, I64, I64, I32, I32, P, F32, P, P, P, P, U64, P, P]
    L.memshare_block_distance.restype = I32
    L.memshare_block_distance_workspace_size.argtypes = [P, I32, I64, I64, I32]
    L.memshare_block_distance_workspace_size.restype = U64
    L.memshare_block_distance_remap.argtypes = [P, P, P, P, P, P, I64, I64, I32, F32, P, P, P, P, I32, I32, P, P, P, I32,
                                                P, P, P, U64, P, P]
    L.memshare_block_distance_remap.restype = I32
    L.memshare_block_distance_remap_workspace_size.argtypes = [P, I32, I64, I64, I32]
    L.memshare_block_distance_remap_workspace_size.restype = U64
    L.memshare_block_distance_finalize_peers.argtypes = [P, I32, P, P, P, P, P, I64, I64, F32, P, P, P, P, U64, P, P]
    L.memshare_block_distance_finalize_peers.restype = I32
    L.memshare_remap.argtypes = [P, I32, I32, P, I32, P, P, P, P, I64, I32, P, P, P, U64, P, P]
    L.memshare_remap.restype = I32
    L.memshare_remap_workspace_size.argtypes = [I32, I64]
    L.memshare_remap_workspace_size.restype = U64
    L.memshare_similarity_ratio.argtypes = [P, P, I64, I32, P, P, P]
    L.memshare_similarity_ratio.restype = I32
    L.memshare_all_pairs.argtypes = [P, I32, P, P, P, I32, I32, I32, P, I64, P, P, I64, P, P, U64, P, P]
    L.memshare_all_pairs.restype = I32
    L.memshare_all_pairs_workspace_size.argtypes = [I32]
    L.memshare_all_pairs_workspace_size.restype = U64
    L.memshare_kv_append.argtypes = [P, P, I64, I64, I32, P, P, I32, I32, P, P, P, P, P, P, P, P, U64, P, P]
    L.memshare_kv_append.restype = I32
    L.memshare_kv_append_workspace_size.argtypes = [I32]
    L.memshare_kv_append_workspace_size.restype = U64
    L.memshare_paged_attention_decode.argtypes = [P, P, I32, P, I32, P, I32, P, I32, I32, F32, P, P, U64, P, P]
    L.memshare_paged_attention_decode.restype = I32
    L.memshare_paged_attention_workspace_size.argtypes = [P, I32, I32, I32]
    L.memshare_paged_attention_workspace_size.restype = U64
    L.memshare_admit.argtypes = [P, I32, I32, I32, I64, P]
    L.memshare_admit.restype = I32
    L.memshare_status_string.argtypes = [I32]
    L.memshare_status_string.restype = ctypes.c_char_p
    L.memshare_profile_distance_events.argtypes = [P, P]
    L.memshare_profile_distance_events.restype = None
    L.memshare_abi_version.argtypes = []
    L.memshare_abi_version.restype = I32
    return L


lib = _load()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def status_string(code: int) -> str:
    return lib.memshare_status_string(code).decode()


def check(code: int, what: str = "memshare"):
    if code != OK:
        raise MemShareError(f"{what}: {status_string(code)}")
    return code


def profile_distance_events(begin, end):
    """Measurement hook: record torch.cuda.Event begin/end around the streaming kernel of every
    following block_distance call on this thread (None, None: off)."""
    lib.memshare_profile_distance_events(None if begin is None else ctypes.c_void_p(begin.cuda_event),
                                         None if end is None else ctypes.c_void_p(end.cuda_event))


def abi_version() -> int:
    return lib.memshare_abi_version()


# ------------------------------------------------------------------------------------- a1
def segment_steps_workspace_size(num_tokens: int, num_seqs: int, step_cap: int) -> int:
    return lib.memshare_segment_steps_workspace_size(num_tokens, num_seqs, step_cap)


def segment_steps(tokens, num_tokens, seq_tok_off, gen_start, seq_final, num_seqs, delim_ids, step_start, step_end,
                  step_nbag, seq_step_off, step_cap, workspace, device_status, stream=None) -> int:
    d = np.ascontiguousarray(delim_ids, np.int32)
    return lib.memshare_segment_steps(_ptr(tokens), num_tokens, _ptr(seq_tok_off), _ptr(gen_start), _ptr(seq_final),
                                      num_seqs, d.ctypes.data, d.size, _ptr(step_start), _ptr(step_end),
                                      _ptr(step_nbag), _ptr(seq_step_off), step_cap, _ptr(workspace),
                                      0 if workspace is None else workspace.numel() * workspace.element_size(),
                                      _ptr(device_status), _stream(stream))


# ----------------------------------------------------------------------------------- a2-a4
def step_candidates_workspace_size(num_tokens, num_seqs, step_cap, match_cap) -> int:
    return lib.memshare_step_candidates_workspace_size(num_tokens, num_seqs, step_cap, match_cap)


def step_candidates(tokens, num_tokens, seq_tok_off, num_seqs, seq_step_off, step_start, step_end, step_nbag,
                    step_cap, delim_ids, cur_mode, cur_begin, cur_end, block_table, table_stride, num_blocks,
                    block_size, tau_s, top_k, pairing, matches, match_cap, num_matches, pairs, pair_cap, num_pairs,
                    target_off, target_cap, num_targets, workspace, device_status, stream=None) -> int:
    d = np.ascontiguousarray(delim_ids, np.int32)
    return lib.memshare_step_candidates(
        _ptr(tokens), num_tokens, _ptr(seq_tok_off), num_seqs, _ptr(seq_step_off), _ptr(step_start), _ptr(step_end),
        _ptr(step_nbag), step_cap, d.ctypes.data, d.size, cur_mode, _ptr(cur_begin), _ptr(cur_end), _ptr(block_table),
        table_stride, num_blocks, block_size, float(tau_s), top_k, pairing, _ptr(matches), match_cap,
        _ptr(num_matches), _ptr(pairs), pair_cap, _ptr(num_pairs), _ptr(target_off), target_cap, _ptr(num_targets),
        _ptr(workspace), 0 if workspace is None else workspace.numel() * workspace.element_size(),
        _ptr(device_status), _stream(stream))


# ----------------------------------------------------------------------------------- a5-a6
def block_distance_workspace_size(dims: Dims, num_blocks: int, pair_cap: int, target_cap: int,
                                  metric: int = METRIC_EUCLIDEAN) -> int:
    return lib.memshare_block_distance_workspace_size(ctypes.byref(dims), num_blocks, pair_cap, target_cap, metric)


def block_distance(pool: KVPool | None, dims: Dims, pairs, target_off, num_pairs, num_targets, pair_cap, target_cap,
                   mode, partial_sq, tau_b, distance, under, decisions, workspace, device_status, stream=None,
                   metric: int = METRIC_EUCLIDEAN) -> int:
    return lib.memshare_block_distance(
        None if pool is None else ctypes.byref(pool), ctypes.byref(dims), _ptr(pairs), _ptr(target_off),
        _ptr(num_pairs), _ptr(num_targets), pair_cap, target_cap, mode, metric, _ptr(partial_sq), float(tau_b),
        _ptr(distance), _ptr(under), _ptr(decisions), _ptr(workspace),
        0 if workspace is None else workspace.numel() * workspace.element_size(), _ptr(device_status),
        _stream(stream))


def block_distance_remap_workspace_size(dims: Dims, num_blocks: int, pair_cap: int, target_cap: int,
                                        metric: int = METRIC_EUCLIDEAN) -> int:
    return lib.memshare_block_distance_remap_workspace_size(ctypes.byref(dims), num_blocks, pair_cap, target_cap,
                                                            metric)


def block_distance_remap(pool: KVPool, dims: Dims, pairs, target_off, num_pairs, num_targets, pair_cap, target_cap,
                         metric, tau_b, distance, under, decisions, block_table, table_stride, num_seqs, refcount,
                         free_list, free_count, block_size, num_freed, affected_tokens, workspace, device_status,
                         stream=None) -> int:
    """a5-a7 in one call (memshare_block_distance FULL + memshare_remap)."""
    return lib.memshare_block_distance_remap(
        ctypes.byref(pool), ctypes.byref(dims), _ptr(pairs), _ptr(target_off), _ptr(num_pairs), _ptr(num_targets),
        pair_cap, target_cap, metric, float(tau_b), _ptr(distance), _ptr(under), _ptr(decisions), _ptr(block_table),
        table_stride, num_seqs, _ptr(refcount), _ptr(free_list), _ptr(free_count), block_size, _ptr(num_freed),
        _ptr(affected_tokens), _ptr(workspace),
        0 if workspace is None else workspace.numel() * workspace.element_size(), _ptr(device_status),
        _stream(stream))


def block_distance_finalize_peers(peer_ptrs_dev, num_peers, dims: Dims, pairs, target_off, num_pairs, num_targets,
                                  pair_cap, target_cap, tau_b, distance, under, decisions, workspace, device_status,
                                  stream=None) -> int:
    """peer_ptrs_dev: int64 CUDA tensor [num_peers] of device pointers (every rank's partial_sq)."""
    return lib.memshare_block_distance_finalize_peers(
        _ptr(peer_ptrs_dev), num_peers, ctypes.byref(dims), _ptr(pairs), _ptr(target_off), _ptr(num_pairs),
        _ptr(num_targets), pair_cap, target_cap, float(tau_b), _ptr(distance), _ptr(under), _ptr(decisions),
        _ptr(workspace), 0 if workspace is None else workspace.numel() * workspace.element_size(),
        _ptr(device_status), _stream(stream))


# -------------------------------------------------------------------------------------- a7
def remap_workspace_size(num_blocks: int, target_cap: int) -> int:
    return lib.memshare_remap_workspace_size(num_blocks, target_cap)


def remap(block_table, table_stride, num_seqs, refcount, num_blocks, free_list, free_count, decisions, num_targets,
          target_cap, block_size, num_freed, affected_tokens, workspace, device_status, stream=None) -> int:
    return lib.memshare_remap(_ptr(block_table), table_stride, num_seqs, _ptr(refcount), num_blocks, _ptr(free_list),
                              _ptr(free_count), _ptr(decisions), _ptr(num_targets), target_cap, block_size,
                              _ptr(num_freed), _ptr(affected_tokens), _ptr(workspace),
                              0 if workspace is None else workspace.numel() * workspace.element_size(),
                              _ptr(device_status), _stream(stream))


# -------------------------------------------------------------------------------------- f4
def similarity_ratio(matches, num_matches, match_cap, num_seqs, redundant_steps, device_status, stream=None) -> int:
    return lib.memshare_similarity_ratio(_ptr(matches), _ptr(num_matches), match_cap, num_seqs, _ptr(redundant_steps),
                                         _ptr(device_status), _stream(stream))


# -------------------------------------------------------------------------------------- f3
def all_pairs_workspace_size(num_seqs: int) -> int:
    return lib.memshare_all_pairs_workspace_size(num_seqs)


def all_pairs(seq_tok_off, num_seqs, blk_begin, blk_end, block_table, table_stride, num_blocks, block_size, pairs,
              pair_cap, num_pairs, target_off, target_cap, num_targets, workspace, device_status, stream=None) -> int:
    return lib.memshare_all_pairs(_ptr(seq_tok_off), num_seqs, _ptr(blk_begin), _ptr(blk_end), _ptr(block_table),
                                  table_stride, num_blocks, block_size, _ptr(pairs), pair_cap, _ptr(num_pairs),
                                  _ptr(target_off), target_cap, _ptr(num_targets), _ptr(workspace),
                                  0 if workspace is None else workspace.numel() * workspace.element_size(),
                                  _ptr(device_status), _stream(stream))


# -------------------------------------------------------------------------------------- f1
def kv_append_workspace_size(num_seqs: int) -> int:
    return lib.memshare_kv_append_workspace_size(num_seqs)


def kv_append(k_pool, v_pool, layer_stride, block_stride, num_blocks, dims: Dims, block_table, table_stride,
              num_seqs, seq_len, active, refcount, free_list, free_count, new_k, new_v, workspace, device_status,
              stream=None) -> int:
    return lib.memshare_kv_append(_ptr(k_pool), _ptr(v_pool), layer_stride, block_stride, num_blocks,
                                  ctypes.byref(dims), _ptr(block_table), table_stride, num_seqs, _ptr(seq_len),
                                  _ptr(active), _ptr(refcount), _ptr(free_list), _ptr(free_count), _ptr(new_k),
                                  _ptr(new_v), _ptr(workspace),
                                  0 if workspace is None else workspace.numel() * workspace.element_size(),
                                  _ptr(device_status), _stream(stream))


def paged_attention_workspace_size(dims: Dims, num_seqs: int, num_q_heads: int, max_seq_len: int) -> int:
    return lib.memshare_paged_attention_workspace_size(ctypes.byref(dims), num_seqs, num_q_heads, max_seq_len)


def paged_attention_decode(pool: KVPool, dims: Dims, layer, q, num_q_heads, block_table, table_stride, seq_len,
                           num_seqs, max_seq_len, scale, out, workspace, device_status, stream=None) -> int:
    return lib.memshare_paged_attention_decode(ctypes.byref(pool), ctypes.byref(dims), layer, _ptr(q), num_q_heads,
                                               _ptr(block_table), table_stride, _ptr(seq_len), num_seqs, max_seq_len,
                                               float(scale), _ptr(out), _ptr(workspace),
                                               0 if workspace is None else workspace.numel() * workspace.element_size(),
                                               _ptr(device_status), _stream(stream))


def admit(prompt_len, reserve: int, block_size: int, free_blocks: int):
    """Host FCFS block-budget admission (native): (admitted, blocks_used)."""
    import numpy as _np
    pl = _np.ascontiguousarray(prompt_len, _np.int32)
    used = ctypes.c_int64(0)
    n = lib.memshare_admit(pl.ctypes.data if pl.size else None, pl.size, reserve, block_size, free_blocks,
                           ctypes.byref(used))
    if n < 0:
        raise MemShareError("admit: invalid arguments")
    return int(n), int(used.value)
