"""Device-buffer plumbing around the four C-ABI calls (no arithmetic of the method here).

``MemSharePath`` owns the torch CUDA buffers of one pool (trace, block table, refcounts, free
list, KV pool, outputs, workspaces) and enqueues the calls in path order on one stream:

    segment_steps -> step_candidates -> block_distance -> remap        (one round)

Counts stay on the device between calls; ``read_*`` methods synchronise and copy to host for
tests and reporting only.
"""
from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


@dataclass
class Caps:
    step: int
    match: int
    pair: int
    target: int


def _dev_i32(a, dev):
    """int32 device tensor; a device int32 tensor passes through (usable inside graph capture)."""
    if isinstance(a, torch.Tensor) and a.device.type == dev.type and a.dtype == torch.int32:
        return a.contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, np.int32), device=dev)


def pack_inputs(tokens, seq_tok_off, gen_start, final, table, refcount, free_list, free_count):
    """Host int32 buffer holding one round's inputs in MemSharePath's layout, and the layout
    (int32 offsets of each part). A serving loop fills a pinned copy of this and uploads it with a
    single host-to-device copy into ``MemSharePath.inputs``."""
    ns = int(len(gen_start))
    tok = tokens if not isinstance(tokens, torch.Tensor) else None
    nt_tok = int(len(tokens))
    table = np.ascontiguousarray(table, np.int32)
    refcount = np.ascontiguousarray(refcount, np.int32)
    free_list = np.ascontiguousarray(free_list, np.int32)
    lay = {"seq_tok_off": 0, "state": 2 * (ns + 1)}
    n_state = 2 + table.size + refcount.size + free_list.size
    lay["tokens"] = lay["state"] + n_state
    lay["gen_start"] = lay["tokens"] + nt_tok
    lay["final"] = lay["gen_start"] + ns
    total = lay["final"] + (ns + 3) // 4
    host = np.zeros(max(total, 1), np.int32)
    host[:lay["state"]] = np.ascontiguousarray(seq_tok_off, np.int64).view(np.int32)
    s0 = lay["state"]
    host[s0:s0 + 2] = np.asarray([int(free_count)], np.int64).view(np.int32)
    o = s0 + 2
    for part in (table.ravel(), refcount, free_list):
        host[o:o + part.size] = part
        o += part.size
    if tok is not None:
        host[lay["tokens"]:lay["gen_start"]] = np.ascontiguousarray(tok, np.int32)
    host[lay["gen_start"]:lay["final"]] = np.ascontiguousarray(gen_start, np.int32)
    fin = np.zeros(((ns + 3) // 4) * 4, np.uint8)
    fin[:ns] = np.ascontiguousarray(final, np.uint8)
    host[lay["final"]:total] = fin.view(np.int32)
    return host, lay


class MemSharePath:
    def __init__(self, tokens, seq_tok_off, gen_start, final, delim_ids, table, refcount, free_list, free_count,
                 k_pool, v_pool, layer_stride, block_stride, num_blocks, num_layers, h_local, h_global, head_dim,
                 block_size, caps: Caps | None = None, device="cuda", stream=None):
        self.dev = torch.device(device)
        self._stream = stream      # None: every call goes to the then-current stream (CUDA-graph capture works)
        self.delims = np.ascontiguousarray(delim_ids, np.int32)
        self.num_seqs = int(len(gen_start))
        self.num_tokens = int(len(tokens))
        table = np.ascontiguousarray(table, np.int32)
        self.table_stride = int(table.shape[1])
        # Every per-round input in ONE int32 buffer (a serving loop uploads a round with one copy;
        # the state remap() mutates is one contiguous sub-range, so one copy snapshots / restores it):
        #   [seq_tok_off int64][free_count int64][block table][refcounts][free list][tokens][gen_start][final u8]
        host, lay = pack_inputs(tokens, seq_tok_off, gen_start, final, table, refcount, free_list, free_count)
        self.layout = lay
        self.inputs = torch.as_tensor(host, device=self.dev)
        if isinstance(tokens, torch.Tensor):         # e.g. a device-resident trace: copied in place
            self.inputs[lay["tokens"]:lay["tokens"] + self.num_tokens].copy_(tokens.view(-1).to(torch.int32))
        i = self.inputs
        self.seq_tok_off = i[lay["seq_tok_off"]:lay["state"]].view(torch.int64)
        self.state = i[lay["state"]:lay["tokens"]]
        st = self.state
        nt, nr = table.size, int(np.asarray(refcount).size)
        self.free_count = st[:2].view(torch.int64)
        self.table = st[2:2 + nt].view(table.shape)
        self.refcount = st[2 + nt:2 + nt + nr]
        self.free_list = st[2 + nt + nr:]
        self.tokens = i[lay["tokens"]:lay["tokens"] + self.num_tokens]
        self.gen_start = i[lay["gen_start"]:lay["gen_start"] + self.num_seqs]
        self.final = i[lay["final"]:].view(torch.uint8)[:self.num_seqs]
        self.num_blocks = int(num_blocks)
        self.k_pool, self.v_pool = k_pool, v_pool
        self.pool = L.KVPool(k_pool.data_ptr() if k_pool is not None else None,
                             v_pool.data_ptr() if v_pool is not None else None, layer_stride, block_stride,
                             num_blocks, 0)
        self.dims = L.Dims(num_layers, h_local, h_global, head_dim, block_size)
        self.block_size = block_size
        self.status = torch.zeros(1, dtype=torch.int32, device=self.dev)
        z64 = lambda: torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.seq_step_off = torch.zeros(self.num_seqs + 1, dtype=torch.int64, device=self.dev)
        self.partial_sq = None
        self.set_caps(caps or Caps(step=max(1, self.num_tokens), match=max(1024, self.num_tokens),
                                   pair=max(4096, self.num_tokens), target=max(2048, self.num_tokens // block_size + 1)))

    @property
    def stream(self):
        return self._stream if self._stream is not None else torch.cuda.current_stream(self.dev)

    def capture(self, fn):
        """Capture `fn` (a sequence of the calls above) into a CUDA graph; returns the graph
        (replay() re-runs the captured launches with the same buffers)."""
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                fn()
        torch.cuda.current_stream(self.dev).wait_stream(side)
        return g

    # ------------------------------------------------------------------ buffers
    def set_caps(self, caps: Caps):
        self.caps = caps
        d = self.dev
        e = lambda n, dt: torch.empty(max(1, n), dtype=dt, device=d)
        self.step_start, self.step_end, self.step_nbag = (e(caps.step, torch.int32) for _ in range(3))
        self.matches = e(caps.match * 24, torch.uint8)
        self.pairs = e(caps.pair * 24, torch.uint8)
        self.target_off = e(caps.target + 1, torch.int64)
        self.distance = e(caps.pair, torch.float32)
        self.under = e(caps.pair, torch.uint8)
        # the per-round outputs a serving loop reads back, in ONE buffer (one copy):
        #   [num_matches, num_pairs, num_targets, num_freed, affected, 3 spare: int64][decisions]
        self.outputs = torch.zeros(64 + max(1, caps.target) * 32, dtype=torch.uint8, device=d)
        self.counters = self.outputs[:64].view(torch.int64)
        c = self.counters
        self.num_matches, self.num_pairs, self.num_targets, self.num_freed, self.affected = (c[j:j + 1] for j in range(5))
        self.decisions = self.outputs[64:]
        ws = max(L.segment_steps_workspace_size(self.num_tokens, self.num_seqs, caps.step),
                 L.step_candidates_workspace_size(self.num_tokens, self.num_seqs, caps.step, caps.match),
                 L.block_distance_workspace_size(self.dims, self.num_blocks, caps.pair, caps.target,
                                                 L.METRIC_COSINE),
                 L.remap_workspace_size(self.num_blocks, caps.target),
                 L.block_distance_remap_workspace_size(self.dims, self.num_blocks, caps.pair, caps.target,
                                                       L.METRIC_COSINE))
        self.workspace = e(ws, torch.uint8)

    def alloc_partial(self):
        self.partial_sq = torch.zeros(max(1, self.caps.pair) * self.dims.num_layers * 2, dtype=torch.float32,
                                      device=self.dev)
        return self.partial_sq

    # ------------------------------------------------------------------ the four calls
    def segment(self):
        L.check(L.segment_steps(self.tokens, self.num_tokens, self.seq_tok_off, self.gen_start, self.final,
                                self.num_seqs, self.delims,
                                self.step_start, self.step_end, self.step_nbag, self.seq_step_off, self.caps.step,
                                self.workspace, self.status, self.stream), "segment_steps")

    def candidates(self, tau_s, top_k=0, pairing=L.PAIR_ALIGNED, cur_mode=L.CUR_ALL, cur_begin=None, cur_end=None):
        cb = None if cur_begin is None else _dev_i32(cur_begin, self.dev)
        ce = None if cur_end is None else _dev_i32(cur_end, self.dev)
        self._cur_keep = (cb, ce)
        # CROSS lists: the targets of a step share their sources -> the grouped distance schedule
        self.grouped_hint = pairing == L.PAIR_CROSS
        L.check(L.step_candidates(self.tokens, self.num_tokens, self.seq_tok_off, self.num_seqs, self.seq_step_off,
                                  self.step_start, self.step_end, self.step_nbag, self.caps.step, self.delims, cur_mode,
                                  cb, ce, self.table, self.table_stride, self.num_blocks, self.block_size, tau_s, top_k,
                                  pairing, self.matches, self.caps.match, self.num_matches, self.pairs, self.caps.pair,
                                  self.num_pairs, self.target_off, self.caps.target, self.num_targets, self.workspace,
                                  self.status, self.stream), "step_candidates")

    def distance_call(self, tau_b, mode=L.DIST_FULL, partial_sq=None, metric=L.METRIC_EUCLIDEAN):
        ps = partial_sq if partial_sq is not None else self.partial_sq
        if mode != L.DIST_FINALIZE:
            mode |= self._grouped(metric)
        L.check(L.block_distance(None if mode == L.DIST_FINALIZE else self.pool, self.dims, self.pairs,
                                 self.target_off, self.num_pairs, self.num_targets, self.caps.pair, self.caps.target,
                                 mode, ps, tau_b, self.distance, self.under, self.decisions, self.workspace,
                                 self.status, self.stream, metric), "block_distance")

    def finalize_peers(self, tau_b, peer_ptrs_dev, num_peers):
        """KV-head-sharded FINALIZE reading every rank's partial_sq over peer memory (rank order)."""
        L.check(L.block_distance_finalize_peers(peer_ptrs_dev, num_peers, self.dims, self.pairs, self.target_off,
                                                self.num_pairs, self.num_targets, self.caps.pair, self.caps.target,
                                                tau_b, self.distance, self.under, self.decisions, self.workspace,
                                                self.status, self.stream), "block_distance_finalize_peers")

    def remap(self):
        L.check(L.remap(self.table, self.table_stride, self.num_seqs, self.refcount, self.num_blocks, self.free_list,
                        self.free_count, self.decisions, self.num_targets, self.caps.target, self.block_size,
                        self.num_freed, self.affected, self.workspace, self.status, self.stream), "remap")

    def _grouped(self, metric):
        """MEMSHARE_DIST_GROUPED for lists whose targets share sources (CROSS, all-pairs; Euclidean
        metric) when MEMSHARE_GROUPED=1. Off by default: on B200 the grouped schedule halves the
        staging cost but the consumer arithmetic bounds both schedules, and it measured slower
        (profiles/r1_tuning_log.md, "Grouped schedule")."""
        if (getattr(self, "grouped_hint", False) and metric == L.METRIC_EUCLIDEAN
                and os.environ.get("MEMSHARE_GROUPED", "0") == "1"):
            return L.DIST_GROUPED
        return 0

    def distance_remap(self, tau_b, metric=L.METRIC_EUCLIDEAN):
        """a5-a7 as one call: distance_call(FULL) + remap() with the finalisation and the remap fused
        into the streaming kernel (identical results)."""
        L.check(L.block_distance_remap(self.pool, self.dims, self.pairs, self.target_off, self.num_pairs,
                                       self.num_targets, self.caps.pair, self.caps.target,
                                       metric | self._grouped(metric), tau_b,
                                       self.distance, self.under, self.decisions, self.table, self.table_stride,
                                       self.num_seqs, self.refcount, self.free_list, self.free_count,
                                       self.block_size, self.num_freed, self.affected, self.workspace, self.status,
                                       self.stream), "block_distance_remap")

    # ------------------------------------------------------------------ analysis (f3, f4)
    def similarity_ratio(self):
        """f4: per-sequence count of steps with a Stage-1 survivor (run candidates() first with the
        threshold of interest); returns the device int64 [num_seqs] tensor."""
        out = torch.zeros(max(1, self.num_seqs), dtype=torch.int64, device=self.dev)
        L.check(L.similarity_ratio(self.matches, self.num_matches, self.caps.match, self.num_seqs, out, self.status,
                                   self.stream), "similarity_ratio")
        return out[:self.num_seqs]

    def all_pairs(self, blk_begin, blk_end):
        """f3: fill the pair buffers with every block pair of the per-sequence windows (then
        distance_call() scores the distance matrix). Caps must hold sum m(m-1)/2 pairs."""
        bb, be = _dev_i32(blk_begin, self.dev), _dev_i32(blk_end, self.dev)
        self._ap_keep = (bb, be)
        self.grouped_hint = True          # target j's sources are blocks lo..j-1: nested prefixes
        ws = torch.empty(max(1, L.all_pairs_workspace_size(self.num_seqs)), dtype=torch.uint8, device=self.dev)
        self._ap_ws = ws
        L.check(L.all_pairs(self.seq_tok_off, self.num_seqs, bb, be, self.table, self.table_stride, self.num_blocks,
                            self.block_size, self.pairs, self.caps.pair, self.num_pairs, self.target_off,
                            self.caps.target, self.num_targets, ws, self.status, self.stream), "all_pairs")

    def round(self, tau_s, tau_b, top_k=0, pairing=L.PAIR_ALIGNED, cur_mode=L.CUR_ALL, cur_begin=None, cur_end=None):
        self.segment()
        self.candidates(tau_s, top_k, pairing, cur_mode, cur_begin, cur_end)
        self.distance_call(tau_b)
        self.remap()

    # ------------------------------------------------------------------ state snapshot (debugging)
    def snapshot(self) -> dict:
        """JSON-serialisable state of the path (SURVEY.md §5 / SPEC.md:412: capacity, dims, tables,
        refcounts, fill): the KV geometry and caps, the block table, refcounts, the live part of the
        free list, the round counters and the device status. Synchronises."""
        st = self.read_state()
        c = self.counts()
        d = self.dims
        fc = st["free_count"]
        return {"version": 1, "num_seqs": self.num_seqs, "num_tokens": self.num_tokens,
                "num_blocks": self.num_blocks, "table_stride": self.table_stride,
                "dims": {"num_layers": d.num_layers, "num_kv_heads_local": d.num_kv_heads_local,
                         "num_kv_heads_global": d.num_kv_heads_global, "head_dim": d.head_dim,
                         "block_size": d.block_size},
                "caps": {"step": self.caps.step, "match": self.caps.match, "pair": self.caps.pair,
                         "target": self.caps.target},
                "table": st["table"].tolist(), "refcount": st["refcount"].tolist(),
                "free_list": st["free_list"][:max(0, min(fc, st["free_list"].size))].tolist(), "free_count": fc,
                "counters": {**c, "freed": st["num_freed"], "affected_tokens": st["affected"]},
                "status": self.read_status()}

    def restore_snapshot(self, snap: dict):
        """Write a snapshot's block table, refcounts, free list and free count back to the device
        (same geometry; the KV pool and the trace are not part of a snapshot)."""
        if snap.get("version") != 1 or snap["num_blocks"] != self.num_blocks or \
                snap["table_stride"] != self.table_stride or snap["num_seqs"] != self.num_seqs:
            raise ValueError("snapshot does not match this path's geometry")
        tab = torch.as_tensor(np.asarray(snap["table"], np.int32).reshape(-1), device=self.dev)
        rc = torch.as_tensor(np.asarray(snap["refcount"], np.int32), device=self.dev)
        fl = np.full(self.free_list.numel(), -1, np.int32)
        fl[:len(snap["free_list"])] = np.asarray(snap["free_list"], np.int32)
        self.table.view(-1).copy_(tab)
        self.refcount.copy_(rc)
        self.free_list.copy_(torch.as_tensor(fl, device=self.dev))
        self.free_count.fill_(int(snap["free_count"]))
        torch.cuda.synchronize(self.dev)

    # ------------------------------------------------------------------ host reads (sync)
    def read_status(self) -> int:
        return int(self.status.item())

    def counts(self):
        torch.cuda.synchronize(self.dev)
        return {"steps": int(self.seq_step_off[-1].item()), "matches": int(self.num_matches.item()),
                "pairs": int(self.num_pairs.item()), "targets": int(self.num_targets.item())}

    def autosize(self, tau_s, top_k=0, pairing=L.PAIR_ALIGNED, cur_mode=L.CUR_ALL, cur_begin=None, cur_end=None,
                 slack=1.0):
        """Count-then-fill: run a1-a4, read the device counts and size every buffer to fit."""
        self.segment()
        self.candidates(tau_s, top_k, pairing, cur_mode, cur_begin, cur_end)
        c = self.counts()
        self.status.zero_()
        caps = Caps(step=self.caps.step, match=max(1, int(c["matches"] * slack)),
                    pair=max(1, int(c["pairs"] * slack)), target=max(1, int(c["targets"] * slack)))
        self.set_caps(caps)
        return c

    def read_steps(self):
        torch.cuda.synchronize(self.dev)
        n = min(int(self.seq_step_off[-1].item()), self.caps.step)
        return {"step_start": self.step_start[:n].cpu().numpy(), "step_end": self.step_end[:n].cpu().numpy(),
                "step_nbag": self.step_nbag[:n].cpu().numpy(), "seq_step_off": self.seq_step_off.cpu().numpy()}

    def read_candidates(self):
        c = self.counts()
        M, P, T = (min(c[k], cap) for k, cap in (("matches", self.caps.match), ("pairs", self.caps.pair),
                                                  ("targets", self.caps.target)))
        m = self.matches[:M * 24].cpu().numpy().view(L.MATCH_DTYPE)
        p = self.pairs[:P * 24].cpu().numpy().view(L.PAIR_DTYPE)
        toff = self.target_off[:T + 1].cpu().numpy()
        return {"matches": {k: m[k].copy() for k in L.MATCH_DTYPE.names},
                "pairs": {k: p[k].copy() for k in L.PAIR_DTYPE.names}, "target_off": toff}

    def read_distance(self):
        c = self.counts()
        P, T = min(c["pairs"], self.caps.pair), min(c["targets"], self.caps.target)
        dec = self.decisions[:T * 32].cpu().numpy().view(L.DECISION_DTYPE)
        return {"distance": self.distance[:P].cpu().numpy(), "under": self.under[:P].cpu().numpy(),
                "decisions": {k: dec[k].copy() for k in L.DECISION_DTYPE.names}}

    def read_state(self):
        torch.cuda.synchronize(self.dev)
        return {"table": self.table.view(self.num_seqs, self.table_stride).cpu().numpy(),
                "refcount": self.refcount.cpu().numpy(), "free_list": self.free_list.cpu().numpy(),
                "free_count": int(self.free_count.item()), "num_freed": int(self.num_freed.item()),
                "affected": int(self.affected.item())}
