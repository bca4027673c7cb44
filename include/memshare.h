/* memshare.h -- C ABI of the B200-native MemShare KV-block reuse path (arXiv 2507.21433).
 *
 * Four calls, one per step of the path:
 *   memshare_segment_steps    a1   split token traces into reasoning steps
 *   memshare_step_candidates  a2-a4 Stage 1 bag-of-words cosine filter and the  PAPER.md:224-234,
 *                                  candidate KV-block pair list                 :252-264, :267, :319
 *   memshare_block_distance   a5-a6 Stage 2 normalized block distance, the      PAPER.md:237-248,
 *                                  threshold and the per-target selection       :267-269, :319-320
 *   memshare_remap            a7   zero-copy sharing: block-table rewrite,
 *                                  refcounts, free list
 * plus, around the path:
 *   memshare_block_distance_finalize_peers   KV-head-sharded FINALIZE reading every rank's
 *                                  partial sums over NVLink (the fused cross-rank reduction)
 *   memshare_kv_append / memshare_paged_attention_decode / memshare_admit   f1 decode loop:
 *                                  append, attention through the (remapped) table, admission
 *   memshare_similarity_ratio / memshare_all_pairs   f4 / f3 analysis on the same machinery
 *   memshare_profile_distance_events   measurement hook (events around the streaming kernel)
 *
 * Conventions (all calls):
 *  - Pointers named *_host are host memory; every other pointer is DEVICE memory (cudaMalloc /
 *    torch CUDA tensors). The caller owns every buffer; the library keeps no device memory
 *    between calls. Scratch comes from `workspace` (device, >= the matching *_workspace_size()
 *    bytes, 256-byte aligned); it need not be initialised and may be reused after the call's
 *    stream work completes.
 *  - `stream` is a cudaStream_t passed as void*. Every call validates its host-visible
 *    arguments, then only ENQUEUES work on `stream` and returns: no host synchronisation, no
 *    allocation. Counts produced on the device (num_pairs, num_targets, ...) stay on the device
 *    and later calls read them there, so a whole round runs without a host round trip and can be
 *    captured in a CUDA graph.
 *  - Host-detectable errors return MEMSHARE_ERR_INVALID_ARGUMENT and enqueue nothing. A launch
 *    failure returns MEMSHARE_ERR_CUDA.
 *  - Device-detected errors are written to `*device_status` (int32, device, sticky: the first
 *    error wins; the caller zeroes it before the first call):
 *      MEMSHARE_ERR_CAPACITY   an output exceeded its capacity; the count still holds the
 *                              required size and writes past the capacity were dropped, so the
 *                              caller can re-size and re-run (count-then-fill);
 *      MEMSHARE_ERR_CORRUPTION an id out of range, a refcount underflow, a full free list.
 *  - Outputs are bit-reproducible run to run on the same GPU for the same inputs.
 *  - Layout of the paged KV pool (memshare_kv_pool): bf16; the (layer l, physical block b)
 *    slice of K is the contiguous [d][h_local][d_h] array at k + l*layer_stride + b*block_stride
 *    (element strides; the vLLM-style layer-major pool has block_stride = d*h_local*d_h and
 *    layer_stride = num_blocks*block_stride); V likewise. Bases and strides must be 16-byte
 *    aligned and d_h % 8 == 0.
 */
#ifndef MEMSHARE_H
#define MEMSHARE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MEMSHARE_ABI_VERSION 1

typedef int32_t memshare_status;
#define MEMSHARE_OK 0
#define MEMSHARE_ERR_INVALID_ARGUMENT 1
#define MEMSHARE_ERR_CAPACITY 2
#define MEMSHARE_ERR_CORRUPTION 3
#define MEMSHARE_ERR_CUDA 4

/* Which steps are CURRENT (compared against their history) in memshare_step_candidates.
 * ALL = offline, every finished step; LAST = online, the last finished step of each sequence
 * ("for each decoding step"); RANGE = local steps [cur_begin[s], cur_end[s]). */
#define MEMSHARE_CUR_ALL 0
#define MEMSHARE_CUR_LAST 1
#define MEMSHARE_CUR_RANGE 2

/* Block pairing between a current step k and a candidate step j (reading R14):
 * ALIGNED = i-th full block of k with the i-th full block of j ("corresponding");
 * CROSS = every full block of k with every full block of j ("pairwise"). */
#define MEMSHARE_PAIR_ALIGNED 0
#define MEMSHARE_PAIR_CROSS 1

/* memshare_block_distance modes: FULL streams the pool and finalizes; PARTIAL streams the
 * pool and writes per-(pair, layer) squared sums for a cross-rank all-reduce (KV-head-sharded
 * mode); FINALIZE reads the (all-reduced) squared sums and finalizes without the pool. */
#define MEMSHARE_DIST_FULL 0
#define MEMSHARE_DIST_PARTIAL 1
#define MEMSHARE_DIST_FINALIZE 2
/* Schedule hint OR'ed into the memshare_block_distance mode (FULL or PARTIAL, Euclidean metric;
 * ignored otherwise): the list's consecutive targets share their sources -- CROSS pairing, the
 * all-pairs matrix -- so runs of targets whose source list is a prefix of the next target's are
 * evaluated together, every shared source slice staged once for up to four targets. Same
 * definitions and outputs; only the fixed fp32 summation order of the partials differs. */
#define MEMSHARE_DIST_GROUPED 0x100

/* Stage-2 block metric. EUCLIDEAN is Alg. 1 Stage 2. COSINE is the variant the
 * paper compares against (Fig. 7, reading R34): per layer the cosine of the K
 * slices and of the V slices, D = 1 - (1/N) sum_l (cos_K + cos_V)/2 in [0, 2], so the same strict
 * D < tau_b test and argmin selection apply; FULL mode only. */
#define MEMSHARE_METRIC_EUCLIDEAN 0
#define MEMSHARE_METRIC_COSINE 1

#define MEMSHARE_MAX_DELIMS 16

/* KV geometry. num_kv_heads_global is the h of Alg. 1's 2dh normaliser (reading R17); the pool
 * holds num_kv_heads_local of them (== global unless head-sharded). */
typedef struct memshare_dims {
  int32_t num_layers;          /* N, 1..256 */
  int32_t num_kv_heads_local;  /* heads stored in this pool */
  int32_t num_kv_heads_global; /* h in (Delta_K + Delta_V)/(2dh) */
  int32_t head_dim;            /* d_h, multiple of 8 */
  int32_t block_size;          /* d, tokens per block (reading R18) */
} memshare_dims;

typedef struct memshare_kv_pool {
  const void* k;        /* bf16, device */
  const void* v;        /* bf16, device */
  int64_t layer_stride; /* elements */
  int64_t block_stride; /* elements */
  int32_t num_blocks;   /* physical blocks addressable through this pool */
  int32_t reserved;
} memshare_kv_pool;

/* One Stage-1 survivor: step `cand_step` of sequence `seq` is a candidate of current step
 * `step` (local step indices), `rank`-th by (cosine desc, cand_step asc). 24 bytes. */
typedef struct memshare_step_match {
  int32_t seq, step, cand_step, rank;
  double cosine;
} memshare_step_match;

/* One candidate KV-block pair: logical blocks of `seq` and their physical ids as read from the
 * block table at call time; pairs are grouped by target (target_idx ascending = ascending
 * (seq, target_logical)), sources ascending by logical. 24 bytes. */
typedef struct memshare_block_pair {
  int32_t seq, target_idx, target_logical, source_logical, target_phys, source_phys;
} memshare_block_pair;

/* One per target: the minimal-distance source (ties -> smaller source_logical) and whether it
 * is reused (distance < tau_b). 32 bytes. */
typedef struct memshare_decision {
  int32_t seq, target_logical, target_phys, source_logical, source_phys, accepted;
  float distance;
  int32_t num_candidates;
} memshare_decision;

/* ---------------------------------------------------------------------------------------- a1
 * Step segmentation (steps "separated by delimiters like \n\n").
 * A step ends at token i when t[i] is a delimiter and t[i+1] is not (the delimiter run belongs
 * to the step it ends), or at the last token of a FINAL sequence; tokens before gen_start[s]
 * are the prompt. Only finished steps are emitted; an open tail is not a step (reading R3).
 *   tokens        int32 [num_tokens]             concatenated token ids of all sequences
 *   num_tokens    host int64 == seq_tok_off[num_seqs] (< 2^31 - 4096; sizes the tile grid)
 *   seq_tok_off   int64 [num_seqs+1]             sequence s = tokens[seq_tok_off[s] .. [s+1]),
 *                                                non-decreasing, seq_tok_off[0] = 0
 *   gen_start     int32 [num_seqs]               first generated position of each sequence
 *   seq_final     uint8 [num_seqs]               1 = sequence finished
 *   delim_ids_host int32 [num_delims] (host)     1..MEMSHARE_MAX_DELIMS delimiter token ids
 * Outputs (global step index g = seq_step_off[s] + local step m):
 *   step_start/step_end int32 [step_cap]         [start, end) relative to the sequence start
 *   step_nbag     int32 [step_cap]               content (non-delimiter) tokens of the step
 *   seq_step_off  int64 [num_seqs+1]             always written in full (the required size is
 *                                                seq_step_off[num_seqs]; CAPACITY if > step_cap)
 * Implementation: one single-pass kernel, tile-parallel over the flat token array (2048 tokens
 * per CTA, tiles handed out by an atomic ticket so a tile only waits on tiles already claimed by
 * running CTAs) with a decoupled look-back scan of (step ends, content tokens, last step
 * boundary), so one long sequence spreads over many SMs; a one-CTA kernel zeroes the per-tile
 * flags and the ticket first (no memset node). A wait that does not end within 2 s reports
 * CORRUPTION instead of hanging.
 * Errors: INVALID_ARGUMENT for null pointers, num_seqs < 0, num_delims outside 1..16, step_cap
 * < 0, a short workspace. */
memshare_status memshare_segment_steps(const int32_t* tokens, int64_t num_tokens, const int64_t* seq_tok_off,
                                       const int32_t* gen_start, const uint8_t* seq_final, int32_t num_seqs,
                                       const int32_t* delim_ids_host, int32_t num_delims, int32_t* step_start,
                                       int32_t* step_end, int32_t* step_nbag, int64_t* seq_step_off, int64_t step_cap,
                                       void* workspace, size_t workspace_bytes, int32_t* device_status, void* stream);
size_t memshare_segment_steps_workspace_size(int64_t num_tokens, int32_t num_seqs, int64_t step_cap);

/* ------------------------------------------------------------------------------------- a2-a4
 * Stage 1 + candidate block pairs (Alg. 1 Stage 1; "bag-of-words",
 * PAPER.md:254; threshold "exceeding"; "their corresponding KV cache blocks",
 * PAPER.md:267).
 * For every CURRENT non-void step k of sequence s (cur_mode) and every earlier non-void step j of
 * the same sequence: dot = <c_k, c_j> over the content-token count vectors (int64, exact),
 * cos = (double)dot / sqrt((double)|c_k|^2 * (double)|c_j|^2) (IEEE round-to-nearest, no
 * contraction); j survives iff cos > tau_s; survivors ordered (cos desc, j asc), the first top_k
 * kept (0 = all). Each survivor yields block pairs between the full blocks
 * F = [ceil(start/d), floor(end/d)) of k (targets) and of j (sources), ALIGNED or CROSS; physical
 * ids come from block_table AS GIVEN (snapshot); per target, a source whose physical id repeats
 * is dropped (the smaller logical is kept).
 *   tokens, num_tokens, seq_tok_off, num_seqs       as for memshare_segment_steps
 *   seq_step_off, step_start, step_end, step_nbag   memshare_segment_steps outputs; step_cap is
 *                                                    their capacity
 *   cur_begin/cur_end int32 [num_seqs]              only for MEMSHARE_CUR_RANGE (else NULL)
 *   block_table   int32 [num_seqs][table_stride]    logical -> physical, entries < num_blocks
 *   tau_s in [-1, 1]; top_k >= 0; pairing ALIGNED|CROSS; block_size = d
 * Outputs: matches [match_cap] ordered (seq, step, rank); pairs [pair_cap] grouped by target;
 *   target_off int64 [target_cap+1] (pairs of target t are [target_off[t], target_off[t+1]));
 *   num_matches/num_pairs/num_targets int64 (device).
 * Limits (CAPACITY if exceeded): <= 1024 survivors per current step when top_k == 0 or
 *   top_k > 512; <= 4096 full blocks per step.
 * Implementation: current steps are work items taken from an atomic ticket (one CTA, or one
 * thread-block cluster sharing the history scan over DSMEM in online LAST and RANGE rounds; RANGE
 * work items are the current steps only, listed by the encode kernel); an item's output offsets
 * are the sum of the counts every earlier item published, so it only ever waits on items running
 * CTAs already hold (a wait beyond 2 s reports CORRUPTION). */
memshare_status memshare_step_candidates(
    const int32_t* tokens, int64_t num_tokens, const int64_t* seq_tok_off, int32_t num_seqs,
    const int64_t* seq_step_off, const int32_t* step_start, const int32_t* step_end, const int32_t* step_nbag,
    int64_t step_cap, const int32_t* delim_ids_host, int32_t num_delims, int32_t cur_mode, const int32_t* cur_begin,
    const int32_t* cur_end, const int32_t* block_table, int32_t table_stride, int32_t num_blocks, int32_t block_size,
    double tau_s, int32_t top_k, int32_t pairing, memshare_step_match* matches, int64_t match_cap,
    int64_t* num_matches, memshare_block_pair* pairs, int64_t pair_cap, int64_t* num_pairs, int64_t* target_off,
    int64_t target_cap, int64_t* num_targets, void* workspace, size_t workspace_bytes, int32_t* device_status,
    void* stream);
size_t memshare_step_candidates_workspace_size(int64_t num_tokens, int32_t num_seqs, int64_t step_cap,
                                               int64_t match_cap);

/* ------------------------------------------------------------------------------------- a5-a6
 * Stage 2 block distance, threshold and selection (Alg. 1 Stage 2):
 *   D = (1/N) * sum_l ( ||K_l[Bt] - K_l[Bs]||_F + ||V_l[Bt] - V_l[Bs]||_F ) / (2 d h_global)
 * for every pair (Bt = target_phys, Bs = source_phys), bf16 inputs, fp32 accumulation (chains of
 * <= 64 terms, warp trees, fixed-order cross-warp sums), fp64 finalisation, fp32 result.
 * under[p] = D_p < tau_b. Per target: the pair of minimal D (exact ties -> smaller
 * source_logical), accepted = D_best < tau_b.
 *   pool, dims (host structs)     geometry; pool unused in FINALIZE mode
 *   pairs, target_off, num_pairs, num_targets   memshare_step_candidates outputs (device);
 *                                 counts are clamped to pair_cap / target_cap
 *   mode FULL | PARTIAL | FINALIZE, optionally | MEMSHARE_DIST_GROUPED (schedule hint, see its
 *                                 definition); metric EUCLIDEAN | COSINE (COSINE: FULL mode only)
 *   workspace                     >= memshare_block_distance_workspace_size(); caller-owned, no
 *                                 initial contents required (every call resets what it uses)
 *   partial_sq float [pair_cap][N][2]   PARTIAL: output (sum over local heads of squared
 *                                 differences, [.][l][0] = K, [.][l][1] = V); FINALIZE: input;
 *                                 FULL: optional output (may be NULL)
 *   distance float [pair_cap], under uint8 [pair_cap], decisions [target_cap]: outputs
 *                                 (FULL and FINALIZE; ignored in PARTIAL and may be NULL)
 * Errors: INVALID_ARGUMENT for bad geometry/alignment/mode, tau_b < 0 or NaN, a short
 * workspace; device CORRUPTION for a physical id outside [0, num_blocks). */
memshare_status memshare_block_distance(const memshare_kv_pool* pool_host, const memshare_dims* dims_host,
                                        const memshare_block_pair* pairs, const int64_t* target_off,
                                        const int64_t* num_pairs, const int64_t* num_targets, int64_t pair_cap,
                                        int64_t target_cap, int32_t mode, int32_t metric, float* partial_sq, float tau_b,
                                        float* distance, uint8_t* under, memshare_decision* decisions,
                                        void* workspace, size_t workspace_bytes, int32_t* device_status,
                                        void* stream);
size_t memshare_block_distance_workspace_size(const memshare_dims* dims_host, int32_t num_blocks, int64_t pair_cap,
                                              int64_t target_cap, int32_t metric);

/* ---------------------------------------------------------------------------------------- a7
 * Zero-copy remap (PAPER.md:276-278 "the mechanism simply updates the block table", :283-284;
 * SPEC.md:358-366). Decisions must be strictly ascending in (seq, target_logical) (as
 * memshare_block_distance emits them; else device INVALID_ARGUMENT and nothing is changed). For
 * each accepted decision: old = block_table[seq][target_logical], new = source_phys; equal ->
 * no-op; else the entry becomes new, refcount[new] += 1, refcount[old] -= 1 and
 * *affected_tokens += block_size. A block is FREED iff it was decremented in this call and its
 * final refcount is 0; freed ids are appended to free_list[*free_count ...] in ascending order of
 * their last decrementing decision, *free_count advances and *num_freed = freed count.
 * No KV byte is read or written (zero-copy).
 *   block_table int32 [num_seqs][table_stride]; refcount int32 [num_blocks];
 *   free_list int32 [num_blocks]; free_count, num_freed, affected_tokens int64 (device)
 *   decisions [target_cap], num_targets int64 (device; clamped to target_cap)
 * Device CORRUPTION: an id outside its range, a final refcount < 0, a free-list overflow (the
 * state is then unspecified). */
memshare_status memshare_remap(int32_t* block_table, int32_t table_stride, int32_t num_seqs, int32_t* refcount,
                               int32_t num_blocks, int32_t* free_list, int64_t* free_count,
                               const memshare_decision* decisions, const int64_t* num_targets, int64_t target_cap,
                               int32_t block_size, int64_t* num_freed, int64_t* affected_tokens, void* workspace,
                               size_t workspace_bytes, int32_t* device_status, void* stream);
size_t memshare_remap_workspace_size(int32_t num_blocks, int64_t target_cap);

/* ------------------------------------------------------------------------------------- a5-a7
 * memshare_block_distance (FULL mode) and memshare_remap as ONE call, for a round that applies its
 * decisions at once (score, select, then "the block table is updated",
 * PAPER.md:276-278). Results are identical to memshare_block_distance(mode = FULL) followed by
 * memshare_remap on the same stream: the same distances, under flags and decisions (bit for bit),
 * the same table / refcount / free-list update and counters, the same device errors (a remap
 * validation failure changes nothing). Arguments are those of the two calls; num_blocks is
 * pool_host->num_blocks; partial_sq is not produced.
 *   workspace >= memshare_block_distance_remap_workspace_size() bytes.
 * Implementation: the streaming kernel and the finalisation kernel of memshare_block_distance; the
 * finalisation kernel's last CTA to finish then applies the decisions -- one launch fewer than the
 * two calls. `metric` may carry MEMSHARE_DIST_GROUPED (the schedule hint of
 * memshare_block_distance's mode). Errors: as memshare_block_distance and memshare_remap. */
memshare_status memshare_block_distance_remap(
    const memshare_kv_pool* pool_host, const memshare_dims* dims_host, const memshare_block_pair* pairs,
    const int64_t* target_off, const int64_t* num_pairs, const int64_t* num_targets, int64_t pair_cap,
    int64_t target_cap, int32_t metric, float tau_b, float* distance, uint8_t* under, memshare_decision* decisions,
    int32_t* block_table, int32_t table_stride, int32_t num_seqs, int32_t* refcount, int32_t* free_list,
    int64_t* free_count, int32_t block_size, int64_t* num_freed, int64_t* affected_tokens, void* workspace,
    size_t workspace_bytes, int32_t* device_status, void* stream);
size_t memshare_block_distance_remap_workspace_size(const memshare_dims* dims_host, int32_t num_blocks,
                                                    int64_t pair_cap, int64_t target_cap, int32_t metric);

/* ---------------------------------------------------------------------------------------- f4
 * Similarity ratio (Fig. 2: "the proportion of reasoning steps whose cosine
 * similarity with any previous step exceeds a specified threshold"). From memshare_step_candidates'
 * matches (run with that threshold as tau_s, cur_mode ALL, any top_k >= 1): redundant_steps[s] =
 * number of steps of sequence s with a rank-0 match; ratio_s = redundant_steps[s] /
 * (seq_step_off[s+1] - seq_step_off[s]) (step 0 never counts: it has no history).
 *   matches [match_cap], num_matches int64 (device); redundant_steps int64 [num_seqs] (device, out) */
memshare_status memshare_similarity_ratio(const memshare_step_match* matches, const int64_t* num_matches,
                                          int64_t match_cap, int32_t num_seqs, int64_t* redundant_steps,
                                          int32_t* device_status, void* stream);

/* ---------------------------------------------------------------------------------------- f3
 * All block pairs of per-sequence logical-block windows (Observation 2: "block-wise
 * Euclidean distance between KV caches" heatmaps; SPEC.md:271-279 all-pairs oracle): for each
 * sequence s, every pair (i, j) with blk_begin[s] <= i < j < min(blk_end[s], full blocks of s),
 * target j / source i, grouped by target (ascending (s, j)), sources ascending; physical ids from
 * block_table. Score with memshare_block_distance (pair_cap >= sum m(m-1)/2); D(i,j) = D(j,i).
 *   seq_tok_off int64 [num_seqs+1]; blk_begin/blk_end int32 [num_seqs] (device); outputs as for
 *   memshare_step_candidates (pairs, num_pairs, target_off, num_targets; CAPACITY semantics). */
memshare_status memshare_all_pairs(const int64_t* seq_tok_off, int32_t num_seqs, const int32_t* blk_begin,
                                   const int32_t* blk_end, const int32_t* block_table, int32_t table_stride,
                                   int32_t num_blocks, int32_t block_size, memshare_block_pair* pairs, int64_t pair_cap,
                                   int64_t* num_pairs, int64_t* target_off, int64_t target_cap, int64_t* num_targets,
                                   void* workspace, size_t workspace_bytes, int32_t* device_status, void* stream);
size_t memshare_all_pairs_workspace_size(int32_t num_seqs);

/* Human-readable name of a status code (static string). */
const char* memshare_status_string(memshare_status status);
/* MEMSHARE_ABI_VERSION of the loaded library. */
int32_t memshare_abi_version(void);

/* Profiling hook (measurement only): when begin/end are non-NULL cudaEvent_t handles, every
 * subsequent memshare_block_distance call on this host thread records `begin` immediately before
 * and `end` immediately after its streaming kernel, on the call's stream, so the kernel's
 * device time can be read apart from the finalisation; NULL, NULL turns it off. */
void memshare_profile_distance_events(void* begin, void* end);

/* memshare_block_distance_finalize_peers -- FINALIZE for the KV-head-sharded mode with the
 * cross-rank reduction fused in (reading R17): instead of an all-reduce of the
 * PARTIAL squared sums followed by FINALIZE, each rank's finalisation loads every rank's
 * partial_sq directly over NVLink / NVSwitch (peer mappings, e.g. symmetric memory) and sums them
 * in rank order, so every rank computes bit-identical distances and decisions.
 *   partial_peers  DEVICE array [num_peers] of device pointers, valid on the calling GPU: rank r's
 *                  float [pair_cap][N][2] PARTIAL output (rank order, 1 <= num_peers <= 64); every
 *                  rank's PARTIAL call must be complete and visible before this call runs (the
 *                  caller issues a device-side barrier, e.g. symmetric-memory barrier, first)
 *   dims           num_kv_heads_global is the h of the 2dh normaliser
 *   other arguments and outputs as memshare_block_distance in FINALIZE mode. */
memshare_status memshare_block_distance_finalize_peers(
    const float* const* partial_peers, int32_t num_peers, const memshare_dims* dims_host,
    const memshare_block_pair* pairs, const int64_t* target_off, const int64_t* num_pairs,
    const int64_t* num_targets, int64_t pair_cap, int64_t target_cap, float tau_b, float* distance, uint8_t* under,
    memshare_decision* decisions, void* workspace, size_t workspace_bytes, int32_t* device_status, void* stream);

/* ---------------------------------------------------------------------------------------- f1
 * Decode-loop integration: the steps on either side of the MemShare path. Shared blocks are
 * read "through the block table" by paged attention, with no copy.
 *
 * memshare_kv_append -- one decode token per active sequence into the paged pool (reading R35).
 *   k_pool/v_pool   bf16 device pools, layout K[l][block][tau][head][x] (written)
 *   layer_stride, block_stride, num_blocks   as in memshare_kv_pool (elements; multiples of 8)
 *   dims_host       num_layers, num_kv_heads_local (heads stored in the pool), head_dim, block_size
 *   block_table     int32 [num_seqs][table_stride] (device, updated)
 *   seq_len         int32 [num_seqs] tokens already stored per sequence (device, +1 per active)
 *   active          uint8 [num_seqs] or NULL (= all active)
 *   refcount        int32 [num_blocks]; free_list int32 [..]; free_count int64 [1] (device, updated)
 *   new_k/new_v     bf16 [num_layers][num_seqs][num_kv_heads_local][head_dim] (device, 16-byte aligned)
 * Sequence s writes its row at position seq_len[s]; when seq_len[s] % block_size == 0 it first
 * takes a fresh block from the END of the free list (LIFO, in sequence order), sets its refcount
 * to 1 and enters it in the table. All-or-nothing: on a device-detected error nothing changes and
 * device_status receives CAPACITY (not enough free blocks, or the table row is full),
 * CORRUPTION (the tail block is shared, refcount != 1, or a popped block is not free) or
 * INVALID_ARGUMENT (negative seq_len). Host errors: INVALID_ARGUMENT. */
memshare_status memshare_kv_append(void* k_pool, void* v_pool, int64_t layer_stride, int64_t block_stride,
                                   int32_t num_blocks, const memshare_dims* dims_host, int32_t* block_table,
                                   int32_t table_stride, int32_t num_seqs, int32_t* seq_len, const uint8_t* active,
                                   int32_t* refcount, int32_t* free_list, int64_t* free_count, const void* new_k,
                                   const void* new_v, void* workspace, size_t workspace_bytes, int32_t* device_status,
                                   void* stream);
size_t memshare_kv_append_workspace_size(int32_t num_seqs);

/* memshare_paged_attention_decode -- one layer of GQA decode attention through the block table
 * (reading R36): for sequence s and query head qh (KV head g = qh / (num_q_heads / h_local)),
 *   out[s][qh] = sum_{j < seq_len[s]} softmax_j(scale * <q[s][qh], K_l[table[s][j/d]][j%d][g]>)
 *                * V_l[table[s][j/d]][j%d][g]
 *   pool_host/dims_host  the KV pool (block_size must be 16, head_dim 64 or 128)
 *   layer           which layer l
 *   q               bf16 [num_seqs][num_q_heads][head_dim] (device); num_q_heads = G * h_local,
 *                   1 <= G <= 8
 *   seq_len         int32 [num_seqs] (device); 0 gives a zero output
 *   max_seq_len     host upper bound of seq_len (sizes the split-KV grid and the workspace);
 *                   table_stride >= ceil(max_seq_len / 16)
 *   out             fp32 [num_seqs][num_q_heads][head_dim] (device)
 * Implementation: split-KV over chunks of 1,024 / 512 / 256 tokens -- the largest that still gives
 * >= 4 CTAs per SM (one CTA per chunk x KV head x sequence, fp32 online softmax) -- then one warp
 * per (sequence, query head) combines the chunks. A table entry
 * outside [0, num_blocks) sets CORRUPTION. Host errors: INVALID_ARGUMENT. */
memshare_status memshare_paged_attention_decode(const memshare_kv_pool* pool_host, const memshare_dims* dims_host,
                                                int32_t layer, const void* q, int32_t num_q_heads,
                                                const int32_t* block_table, int32_t table_stride,
                                                const int32_t* seq_len, int32_t num_seqs, int32_t max_seq_len,
                                                float scale, float* out, void* workspace, size_t workspace_bytes,
                                                int32_t* device_status, void* stream);
size_t memshare_paged_attention_workspace_size(const memshare_dims* dims_host, int32_t num_seqs, int32_t num_q_heads,
                                               int32_t max_seq_len);

/* memshare_admit -- HOST function, block-budget admission (reading R37; the mechanism behind
 * PAPER.md Fig. 6: blocks freed by sharing admit more concurrent sequences). Waiting request i
 * (in queue order) needs ceil((prompt_len_host[i] + reserve) / block_size) blocks; requests are
 * admitted first-come-first-served while their need fits in free_blocks and admission stops at
 * the first that does not fit. Returns the number admitted (a prefix of the queue) and writes
 * their total need to *blocks_used_host (if not NULL); -1 for invalid arguments. */
int32_t memshare_admit(const int32_t* prompt_len_host, int32_t num_waiting, int32_t reserve, int32_t block_size,
                       int64_t free_blocks, int64_t* blocks_used_host);

#ifdef __cplusplus
}
#endif

#endif /* MEMSHARE_H */
