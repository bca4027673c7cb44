/* memshare_oracle.c -- TEST INFRASTRUCTURE, NOT THE PRODUCT.
 *
 * A plain, slow, single-threaded C99 reference of MemShare's collaborative-filtering
 * KV-block reuse path (arXiv 2507.21433), written from /root/reference/PAPER.md:
 *   Algorithm 1 Stage 1, Stage 2,
 *   the zero-copy block-table sharing mechanism, and the cosine block
 *   metric the paper compares Stage 2 against (f2).
 * Floating point is fp64 throughout (bf16 -> double is exact). No SIMD, no threads, no
 * blocking or reordering beyond what the definitions state. Where the paper is silent or
 * ambiguous the reading taken is the one listed in DESIGN.md §"Readings" (R-numbers below).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg, --impl reference)
 * may load this library. It shares no code and no header with the CUDA path
 * (paper_2507_21433_b200/), and neither imports the other.
 *
 * Parity pins: every function below is pinned by -m "not gpu" tests in tests/test_oracle_*.py
 * (worked examples, closed forms, brute force); see DESIGN.md §"Oracle pins".
 *
 * Return codes: 0 ok, 1 invalid argument, 2 capacity (counts hold the required sizes),
 * 3 corruption.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_INVALID 1
#define OR_CAPACITY 2
#define OR_CORRUPTION 3

static int is_delim(int32_t t, const int32_t* delims, int32_t num_delims) {
  for (int32_t i = 0; i < num_delims; ++i)
    if (t == delims[i]) return 1;
  return 0;
}

/* ------------------------------------------------------------------------------------
 * a1. Step segmentation. PAPER.md:119 ("The reasoning model inherently segments the
 * reasoning process into discrete steps, typically separated by delimiters like \n\n").
 * Readings R1-R4: delimiters are a caller-given set of token ids; a step ends at the END
 * of a delimiter run (t[i] in Delta and t[i+1] not in Delta), so the run belongs to the
 * step it terminates and no empty step appears between consecutive delimiters
 * (SPEC.md:176-179); the last token ends a step only if the sequence is final (an open
 * delimiter run may still grow); tokens before gen_start are the prompt, never a step.
 * Outputs per finished step: [start, end) relative to the sequence start and the number of
 * content (non-delimiter) tokens. Returns the total number of finished steps.
 * ------------------------------------------------------------------------------------ */
int64_t oracle_segment_steps(const int32_t* tokens, const int64_t* seq_tok_off, const int32_t* gen_start,
                             const uint8_t* seq_final, int32_t num_seqs, const int32_t* delims,
                             int32_t num_delims, int32_t* step_start, int32_t* step_end, int32_t* step_nbag,
                             int64_t* seq_step_off, int64_t step_cap) {
  int64_t total = 0;
  for (int32_t s = 0; s < num_seqs; ++s) {
    const int32_t* t = tokens + seq_tok_off[s];
    const int64_t n = seq_tok_off[s + 1] - seq_tok_off[s];
    seq_step_off[s] = total;
    int64_t cur_start = gen_start[s];
    int32_t nbag = 0;
    for (int64_t i = gen_start[s]; i < n; ++i) {
      const int d_here = is_delim(t[i], delims, num_delims);
      if (!d_here) nbag += 1;
      int ends;
      if (i + 1 < n)
        ends = d_here && !is_delim(t[i + 1], delims, num_delims);
      else
        ends = seq_final[s] != 0;
      if (ends) {
        if (total < step_cap) {
          step_start[total] = (int32_t)cur_start;
          step_end[total] = (int32_t)(i + 1);
          step_nbag[total] = nbag;
        }
        total += 1;
        cur_start = i + 1;
        nbag = 0;
      }
    }
  }
  seq_step_off[num_seqs] = total;
  return total;
}

/* ------------------------------------------------------------------------------------
 * a2. Bag-of-words encoding. PAPER.md:228-230 (v <- T.encode(s)) and :254 ("Each step is
 * converted into a bag-of-words vector representation"). Reading R6/R7: the generated
 * token ids are used directly; the vector is the count vector of the step's content
 * (non-delimiter) tokens, stored sparse as ascending (id, count).
 * ------------------------------------------------------------------------------------ */
static int cmp_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

typedef struct {
  int32_t n;       /* distinct ids */
  int32_t* ids;    /* ascending */
  int64_t* cnt;
  int64_t n2;      /* sum of count^2 = ||v||^2 */
} bag_t;

static void bag_of_words(const int32_t* t, int64_t len, const int32_t* delims, int32_t num_delims, bag_t* out) {
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(len > 0 ? len : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < len; ++i)
    if (!is_delim(t[i], delims, num_delims)) tmp[m++] = t[i];
  qsort(tmp, (size_t)m, sizeof(int32_t), cmp_i32);
  out->ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  out->cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
  out->n = 0;
  out->n2 = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (out->n > 0 && out->ids[out->n - 1] == tmp[i]) {
      out->cnt[out->n - 1] += 1;
    } else {
      out->ids[out->n] = tmp[i];
      out->cnt[out->n] = 1;
      out->n += 1;
    }
  }
  for (int32_t i = 0; i < out->n; ++i) out->n2 += out->cnt[i] * out->cnt[i];
  free(tmp);
}

static void bag_free(bag_t* b) {
  free(b->ids);
  free(b->cnt);
}

/* <v_a, v_b> over the common ids (sparse merge of the two ascending lists) */
static int64_t bag_dot(const bag_t* a, const bag_t* b) {
  int64_t dot = 0;
  int32_t i = 0, j = 0;
  while (i < a->n && j < b->n) {
    if (a->ids[i] < b->ids[j]) i++;
    else if (a->ids[i] > b->ids[j]) j++;
    else { dot += a->cnt[i] * b->cnt[j]; i++; j++; }
  }
  return dot;
}

/* sim = <v_curr, v_i> / (||v_curr||_2 * ||v_i||_2), PAPER.md:231 (Alg. 1 Stage 1 line 4).
 * Reading R12: one IEEE round-to-nearest expression, product of the squared norms under one
 * square root. */
double oracle_cosine(int64_t dot, int64_t n2_a, int64_t n2_b) {
  return (double)dot / sqrt((double)n2_a * (double)n2_b);
}

/* exposed for pins: bag of one token list (ids ascending, counts) */
int32_t oracle_bag(const int32_t* t, int64_t len, const int32_t* delims, int32_t num_delims, int32_t* ids_out,
                   int64_t* cnt_out, int64_t* n2_out) {
  bag_t b;
  bag_of_words(t, len, delims, num_delims, &b);
  for (int32_t i = 0; i < b.n; ++i) { ids_out[i] = b.ids[i]; cnt_out[i] = b.cnt[i]; }
  *n2_out = b.n2;
  const int32_t n = b.n;
  bag_free(&b);
  return n;
}

/* ------------------------------------------------------------------------------------
 * a3 + a4. Stage 1 candidates and candidate block pairs.
 * Stage 1 ("all preceding steps" PAPER.md:121; "scores exceeding the
 * predefined threshold (e.g., 0.8 or 0.9) proceed" PAPER.md:318): for each CURRENT step k of
 * a sequence and each earlier non-void step j of the same sequence (R5, R9), keep j iff
 * cos > tau_s (strict, R10); order kept j by (cos desc, j asc) and keep the first top_k
 * (0 = all) (R11).
 * Pairs (PAPER.md:267 "their corresponding KV cache blocks", :319-320 "pairwise distances
 * between candidate blocks"): F_k = [ceil(start_k/d), floor(end_k/d)) are the blocks fully
 * inside step k (R13). ALIGNED pairs the i-th full block of k with the i-th of j; CROSS pairs
 * F_k x F_j (R14). Physical ids come from the block table as given (snapshot, R25). Per
 * target, sources are listed by ascending source logical and a source whose physical id
 * already appeared is dropped (dedupe keeps the smallest logical). Targets are numbered in
 * ascending (seq, target logical).
 * cur_mode: 0 = every step is current, 1 = only the last finished step of each sequence,
 * 2 = local steps [cur_begin[s], cur_end[s]).
 * Outputs (SoA): matches (seq, step, cand_step, rank, cosine), pairs (seq, target_idx,
 * target_logical, source_logical, target_phys, source_phys), target_off[T+1].
 * ------------------------------------------------------------------------------------ */
typedef struct { double cos; int32_t j; } cand_t;

static int32_t ceil_div(int32_t a, int32_t b) { return (a + b - 1) / b; }

int oracle_step_candidates(const int32_t* tokens, const int64_t* seq_tok_off, int32_t num_seqs,
                           const int64_t* seq_step_off, const int32_t* step_start, const int32_t* step_end,
                           const int32_t* delims, int32_t num_delims, int32_t cur_mode, const int32_t* cur_begin,
                           const int32_t* cur_end, const int32_t* block_table, int32_t table_stride,
                           int32_t block_size, double tau_s, int32_t top_k, int32_t pairing,
                           int32_t* m_seq, int32_t* m_step, int32_t* m_cand, int32_t* m_rank, double* m_cos,
                           int64_t match_cap, int64_t* num_matches,
                           int32_t* p_seq, int32_t* p_tidx, int32_t* p_tl, int32_t* p_sl, int32_t* p_tp,
                           int32_t* p_sp, int64_t pair_cap, int64_t* num_pairs,
                           int64_t* target_off, int64_t target_cap, int64_t* num_targets) {
  int64_t M = 0, P = 0, T = 0;
  for (int32_t s = 0; s < num_seqs; ++s) {
    const int64_t first = seq_step_off[s];
    const int32_t S = (int32_t)(seq_step_off[s + 1] - first);
    const int32_t* t = tokens + seq_tok_off[s];
    bag_t* bags = (bag_t*)malloc(sizeof(bag_t) * (size_t)(S > 0 ? S : 1));
    for (int32_t m = 0; m < S; ++m)
      bag_of_words(t + step_start[first + m], step_end[first + m] - step_start[first + m], delims, num_delims,
                   &bags[m]);
    int32_t lo = 0, hi = S;
    if (cur_mode == 1) lo = S > 0 ? S - 1 : 0;
    if (cur_mode == 2) {
      lo = cur_begin[s] < 0 ? 0 : cur_begin[s];
      hi = cur_end[s] > S ? S : cur_end[s];
    }
    cand_t* cands = (cand_t*)malloc(sizeof(cand_t) * (size_t)(S > 0 ? S : 1));
    for (int32_t k = lo; k < hi; ++k) {
      if (bags[k].n == 0) continue;                     /* void step: never current (R5) */
      int32_t nc = 0;
      for (int32_t j = 0; j < k; ++j) {
        if (bags[j].n == 0) continue;                   /* void step: never a candidate */
        const double c = oracle_cosine(bag_dot(&bags[k], &bags[j]), bags[k].n2, bags[j].n2);
        if (c > tau_s) { cands[nc].cos = c; cands[nc].j = j; nc++; }
      }
      /* stable insertion sort by cos descending; j ascending already holds for ties */
      for (int32_t a = 1; a < nc; ++a) {
        cand_t x = cands[a];
        int32_t b = a - 1;
        while (b >= 0 && cands[b].cos < x.cos) { cands[b + 1] = cands[b]; b--; }
        cands[b + 1] = x;
      }
      if (top_k > 0 && nc > top_k) nc = top_k;
      for (int32_t r = 0; r < nc; ++r) {
        if (M < match_cap) {
          m_seq[M] = s; m_step[M] = k; m_cand[M] = cands[r].j; m_rank[M] = r; m_cos[M] = cands[r].cos;
        }
        M++;
      }
      /* candidate steps in ascending j for the ascending-source-logical listing */
      int32_t* js = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nc > 0 ? nc : 1));
      for (int32_t r = 0; r < nc; ++r) js[r] = cands[r].j;
      qsort(js, (size_t)nc, sizeof(int32_t), cmp_i32);
      const int32_t fk_lo = ceil_div(step_start[first + k], block_size);
      const int32_t fk_hi = step_end[first + k] / block_size;
      int32_t max_src = 0;
      for (int32_t r = 0; r < nc; ++r) {
        const int32_t flo = ceil_div(step_start[first + js[r]], block_size), fhi = step_end[first + js[r]] / block_size;
        max_src += (fhi > flo ? fhi - flo : 0);
      }
      int32_t* src_l = (int32_t*)malloc(sizeof(int32_t) * (size_t)(max_src > 0 ? max_src : 1));
      for (int32_t tl = fk_lo; tl < fk_hi; ++tl) {
        const int32_t i = tl - fk_lo;
        int32_t ns = 0;
        for (int32_t r = 0; r < nc; ++r) {
          const int32_t flo = ceil_div(step_start[first + js[r]], block_size), fhi = step_end[first + js[r]] / block_size;
          if (pairing == 0) {
            if (flo + i < fhi) src_l[ns++] = flo + i;
          } else {
            for (int32_t b = flo; b < fhi; ++b) src_l[ns++] = b;
          }
        }
        if (ns == 0) continue;
        const int32_t tp = block_table[(int64_t)s * table_stride + tl];
        int64_t kept = 0;
        for (int32_t a = 0; a < ns; ++a) {
          const int32_t sp = block_table[(int64_t)s * table_stride + src_l[a]];
          int dup = 0;
          for (int32_t b = 0; b < a; ++b)
            if (block_table[(int64_t)s * table_stride + src_l[b]] == sp) { dup = 1; break; }
          if (dup) continue;
          if (P < pair_cap) {
            p_seq[P] = s; p_tidx[P] = (int32_t)T; p_tl[P] = tl; p_sl[P] = src_l[a]; p_tp[P] = tp; p_sp[P] = sp;
          }
          P++;
          kept++;
        }
        if (T < target_cap) target_off[T] = P - kept;
        T++;
      }
      free(src_l);
      free(js);
    }
    free(cands);
    for (int32_t m = 0; m < S; ++m) bag_free(&bags[m]);
    free(bags);
  }
  if (T < target_cap + 1) target_off[T] = P;
  *num_matches = M;
  *num_pairs = P;
  *num_targets = T;
  return (M > match_cap || P > pair_cap || T > target_cap) ? OR_CAPACITY : OR_OK;
}

/* ------------------------------------------------------------------------------------
 * a5. Stage 2 per-layer squared Frobenius distances (Alg. 1 Stage 2
 * lines 3-4: Delta_K <- ||K_i[B1] - K_i[B2]||_2, Delta_V likewise; R16: Frobenius norm
 * over the block's [d x h x d_h] slice). Pool: bf16 bits, layer-major, slice (l, block) =
 * [tau][head][x] contiguous at base + l*layer_stride + block*block_stride (elements).
 * sk/sv[p*N + l] = sum over (tau, head, x) in natural order of (B1 - B2)^2 in fp64.
 * ------------------------------------------------------------------------------------ */
static double bf16_to_double(uint16_t b) {
  union { uint32_t u; float f; } c;
  c.u = (uint32_t)b << 16;
  return (double)c.f;
}

void oracle_partial_sq(const uint16_t* k, const uint16_t* v, int64_t layer_stride, int64_t block_stride,
                       int32_t num_layers, int32_t h_local, int32_t head_dim, int32_t block_size,
                       const int32_t* tphys, const int32_t* sphys, int64_t P, double* sk, double* sv) {
  const int64_t slice = (int64_t)block_size * h_local * head_dim;
  for (int64_t p = 0; p < P; ++p) {
    for (int32_t l = 0; l < num_layers; ++l) {
      const uint16_t* kt = k + (int64_t)l * layer_stride + (int64_t)tphys[p] * block_stride;
      const uint16_t* ks = k + (int64_t)l * layer_stride + (int64_t)sphys[p] * block_stride;
      const uint16_t* vt = v + (int64_t)l * layer_stride + (int64_t)tphys[p] * block_stride;
      const uint16_t* vs = v + (int64_t)l * layer_stride + (int64_t)sphys[p] * block_stride;
      double SK = 0.0, SV = 0.0;
      for (int64_t e = 0; e < slice; ++e) {
        const double dk = bf16_to_double(kt[e]) - bf16_to_double(ks[e]);
        const double dv = bf16_to_double(vt[e]) - bf16_to_double(vs[e]);
        SK += dk * dk;
        SV += dv * dv;
      }
      sk[p * num_layers + l] = SK;
      sv[p * num_layers + l] = SV;
    }
  }
}

/* a6 (first half). Alg. 1 Stage 2 lines 1, 5, 7:
 *   D <- 0; for each layer: D <- D + (Delta_K + Delta_V)/(2dh); return D/N
 * with d = tokens per block (R18), h = KV heads, global in head-sharded mode (R17). */
void oracle_finalize(const double* sk, const double* sv, int64_t P, int32_t num_layers, int32_t block_size,
                     int32_t h_global, double* D) {
  for (int64_t p = 0; p < P; ++p) {
    double acc = 0.0;
    for (int32_t l = 0; l < num_layers; ++l)
      acc = acc + (sqrt(sk[p * num_layers + l]) + sqrt(sv[p * num_layers + l])) / (2.0 * block_size * h_global);
    D[p] = acc / num_layers;
  }
}

/* Stage 2 end to end for P pairs (partial squares then the Alg. 1 normalisation). */
void oracle_block_distance(const uint16_t* k, const uint16_t* v, int64_t layer_stride, int64_t block_stride,
                           int32_t num_layers, int32_t h_local, int32_t h_global, int32_t head_dim,
                           int32_t block_size, const int32_t* tphys, const int32_t* sphys, int64_t P, double* D) {
  double* sk = (double*)malloc(sizeof(double) * (size_t)(P * num_layers > 0 ? P * num_layers : 1));
  double* sv = (double*)malloc(sizeof(double) * (size_t)(P * num_layers > 0 ? P * num_layers : 1));
  oracle_partial_sq(k, v, layer_stride, block_stride, num_layers, h_local, head_dim, block_size, tphys, sphys, P,
                    sk, sv);
  oracle_finalize(sk, sv, P, num_layers, block_size, h_global, D);
  free(sk);
  free(sv);
}

/* a6 (second half). Selection ("selecting those with minimal distances";
 * :268 "small Euclidean distance are flagged as reusable"). R21/R22: per target the source
 * with minimal D, exact ties to the smaller source logical; accepted iff D_best < tau_b
 * (strict); under[p] = D_p < tau_b. tau_b arrives as fp32 and is compared in fp64. */
void oracle_select(const double* D, int64_t P, const int64_t* target_off, int64_t T, const int32_t* src_logical,
                   float tau_b, int64_t* best, uint8_t* accepted, uint8_t* under) {
  const double tb = (double)tau_b;
  for (int64_t p = 0; p < P; ++p) under[p] = D[p] < tb;
  for (int64_t t = 0; t < T; ++t) {
    int64_t b = target_off[t];
    for (int64_t p = target_off[t] + 1; p < target_off[t + 1]; ++p)
      if (D[p] < D[b] || (D[p] == D[b] && src_logical[p] < src_logical[b])) b = p;
    best[t] = b;
    accepted[t] = D[b] < tb;
  }
}

/* ------------------------------------------------------------------------------------
 * a7. Zero-copy remap ("Upon identifying shareable blocks, the mechanism
 * simply updates the block table", :283-284 zero-copy; SPEC.md:358-366 share_block).
 * R23, R26: accepted decisions are applied in canonical ascending (seq, target logical)
 * order (decisions must be strictly ascending, else INVALID). For each: old = table[T],
 * new = source_phys; equal -> no-op; otherwise table[T] = new, refcount[new] += 1,
 * refcount[old] -= 1, affected += d. After all decisions: a block is FREED iff it was
 * decremented in this call and its final refcount is 0; freed ids are appended to
 * free_list[free_count ...] in the canonical order of their last decrementing decision.
 * A final refcount < 0, an id outside [0, num_blocks) or a full free list is CORRUPTION.
 * ------------------------------------------------------------------------------------ */
int oracle_remap(int32_t* block_table, int32_t table_stride, int32_t* refcount, int32_t num_blocks,
                 int32_t* free_list, int64_t* free_count, const int32_t* dec_seq, const int32_t* dec_tl,
                 const int32_t* dec_sp, const uint8_t* dec_acc, int64_t T, int32_t block_size,
                 int64_t* num_freed, int64_t* affected) {
  *num_freed = 0;
  *affected = 0;
  for (int64_t i = 1; i < T; ++i)
    if (dec_seq[i] < dec_seq[i - 1] || (dec_seq[i] == dec_seq[i - 1] && dec_tl[i] <= dec_tl[i - 1]))
      return OR_INVALID;
  int64_t* last_dec = (int64_t*)malloc(sizeof(int64_t) * (size_t)(num_blocks > 0 ? num_blocks : 1));
  int32_t* old_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(T > 0 ? T : 1));
  for (int32_t b = 0; b < num_blocks; ++b) last_dec[b] = -1;
  int rc = OR_OK;
  for (int64_t i = 0; i < T; ++i) {
    old_of[i] = -1;
    if (!dec_acc[i]) continue;
    int32_t* entry = &block_table[(int64_t)dec_seq[i] * table_stride + dec_tl[i]];
    const int32_t old = *entry, nw = dec_sp[i];
    if (old < 0 || old >= num_blocks || nw < 0 || nw >= num_blocks) { rc = OR_CORRUPTION; goto done; }
    if (old == nw) continue;
    *entry = nw;
    refcount[nw] += 1;
    refcount[old] -= 1;
    last_dec[old] = i;
    old_of[i] = old;
    *affected += block_size;
  }
  for (int32_t b = 0; b < num_blocks; ++b)
    if (refcount[b] < 0) { rc = OR_CORRUPTION; goto done; }
  for (int64_t i = 0; i < T; ++i) {
    const int32_t old = old_of[i];
    if (old < 0) continue;
    if (last_dec[old] == i && refcount[old] == 0) {
      if (*free_count + *num_freed >= num_blocks) { rc = OR_CORRUPTION; goto done; }
      free_list[*free_count + *num_freed] = old;
      *num_freed += 1;
    }
  }
  *free_count += *num_freed;
done:
  free(last_dec);
  free(old_of);
  return rc;
}

/* ------------------------------------------------------------------------------------
 * f4. Similarity ratio numerator ("the proportion of reasoning steps whose
 * cosine similarity with any previous step exceeds a specified threshold"): per sequence, the
 * number of current steps k with max_{j<k} cos(k, j) > tau, i.e. with at least one Stage-1
 * survivor in the match list produced at that tau (rank 0 present).
 * ------------------------------------------------------------------------------------ */
void oracle_similarity_ratio(const int32_t* m_seq, const int32_t* m_rank, int64_t M, int32_t num_seqs,
                             int64_t* redundant_steps) {
  for (int32_t s = 0; s < num_seqs; ++s) redundant_steps[s] = 0;
  for (int64_t i = 0; i < M; ++i)
    if (m_rank[i] == 0) redundant_steps[m_seq[i]] += 1;
}

/* ------------------------------------------------------------------------------------
 * f3. All block pairs of per-sequence windows (Observation 2 heatmaps;
 * SPEC.md:271-279): for each sequence, every (i, j), i < j, of the logical blocks in
 * [blk_begin, min(blk_end, full blocks)), target j, source i, target-major, sources ascending.
 * Returns the pair count (written only below pair_cap); target_off gets T+1 entries.
 * ------------------------------------------------------------------------------------ */
int64_t oracle_all_pairs(const int64_t* seq_tok_off, int32_t num_seqs, const int32_t* blk_begin,
                         const int32_t* blk_end, const int32_t* block_table, int32_t table_stride,
                         int32_t block_size, int32_t* p_seq, int32_t* p_tidx, int32_t* p_tl, int32_t* p_sl,
                         int32_t* p_tp, int32_t* p_sp, int64_t pair_cap, int64_t* target_off, int64_t target_cap,
                         int64_t* num_targets) {
  int64_t P = 0, T = 0;
  for (int32_t s = 0; s < num_seqs; ++s) {
    const int32_t full = (int32_t)((seq_tok_off[s + 1] - seq_tok_off[s]) / block_size);
    const int32_t lo = blk_begin[s] < 0 ? 0 : blk_begin[s];
    int32_t hi = blk_end[s] > full ? full : blk_end[s];
    if (hi < lo) hi = lo;
    for (int32_t j = lo + 1; j < hi; ++j) {
      if (T < target_cap) target_off[T] = P;
      for (int32_t i = lo; i < j; ++i) {
        if (P < pair_cap) {
          p_seq[P] = s; p_tidx[P] = (int32_t)T; p_tl[P] = j; p_sl[P] = i;
          p_tp[P] = block_table[(int64_t)s * table_stride + j];
          p_sp[P] = block_table[(int64_t)s * table_stride + i];
        }
        P++;
      }
      T++;
    }
  }
  if (T <= target_cap) target_off[T] = P;
  *num_targets = T;
  return P;
}

/* ------------------------------------------------------------------------------------
 * f2. Cosine block similarity, the Stage-2 variant the paper compares against (PAPER.md:271-273
 * "While cosine similarity measures only angular alignment between vectors, Euclidean distance
 * captures both directional and magnitude differences"; Fig. 7). Reading R34: per layer the
 * cosine of the flattened K slices and of the V slices; D = 1 - (1/N) sum_l (cos_K + cos_V)/2,
 * so that smaller is more similar like Alg. 1's D. Two all-zero slices have cosine 1, one
 * all-zero slice cosine 0.
 * ------------------------------------------------------------------------------------ */
static double slice_cos(const uint16_t* a, const uint16_t* b, int64_t n) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int64_t e = 0; e < n; ++e) {
    const double x = bf16_to_double(a[e]), y = bf16_to_double(b[e]);
    dot += x * y;
    na += x * x;
    nb += y * y;
  }
  if (na == 0.0 && nb == 0.0) return 1.0;
  if (na == 0.0 || nb == 0.0) return 0.0;
  return dot / sqrt(na * nb);
}

void oracle_block_cosine(const uint16_t* k, const uint16_t* v, int64_t layer_stride, int64_t block_stride,
                         int32_t num_layers, int32_t h_local, int32_t head_dim, int32_t block_size,
                         const int32_t* tphys, const int32_t* sphys, int64_t P, double* D) {
  const int64_t slice = (int64_t)block_size * h_local * head_dim;
  for (int64_t p = 0; p < P; ++p) {
    double acc = 0.0;
    for (int32_t l = 0; l < num_layers; ++l) {
      const int64_t ot = (int64_t)l * layer_stride + (int64_t)tphys[p] * block_stride;
      const int64_t os = (int64_t)l * layer_stride + (int64_t)sphys[p] * block_stride;
      acc += 0.5 * (slice_cos(k + ot, k + os, slice) + slice_cos(v + ot, v + os, slice));
    }
    D[p] = 1.0 - acc / num_layers;
  }
}

/* ------------------------------------------------------------------------------------
 * f1. Decode-loop integration (shared blocks are read "through the block
 * table" by paged attention; :322 vLLM). Readings R35-R37.
 * ------------------------------------------------------------------------------------ */

/* Paged KV append of one decode token per active sequence (reading R35). Sequences are visited
 * in index order; a sequence whose length is a multiple of d takes a fresh block from the END of
 * the free list (LIFO: the last block freed by remap is reused first). The call is all-or-nothing:
 * it returns OR_CAPACITY (nothing changed) if the fresh blocks needed exceed free_count or a
 * position exceeds the table row, and OR_CORRUPTION if a tail block being appended to is not
 * private (refcount != 1) or a popped block is not free (refcount != 0).
 * new_k / new_v: bf16 [num_layers][num_seqs][h][d_h]. */
int oracle_kv_append(uint16_t* k, uint16_t* v, int64_t layer_stride, int64_t block_stride, int32_t num_layers,
                     int32_t h, int32_t head_dim, int32_t block_size, int32_t* block_table, int32_t table_stride,
                     int32_t num_seqs, int32_t* seq_len, const uint8_t* active, int32_t* refcount, int32_t num_blocks,
                     int32_t* free_list, int64_t* free_count, const uint16_t* new_k, const uint16_t* new_v) {
  int64_t need = 0;
  for (int32_t s = 0; s < num_seqs; ++s) {
    if (active && !active[s]) continue;
    const int32_t pos = seq_len[s];
    if (pos < 0) return OR_INVALID;
    const int32_t lb = pos / block_size, off = pos % block_size;
    if (lb >= table_stride) return OR_CAPACITY;
    if (off == 0) {
      ++need;
    } else {
      const int32_t b = block_table[(int64_t)s * table_stride + lb];
      if (b < 0 || b >= num_blocks || refcount[b] != 1) return OR_CORRUPTION;
    }
  }
  if (need > *free_count) return OR_CAPACITY;
  for (int64_t r = 0; r < need; ++r) {
    const int32_t b = free_list[*free_count - 1 - r];
    if (b < 0 || b >= num_blocks || refcount[b] != 0) return OR_CORRUPTION;
  }
  const int64_t row = (int64_t)h * head_dim;
  for (int32_t s = 0; s < num_seqs; ++s) {
    if (active && !active[s]) continue;
    const int32_t pos = seq_len[s];
    const int32_t lb = pos / block_size, off = pos % block_size;
    int32_t b;
    if (off == 0) {
      *free_count -= 1;
      b = free_list[*free_count];
      refcount[b] = 1;
      block_table[(int64_t)s * table_stride + lb] = b;
    } else {
      b = block_table[(int64_t)s * table_stride + lb];
    }
    for (int32_t l = 0; l < num_layers; ++l) {
      const int64_t dst = (int64_t)l * layer_stride + (int64_t)b * block_stride + (int64_t)off * row;
      const int64_t src = ((int64_t)l * num_seqs + s) * row;
      for (int64_t e = 0; e < row; ++e) {
        k[dst + e] = new_k[src + e];
        v[dst + e] = new_v[src + e];
      }
    }
    seq_len[s] = pos + 1;
  }
  return OR_OK;
}

/* Decode attention of one layer through the block table (reading R36): for sequence s and query
 * head qh (KV head g = qh / (hq / h), GQA),
 *   score_j = scale * <q[s][qh], K_l[table[s][j / d]][j % d][g]>,  j < seq_len[s]
 *   out[s][qh] = sum_j softmax(score)_j * V_l[table[s][j / d]][j % d][g]
 * in fp64 (q is bf16, as the kernel reads it). seq_len[s] == 0 gives a zero output. */
int oracle_paged_attention(const uint16_t* k, const uint16_t* v, int64_t layer_stride, int64_t block_stride,
                           int32_t layer, int32_t h, int32_t head_dim, int32_t block_size, const uint16_t* q,
                           int32_t num_q_heads, const int32_t* block_table, int32_t table_stride,
                           const int32_t* seq_len, int32_t num_seqs, double scale, double* out) {
  if (h < 1 || num_q_heads < h || num_q_heads % h != 0) return OR_INVALID;
  const int32_t G = num_q_heads / h;
  for (int32_t s = 0; s < num_seqs; ++s) {
    const int32_t n = seq_len[s];
    double* sc = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int32_t qh = 0; qh < num_q_heads; ++qh) {
      const int32_t g = qh / G;
      const uint16_t* qv = q + ((int64_t)s * num_q_heads + qh) * head_dim;
      double* o = out + ((int64_t)s * num_q_heads + qh) * head_dim;
      for (int32_t x = 0; x < head_dim; ++x) o[x] = 0.0;
      if (n == 0) continue;
      double mx = -INFINITY;
      for (int32_t j = 0; j < n; ++j) {
        const int32_t b = block_table[(int64_t)s * table_stride + j / block_size];
        const uint16_t* kr = k + (int64_t)layer * layer_stride + (int64_t)b * block_stride +
                             ((int64_t)(j % block_size) * h + g) * head_dim;
        double dot = 0.0;
        for (int32_t x = 0; x < head_dim; ++x) dot += bf16_to_double(qv[x]) * bf16_to_double(kr[x]);
        sc[j] = scale * dot;
        if (sc[j] > mx) mx = sc[j];
      }
      double z = 0.0;
      for (int32_t j = 0; j < n; ++j) {
        sc[j] = exp(sc[j] - mx);
        z += sc[j];
      }
      for (int32_t j = 0; j < n; ++j) {
        const int32_t b = block_table[(int64_t)s * table_stride + j / block_size];
        const uint16_t* vr = v + (int64_t)layer * layer_stride + (int64_t)b * block_stride +
                             ((int64_t)(j % block_size) * h + g) * head_dim;
        const double p = sc[j] / z;
        for (int32_t x = 0; x < head_dim; ++x) o[x] += p * bf16_to_double(vr[x]);
      }
    }
    free(sc);
  }
  return OR_OK;
}

/* Block-budget admission (reading R37; the mechanism behind PAPER.md Fig. 6: blocks freed by
 * sharing admit more concurrent sequences). Waiting requests are taken first-come-first-served;
 * request i needs ceil((prompt_len[i] + reserve) / d) blocks; it is admitted while the need fits
 * in the free blocks left, and admission stops at the first request that does not fit (no
 * skipping ahead). Returns the number admitted; blocks_used receives their total need. */
int32_t oracle_admit(const int32_t* prompt_len, int32_t num_waiting, int32_t reserve, int32_t block_size,
                     int64_t free_blocks, int64_t* blocks_used) {
  int64_t used = 0;
  int32_t i = 0;
  for (; i < num_waiting; ++i) {
    const int64_t need = ((int64_t)prompt_len[i] + reserve + block_size - 1) / block_size;
    if (used + need > free_blocks) break;
    used += need;
  }
  *blocks_used = used;
  return i;
}
