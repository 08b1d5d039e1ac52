/*
 * tinyserve.h — C ABI of libtinyserve.so, the B200 (sm_100a) decode-time hot path of
 * TinyServe (arXiv 2509.12211, §3.5 "Query-Aware Page Selection", Alg. 1).
 *
 * One decode step of one attention layer, for a batch of sequences held in a paged KV
 * cache (vLLM-style block table):
 *
 *   ts_meta_append        metadata maintenance on KV append      Eq. 1
 *   ts_score_pages        bounding-box relevance of every page   Eq. 2; Alg. 1 Step 1
 *   ts_select_topk        top-K pages per (sequence, kv head)    PAPER.md:162-167; Alg. 1 Step 2
 *   ts_sparse_decode_attn softmax attention over selected pages  PAPER.md:169-172; Alg. 1 Steps 3-4
 *   ts_decode_step        score -> select -> attend in one call  Alg. 1, PAPER.md:209-249 ("single pass")
 *   ts_decode_step_append append the new token, then the step     Eq. 1 + Alg. 1 (one launch, bf16)
 *   ts_decode_step_prefetch the step + L2 prefetch of the previous selection
 *   ts_select_candidates  score + local top-k of a sequence shard (one launch)
 *   ts_shard_attend       candidate merge + partial attention of a shard (one launch)
 *   ts_lse_merge          merge of partial attentions (split-K / multi-GPU)
 *   ts_kv_quantize        bf16 rows -> FP8 E4M3 codes + row exponents (NEXT-3, reading R21)
 *
 * Conventions (apply to every entry point):
 *  - POINTERS: every tensor argument is a DEVICE pointer (cudaMalloc'd or torch CUDA
 *    storage) owned by the caller, except `ts_layout*`, which is a HOST pointer read
 *    during the call only.  The library never allocates, frees, synchronises or keeps a
 *    pointer after returning.  `stream` is a cudaStream_t passed as void* (NULL = the
 *    legacy default stream); all work is enqueued asynchronously on it.
 *  - LAYOUT, all row-major, contiguous:
 *      q          [batch][num_q_heads][head_dim]             kv_dtype
 *      k_pool     [num_blocks][num_kv_heads][page_size][head_dim]   kv_dtype
 *      v_pool     [num_blocks][num_kv_heads][page_size][head_dim]   kv_dtype
 *      meta       [batch][num_kv_heads][max_pages][2][head_dim]   kv_dtype, LOGICAL page
 *                 order: [b][g][jl][0][:] = m (min), [..][1][:] = M (max) of the valid keys
 *                 of local page jl of sequence b, kv head g (Eq. 1).  Row (b, g) is one
 *                 contiguous run, so scoring streams it with no page-table lookup.
 *      page_table [batch][max_pages] int32: LOCAL page index -> physical block
 *      seq_lens   [batch] int32: GLOBAL number of tokens in the cache (before the append
 *                 for ts_meta_append, after it for everything else)
 *      scores     [batch][num_kv_heads][max_pages] fp32, indexed by LOCAL page
 *      o          [batch][num_q_heads][head_dim] fp32;  lse [batch][num_q_heads] fp32
 *    q head h belongs to kv head h / (num_q_heads / num_kv_heads) (GQA, reading R16).
 *  - SEQUENCE SHARDING: a rank owns global pages j with
 *    j % shard_stride == shard_offset and stores global page j at local index
 *    j / shard_stride.  Unsharded: shard_stride = 1, shard_offset = 0.  Page ids that
 *    cross the boundary (sel_ids) are always GLOBAL.
 *  - PRECISION: q, K, V and meta share kv_dtype (bf16 or fp32; for TS_FP8E4M3 K and V are
 *    E4M3 codes with row exponents and q / meta are bf16); scores, o and lse are fp32
 *    (reading R10).  K_b = min(P_b, max(1, floor(budget_tokens / page_size))).
 *  - ERRORS: host-side validation only (no device synchronisation):
 *      TS_ERR_CONFIG       non-positive size, budget < 1, unknown dtype
 *      TS_ERR_SHAPE        num_q_heads % num_kv_heads != 0, k < 1, bad shard
 *      TS_ERR_ALIGN        a tensor pointer not 16-byte aligned (128-bit loads / TMA)
 *      TS_ERR_UNSUPPORTED  head_dim / page_size / group size outside the compiled set
 *      TS_ERR_WORKSPACE    ws NULL or smaller than ts_workspace_bytes()
 *      TS_ERR_CUDA         a CUDA launch failed (cudaGetLastError)
 *    Data-dependent faults (page_table entry >= num_blocks, seq_len > max_pages*page_size,
 *    non-finite inputs) are undefined behaviour, not detected.
 *    seq_len == 0 is valid: the sequence selects nothing, o = 0, lse = -inf (reading R8).
 *  - Compiled set: head_dim 64 or 128 for metadata, scoring and fp32 attention; the bf16
 *    attention (ts_sparse_decode_attn, ts_decode_step) needs head_dim 64, page_size in
 *    {4, 8, 16, 32, 64} and group size 1..8 (tensor-core tiles); fp32 takes any page_size
 *    and group size.  At most 4096 selected pages per row.
 */
#ifndef TINYSERVE_H
#define TINYSERVE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TS_OK = 0,
    TS_ERR_CONFIG = 1,
    TS_ERR_SHAPE = 2,
    TS_ERR_ALIGN = 3,
    TS_ERR_UNSUPPORTED = 4,
    TS_ERR_CUDA = 5,
    TS_ERR_WORKSPACE = 6
} ts_status;

/* KV storage type.  TS_FP8E4M3 ("FP16/INT8 KV formats" PAPER.md:94,
 * reading R21): each stored row (one token, one kv head) is 64 OCP FP8 E4M3 codes plus one
 * int8 exponent e (value = code * 2^e, e in [-64, 64] the smallest with max |x| <= 448 * 2^e).
 * k_pool / v_pool are sequences of 1040-byte SUB-PAGE RECORDS, one per 16 consecutive rows of
 * [num_blocks][Hkv][S] (S a multiple of 16): the 16 rows' codes [16][64], then their 16
 * exponent bytes — so row r's codes are at (r/16)*1040 + (r%16)*64 and its exponent at
 * (r/16)*1040 + 1024 + r%16; num_blocks*Hkv*S*65 bytes (ts_pool_bytes).  q, meta, k_new and
 * v_new stay bf16, and the
 * metadata is the exact min / max of the DEQUANTISED keys.  head_dim 64 only; attention
 * over an FP8 cache (ts_decode_step(_append / _prefetch), ts_sparse_decode_attn,
 * ts_dense_decode_attn, ts_shard_attend) needs page_size a multiple of 16 and G <= 8. */
typedef enum { TS_F32 = 0, TS_BF16 = 1, TS_FP8E4M3 = 2 } ts_dtype;

typedef struct {
    int32_t batch;          /* B: sequences in the batch                                   */
    int32_t num_q_heads;    /* Hq                                                          */
    int32_t num_kv_heads;   /* Hkv, Hq % Hkv == 0, group size G = Hq / Hkv                  */
    int32_t head_dim;       /* d                                            */
    int32_t page_size;      /* S tokens per page                             */
    int32_t max_pages;      /* row stride of page_table and scores (local pages);          *
                             * max_pages * page_size <= 2^26 tokens (else TS_ERR_UNSUPPORTED) */
    int32_t num_blocks;     /* physical blocks in k_pool / v_pool / meta                   */
    int32_t shard_stride;   /* 1 unsharded; G ranks for block-cyclic sequence sharding     */
    int32_t shard_offset;   /* this rank's residue, 0 <= shard_offset < shard_stride       */
    int32_t kv_dtype;       /* ts_dtype of q, k_pool, v_pool and meta                      */
} ts_layout;

/* Metadata maintenance on KV append ("lightweight metadata — channel-wise
 * min and max values of stored Key vectors — is maintained"; Eq. 1).
 * For each sequence b with t = seq_lens[b] (length BEFORE the append): global page
 * j = t / S, slot = t % S.  If this rank owns j: writes k_new[b] / v_new[b]
 * ([B][Hkv][d], kv_dtype) into slot `slot` of block page_table[b][j / shard_stride] and
 * sets, per kv head, in meta[b][g][j / shard_stride]
 *   m = slot == 0 ? k : min(m, k),   M = slot == 0 ? k : max(M, k)   (exact, no rounding).
 * If `advance` != 0 the kernel then sets seq_lens[b] = t + 1 (every rank advances its copy
 * of the global length, owner or not); otherwise seq_lens is left unchanged. */
ts_status ts_meta_append(const ts_layout *layout, const void *k_new, const void *v_new,
                         int32_t *seq_lens, int32_t advance, const int32_t *page_table,
                         void *k_pool, void *v_pool, void *meta, void *stream);

/* Bulk metadata (SPEC.md:65-73 recompute_metadata; prefill / cache import): for every
 * owned page j < P_b of every sequence, meta[b][g][j / shard_stride] = min / max over the
 * page's valid keys (tokens t < seq_lens[b]).  Entries of pages >= P_b are not touched. */
ts_status ts_meta_build(const ts_layout *layout, const void *k_pool, const int32_t *page_table,
                        const int32_t *seq_lens, void *meta, void *stream);

/* Page scoring (Eq. 2; Alg. 1 Step 1).  For every sequence b, kv head g
 * and owned local page jl (global j = jl*stride + offset < P_b = ceil(seq_lens[b]/S)):
 *   scores[b][g][jl] = max_{h in group(g)} sum_i max(q[b][h][i]*m_i, q[b][h][i]*M_i)
 * (= Eq. 2 per head; GQA max over the group, reading R9), accumulated in fp32.  Entries
 * for non-existent pages are -inf.  A page's score depends only on (q, its meta): the same
 * bits whatever the sharding.  -0.0 is written as +0.0. */
ts_status ts_score_pages(const ts_layout *layout, const void *q, const void *meta,
                         const int32_t *page_table, const int32_t *seq_lens, float *scores,
                         void *stream);

/* Top-K selection (Alg. 1 Step 2 "radix select").
 * scores [rows][stride] fp32.  Row r's candidates are the entries i < row_len[r]
 * (row_len NULL: all `stride`) whose score is not -inf.  The id of entry i is
 * ids_in[r][i] if ids_in != NULL, else i*id_stride + id_offset.  Selects
 * kk = min(k, #candidates) entries with the largest scores; equal scores go to the lower
 * id (reading R6).  Outputs: sel_ids [rows][k] int32, the kk ids ascending then -1
 * padding; sel_scores [rows][k] fp32 (nullable), aligned with sel_ids, -inf padding;
 * sel_count [rows] int32 = kk.  Deterministic; exact (integer key comparisons). */
ts_status ts_select_topk(const float *scores, int32_t rows, int32_t stride, const int32_t *row_len,
                         const int32_t *ids_in, int32_t id_stride, int32_t id_offset, int32_t k,
                         int32_t *sel_ids, float *sel_scores, int32_t *sel_count, void *stream);

/* Sparse attention (SparseAttn PAPER.md:169-172; Alg. 1 Steps 3-4).
 * For q head h of sequence b (kv head g = h / G): over the valid tokens (t < seq_lens[b],
 * reading R7) of the OWNED pages among sel_ids[b][g][0 .. sel_count[b][g]) (global ids,
 * [B][Hkv][sel_stride]), a_t = scale * q.k_t, o = softmax(a) . V, lse = ln sum exp(a_t),
 * fp32.  No attended token: o = 0, lse = -inf.  lse may be NULL.  Split-K over CTAs with an
 * in-kernel log-sum-exp merge; ws (>= ts_attn_workspace_bytes, zero-filled once before
 * first use; the library leaves it reusable) holds the partials. */
ts_status ts_sparse_decode_attn(const ts_layout *layout, const void *q, const void *k_pool,
                                const void *v_pool, const int32_t *page_table,
                                const int32_t *seq_lens, const int32_t *sel_ids,
                                const int32_t *sel_count, int32_t sel_stride, float scale,
                                float *o, float *lse, void *ws, size_t ws_bytes, void *stream);

/* The fused decode step (Alg. 1 end to end): score every page from
 * meta, select K_b = min(P_b, max(1, floor(budget_tokens/S))) pages per (b, g), attend.
 * bf16 with page_size a multiple of 16: one launch (a thread-block cluster per (b, g):
 * score -> exact top-K in the cluster leader -> TMA gather -> attention, PDL-launched so
 * that its prologue overlaps the previous kernel); bf16 with page_size 8: score/select
 * kernel -> attention kernel (PDL); fp32: score -> select -> attention kernels.
 * Unsharded layouts only (shard_stride == 1; the sequence-sharded step is composed from
 * the calls above plus two all-gathers).  sel_ids_out [B][Hkv][Kmax] and
 * sel_count_out [B][Hkv] (Kmax = min(max_pages, max(1, budget_tokens/S))) may be NULL.
 * ws >= ts_workspace_bytes(layout, budget_tokens), zero-filled once before first use. */
ts_status ts_decode_step(const ts_layout *layout, const void *q, const void *k_pool,
                         const void *v_pool, const void *meta, const int32_t *page_table,
                         const int32_t *seq_lens, int32_t budget_tokens, float scale, float *o,
                         float *lse, int32_t *sel_ids_out, int32_t *sel_count_out, void *ws,
                         size_t ws_bytes, void *stream);

/* ts_decode_step_append — one decode step of a serving loop: append the newest token, then
 * Alg. 1.  For every sequence b with seq_lens[b] = t + 1 > 0 (seq_lens
 * ALREADY counts the new token), k_new[b] / v_new[b] ([batch][num_kv_heads][head_dim],
 * kv_dtype, device) are written to slot t % page_size of the block holding logical page
 * t / page_size, the (m, M) record of that page is updated as ts_meta_append does (Eq. 1,
 * PAPER.md:177-178; m = M = k for the first key of a page), and then the step runs exactly
 * as ts_decode_step with the same arguments — in ONE launch for the bf16 and FP8 cluster path (the
 * page's scorer patches its staged record and persists it; the K/V row is published to the
 * attention phase by the cluster barrier; FP8: the row is quantised as ts_kv_quantize and the
 * record updated with the dequantised key).  Other layouts fall back to ts_meta_append's
 * kernel followed by ts_decode_step.  k_pool, v_pool and meta are modified in place; the
 * results equal ts_meta_append(seq_lens - 1) followed by ts_decode_step bit for bit in the
 * metadata and the page sets.  Unsharded layouts only (TS_ERR_UNSUPPORTED otherwise). */
ts_status ts_decode_step_append(const ts_layout *layout, const void *q, const void *k_new,
                                const void *v_new, void *k_pool, void *v_pool, void *meta,
                                const int32_t *page_table, const int32_t *seq_lens,
                                int32_t budget_tokens, float scale, float *o, float *lse,
                                int32_t *sel_ids, int32_t *sel_count, void *ws, size_t ws_bytes,
                                void *stream);

/* ts_decode_step_prefetch — ts_decode_step with cross-step page reuse (
 * PAPER.md:203 "prefetching selected pages", the reuse fraction rho of the load model
 * PAPER.md:263-271, the KV-reuse study PAPER.md:623).  On entry sel_ids [B][Hkv][Kmax] and
 * sel_count [B][Hkv] (device, required) hold the PREVIOUS step's selection of the same
 * cache (as this call writes it; any content is safe: entries outside [0, P_b) are
 * ignored).  While it scores the pages, the step prefetches the K and V blocks of those
 * pages into L2, so the HBM keeps streaming through the top-K and the gather of pages
 * selected again hits L2.  Results are identical to ts_decode_step (the prefetch is a
 * hint); on return sel_ids / sel_count hold this step's selection.  The bf16 one-launch path
 * (page_size a multiple of 16) prefetches; other layouts run ts_decode_step unchanged. */
ts_status ts_decode_step_prefetch(const ts_layout *layout, const void *q, const void *k_pool,
                                  const void *v_pool, const void *meta, const int32_t *page_table,
                                  const int32_t *seq_lens, int32_t budget_tokens, float scale,
                                  float *o, float *lse, int32_t *sel_ids, int32_t *sel_count,
                                  void *ws, size_t ws_bytes, void *stream);

/* Candidate merge — the exchange step of sequence sharding: the global
 * top-k over the union of per-rank candidate lists.  Part p (< parts) of row r holds k_part
 * entries at cand_scores[p*part_stride + r*k_part + e] with global page ids at the same
 * offsets of cand_ids (e.g. the rank-major output of an all-gather of every rank's
 * ts_select_topk result; part_stride 0 = rows*k_part, i.e. [parts][rows][k_part]).
 * -inf entries are ignored.  Output exactly as ts_select_topk (ids ascending, ties to
 * the lower id).  Because a page's score bits do not depend on sharding and every global
 * top-k page is in its owner's local top-k, the result equals the unsharded selection. */
ts_status ts_select_merge(const float *cand_scores, const int32_t *cand_ids, int32_t parts,
                          int64_t part_stride, int32_t rows, int32_t k_part, int32_t k,
                          int32_t *sel_ids, float *sel_scores, int32_t *sel_count, void *stream);

/* Sequence sharding, fused (the north star's "each GPU scores its pages and
 * keeps a local top-k of candidates ... computes partial (o, m, l) on its own selected
 * pages"): the two halves of one rank's step, one launch each, around the two exchanges.
 *
 * ts_select_candidates — ts_score_pages + ts_select_topk in one launch: for every row
 * (b, g), the k owned pages with the largest scores (Eq. 2, reading R9), ties to the lower
 * id, as GLOBAL ids ascending in cand_ids [rows][k] (-1 padding) with their fp32 scores in
 * cand_scores [rows][k] (-inf padding) and the count in cand_count [rows].  Equals
 * ts_score_pages followed by ts_select_topk(id_stride = shard_stride, id_offset =
 * shard_offset).  bf16 q / metadata (bf16 or FP8 caches), head_dim 64, G <= 8, k <= 4096;
 * TS_ERR_UNSUPPORTED otherwise (compose the two calls instead). */
ts_status ts_select_candidates(const ts_layout *layout, const void *q, const void *meta,
                               const int32_t *page_table, const int32_t *seq_lens, int32_t k,
                               float *cand_scores, int32_t *cand_ids, int32_t *cand_count,
                               void *stream);

/* ts_shard_attend — ts_select_merge + ts_sparse_decode_attn in one launch: the global top-k
 * over `parts` candidate lists (part p of row r: k entries at p*part_stride + r*k of
 * cand_scores / cand_ids, e.g. the all-gathered ts_select_candidates outputs; part_stride 0
 * = rows*k; -inf entries ignored; ties to the lower global id), then the partial attention
 * over the OWNED selected pages exactly as ts_sparse_decode_attn: o [B][Hq][d], lse [B][Hq]
 * (o = 0, lse = -inf for a row with no owned selected page).  The selection itself is
 * written to sel_ids_out [rows][k] / sel_count_out [rows] when non-NULL (identical on every
 * rank).  bf16 or FP8 K/V, head_dim 64, page_size a multiple of 16, G <= 8, parts*k <= 4096;
 * ws >= ts_attn_workspace_bytes(layout, k), zero-filled once; TS_ERR_UNSUPPORTED otherwise. */
ts_status ts_shard_attend(const ts_layout *layout, const void *q, const void *k_pool,
                          const void *v_pool, const int32_t *page_table, const int32_t *seq_lens,
                          const float *cand_scores, const int32_t *cand_ids, int32_t parts,
                          int64_t part_stride, int32_t k, float scale, float *o, float *lse,
                          int32_t *sel_ids_out, int32_t *sel_count_out, void *ws, size_t ws_bytes,
                          void *stream);

/* Log-sum-exp merge of `parts` partial attentions over disjoint token sets.  Part p of
 * o_parts starts at p*part_stride and holds [rows][d]; part p of lse_parts starts at
 * p*part_stride and holds [rows] (part_stride 0: dense, rows*d and rows respectively):
 *   lse = ln sum_p exp(lse_p),   o = sum_p exp(lse_p - lse) * o_p.
 * Parts with lse = -inf contribute nothing; all -inf gives o = 0, lse = -inf. */
ts_status ts_lse_merge(int32_t parts, int32_t rows, int32_t d, const float *o_parts,
                       const float *lse_parts, int64_t part_stride, float *o, float *lse,
                       void *stream);

/* FullCache baseline (dense attention): for every
 * q head h of sequence b, softmax attention over ALL valid tokens t < seq_lens[b] of the
 * sequence's pages, through the same paged pool and attention kernel as the sparse path
 * (bf16, head_dim 64, page_size a multiple of 16, unsharded).  Equals
 * ts_sparse_decode_attn with every page selected.  ws >= ts_dense_workspace_bytes(),
 * zero-filled once before first use.  Used to measure the sparse/dense speedup. */
ts_status ts_dense_decode_attn(const ts_layout *layout, const void *q, const void *k_pool,
                               const void *v_pool, const int32_t *page_table,
                               const int32_t *seq_lens, float scale, float *o, float *lse,
                               void *ws, size_t ws_bytes, void *stream);
size_t ts_dense_workspace_bytes(const ts_layout *layout);

/* FP8 KV quantisation (reading R21; ts_dtype TS_FP8E4M3): rows x 64 bf16 values at src
 * (device, 16-byte aligned; e.g. a bf16 pool [num_blocks][Hkv][S][64]) -> the FP8 pool format
 * above at pool (device, 16-byte aligned, rows*65 bytes): per row e = smallest integer in
 * [-64, 64] with max |x| <= 448 * 2^e, code = E4M3 nearest to x * 2^-e (round to nearest
 * even, saturating).  Used for prefill / cache import; decode-time appends quantise inside
 * ts_meta_append / ts_decode_step_append.  TS_ERR_SHAPE unless rows % 16 == 0;
 * TS_ERR_UNSUPPORTED unless head_dim == 64. */
ts_status ts_kv_quantize(int64_t rows, int32_t head_dim, const void *src, void *pool, void *stream);

/* Bytes of one K (or V) pool for the layout: num_blocks*Hkv*S*d*elem, or *65 for FP8
 * (codes + exponents).  Host-only; 0 for an invalid layout. */
size_t ts_pool_bytes(const ts_layout *layout);

/* Workspace sizes in bytes (host-only, no CUDA call). */
size_t ts_workspace_bytes(const ts_layout *layout, int32_t budget_tokens);
size_t ts_attn_workspace_bytes(const ts_layout *layout, int32_t sel_stride);

/* Static strings (host-only). */
const char *ts_status_str(ts_status status);
const char *ts_version(void);

/* Number of kernel launches the last successful host call on this thread enqueued
 * (bench.py's gpu_launches accounting; host-only). */
int32_t ts_last_launch_count(void);

/* Measurement hook (bench.py roofline): while set, ts_decode_step on this thread records
 * events[0..3] (cudaEvent_t, created by the caller; NULL entries skipped) on its stream
 * before the first kernel, after scoring, after selection and after attention, as external
 * records (valid inside CUDA-graph capture).  The bf16 path (S a multiple of 16) is ONE
 * kernel (score + select + gather + attend) and records only events[0] and events[3].
 * events == NULL or n == 0 clears it.  Host-only. */
void ts_profile_events(void *const *events, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* TINYSERVE_H */
