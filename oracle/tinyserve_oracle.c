/*
 * tinyserve_oracle.c — float64 CPU oracle for the TinyServe decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2509_12211_b200/) never imports, links or executes it, and the two share no
 * source, header, table or helper.
 *
 * It is a plain, slow, step-by-step transcription of PAPER.md §3.5 ("Query-Aware Page
 * Selection") in double precision, following the paper's order and
 * notation.  Readings where the paper is silent are the R-numbered entries of DESIGN.md §2
 * (same numbering as SURVEY.md §8c G1-G20).
 *
 *   step 1  pages:    P = ceil(t / S)
 *   step 2  metadata: phi_j = (m_j, M_j), channel-wise min / max of keys  PAPER.md:129, Eq. 1 (177-178)
 *   step 3  score:    r = sum_i (q_i >= 0 ? q_i M_ji : q_i m_ji)          Eq. 2 (179-185), Alg. 1 Step 1 (217-224)
 *                     GQA: s = max over the group's q heads of r        reading R9
 *   step 4  select:   S_t = TopK_j s_j, |S_t| = K                        PAPER.md:162-167, Alg. 1 Step 2 (227-228)
 *                     ties -> lower page id, ids ascending             reading R6
 *   step 5  attend:   softmax(scale * q.k) v over the selected pages    SparseAttn PAPER.md:169-172, Alg. 1 Steps 3-4
 *                     stable softmax (max subtracted)                  reading R11
 *
 * Inputs are the raw bf16 / fp32 bytes of the paged cache; every element is widened
 * exactly to double.  All arithmetic is double; summations run in ascending index order.
 * OpenMP parallelises over (sequence, kv-head) rows only; each row is computed by one
 * thread in a fixed order, so results do not depend on the thread count.
 *
 * Pins: tests/test_oracle_pins.py (golden examples from SPEC.md, closed forms,
 * brute force, torch SDPA float64 for the dense special case).  Parity unpinned: none of
 * the functions below (each has at least one pin); the paper itself prints no worked
 * example (DESIGN.md §2 "What pins what").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- layout description (oracle-private; the CUDA header is NOT included) --------- */
typedef struct {
    int32_t batch, num_q_heads, num_kv_heads;
    int32_t head_dim, page_size;
    int32_t max_pages, num_blocks;
    int32_t dtype;            /* 0 = fp32, 1 = bf16 */
} or_layout;

/* Exact widening of one stored element to double. */
static double widen(const void *base, int dtype, size_t idx) {
    if (dtype == 1) {
        uint16_t h = ((const uint16_t *)base)[idx];
        uint32_t u = (uint32_t)h << 16;   /* bf16 is the top half of an fp32 */
        float f;
        memcpy(&f, &u, 4);
        return (double)f;
    }
    return (double)((const float *)base)[idx];
}

/* element index into a pool [num_blocks][Hkv][S][d] */
static size_t pool_idx(const or_layout *L, int blk, int h, int slot, int i) {
    return (((size_t)blk * L->num_kv_heads + h) * L->page_size + slot) * L->head_dim + i;
}

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Step 1: number of pages of a sequence of t tokens. */
static int num_pages(int t, int S) { return (t + S - 1) / S; }

/* ------------------------------------------------------------------------------------
 * Step 2 — page metadata, batch form (Eq. 1).
 * Output in LOGICAL layout: mmin/mmax [B][Hkv][max_pages][d]; pages j >= P_b untouched.
 * Only valid tokens t < seq_len contribute (reading R7).
 * ---------------------------------------------------------------------------------- */
int or_meta_build(const or_layout *L, const void *k_pool, const int32_t *page_table,
                  const int32_t *seq_lens, double *mmin, double *mmax, int threads) {
    const int B = L->batch, H = L->num_kv_heads, d = L->head_dim, S = L->page_size;
    set_threads(threads);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int b = 0; b < B; ++b)
        for (int g = 0; g < H; ++g) {
            const int t = seq_lens[b];
            const int P = num_pages(t, S);
            for (int j = 0; j < P; ++j) {
                const int blk = page_table[(size_t)b * L->max_pages + j];
                const int n = (t - j * S < S) ? (t - j * S) : S;
                double *mn = mmin + (((size_t)b * H + g) * L->max_pages + j) * d;
                double *mx = mmax + (((size_t)b * H + g) * L->max_pages + j) * d;
                for (int i = 0; i < d; ++i) {
                    double lo = widen(k_pool, L->dtype, pool_idx(L, blk, g, 0, i));
                    double hi = lo;
                    for (int s = 1; s < n; ++s) {
                        double x = widen(k_pool, L->dtype, pool_idx(L, blk, g, s, i));
                        if (x < lo) lo = x;
                        if (x > hi) hi = x;
                    }
                    mn[i] = lo;
                    mx[i] = hi;
                }
            }
        }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Step 2, incremental form — one append: the new key of sequence b goes
 * to slot (t mod S) of page floor(t/S); for the first key of a page m = M = k, else
 * m <- min(m, k), M <- max(M, k).  Operates on LOGICAL double metadata; also writes the
 * raw key/value bytes into the pools (a byte copy, no arithmetic).
 * ---------------------------------------------------------------------------------- */
int or_meta_append(const or_layout *L, const void *k_new, const void *v_new,
                   const int32_t *seq_lens_before, const int32_t *page_table,
                   void *k_pool, void *v_pool, double *mmin, double *mmax) {
    const int B = L->batch, H = L->num_kv_heads, d = L->head_dim, S = L->page_size;
    const size_t es = (L->dtype == 1) ? 2 : 4;
    for (int b = 0; b < B; ++b) {
        const int t = seq_lens_before[b];
        const int j = t / S, slot = t % S;
        if (j >= L->max_pages) return 2; /* shape error: no page for this token */
        const int blk = page_table[(size_t)b * L->max_pages + j];
        for (int g = 0; g < H; ++g) {
            const size_t src = ((size_t)b * H + g) * d;
            memcpy((char *)k_pool + pool_idx(L, blk, g, slot, 0) * es, (const char *)k_new + src * es, d * es);
            memcpy((char *)v_pool + pool_idx(L, blk, g, slot, 0) * es, (const char *)v_new + src * es, d * es);
            double *mn = mmin + (((size_t)b * H + g) * L->max_pages + j) * d;
            double *mx = mmax + (((size_t)b * H + g) * L->max_pages + j) * d;
            for (int i = 0; i < d; ++i) {
                const double k = widen(k_new, L->dtype, src + i);
                if (slot == 0) {
                    mn[i] = k;
                    mx[i] = k;
                } else {
                    if (k < mn[i]) mn[i] = k;
                    if (k > mx[i]) mx[i] = k;
                }
            }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Step 3 — relevance score (Eq. 2; Alg. 1 Step 1):
 *     r(q, phi_j) = sum_{i=1..d} ( q_i >= 0 ? q_i * M_ji : q_i * m_ji )
 * summed in ascending i.  GQA (reading R9): the kv-head g is shared by the q heads
 * h = g*G .. g*G+G-1 (reading R16); the group score is the max of their r.
 * scores [B][Hkv][max_pages]; -inf for j >= P_b (reading R7/R8).
 * ---------------------------------------------------------------------------------- */
double or_relevance(const double *q, const double *m, const double *M, int d) {
    double r = 0.0;
    for (int i = 0; i < d; ++i) r += (q[i] >= 0.0) ? q[i] * M[i] : q[i] * m[i];
    return r;
}

int or_score_pages(const or_layout *L, const void *q, const double *mmin, const double *mmax,
                   const int32_t *seq_lens, double *scores, int threads) {
    const int B = L->batch, H = L->num_kv_heads, d = L->head_dim, S = L->page_size;
    const int G = L->num_q_heads / L->num_kv_heads;
    set_threads(threads);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int b = 0; b < B; ++b)
        for (int g = 0; g < H; ++g) {
            double qd[8 * 256];   /* G * d doubles, G*d <= 2048 */
            for (int hh = 0; hh < G; ++hh)
                for (int i = 0; i < d; ++i)
                    qd[hh * d + i] = widen(q, L->dtype, ((size_t)b * L->num_q_heads + g * G + hh) * d + i);
            const int P = num_pages(seq_lens[b], S);
            double *row = scores + ((size_t)b * H + g) * L->max_pages;
            for (int j = 0; j < L->max_pages; ++j) {
                if (j >= P) { row[j] = -INFINITY; continue; }
                const double *mn = mmin + (((size_t)b * H + g) * L->max_pages + j) * d;
                const double *mx = mmax + (((size_t)b * H + g) * L->max_pages + j) * d;
                double s = -INFINITY;
                for (int hh = 0; hh < G; ++hh) {
                    const double r = or_relevance(qd + hh * d, mn, mx, d);
                    if (r > s) s = r;
                }
                row[j] = s;
            }
        }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Step 4 — Top-K (Alg. 1 Step 2): per row, kk = min(k, n) entries with
 * the largest score; equal scores go to the lower id (reading R6); output ids
 * ascending.  Entries with score -inf are "no page" and never selected
 * (reading R8), so kk = min(k, #finite entries among the first row_len).  ids_in (nullable) gives each entry's id (candidate merge,
 * DESIGN.md §6); otherwise the id of entry i is i.  -0.0 and +0.0 compare equal.
 * Implemented as a full sort by (score desc, id asc) — a library sort, no selection trick.
 * ---------------------------------------------------------------------------------- */
typedef struct { double s; int32_t id; } or_cand;

static int cmp_score_desc_id_asc(const void *a, const void *b) {
    const or_cand *x = (const or_cand *)a, *y = (const or_cand *)b;
    if (x->s > y->s) return -1;
    if (x->s < y->s) return 1;
    return (x->id < y->id) ? -1 : (x->id > y->id);
}

static int cmp_id_asc(const void *a, const void *b) {
    const or_cand *x = (const or_cand *)a, *y = (const or_cand *)b;
    return (x->id < y->id) ? -1 : (x->id > y->id);
}

int or_select_topk(const double *scores, int rows, int stride, const int32_t *row_len,
                   const int32_t *ids_in, int k, int32_t *sel_ids, double *sel_scores,
                   int32_t *sel_count, int threads) {
    if (k < 1) return 1;
    set_threads(threads);
#pragma omp parallel for schedule(dynamic)
    for (int r = 0; r < rows; ++r) {
        const int len = row_len ? row_len[r] : stride;
        or_cand *c = (or_cand *)malloc(sizeof(or_cand) * (len > 0 ? len : 1));
        int n = 0;
        for (int i = 0; i < len; ++i) {
            const double s = scores[(size_t)r * stride + i];
            if (s == -INFINITY) continue;       /* -inf = "no page" (reading R8) */
            c[n].s = s + 0.0;                   /* -0.0 -> +0.0 (reading R6) */
            c[n].id = ids_in ? ids_in[(size_t)r * stride + i] : i;
            ++n;
        }
        const int kk = n < k ? n : k;
        qsort(c, n, sizeof(or_cand), cmp_score_desc_id_asc);
        qsort(c, kk, sizeof(or_cand), cmp_id_asc);
        for (int i = 0; i < k; ++i) {
            sel_ids[(size_t)r * k + i] = i < kk ? c[i].id : -1;
            if (sel_scores) sel_scores[(size_t)r * k + i] = i < kk ? c[i].s : -INFINITY;
        }
        sel_count[r] = kk;
        free(c);
    }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Step 5 — sparse attention (SparseAttn; Alg. 1 Steps 3-4, 231-244):
 * for q head h of group g = h / G, gather the valid tokens (t < seq_len, reading R7/R19)
 * of the selected pages in ascending page then slot order (Step 3, reading R18), then
 *     a_t = scale * q_h . k_t                 (Step 4 line 1; scale: reading R1)
 *     alpha = softmax(a)  (max-subtracted, reading R11)
 *     o_h = sum_t alpha_t v_t,   lse_h = max a + ln sum_t exp(a_t - max a)
 * No valid token (seq_len 0 or empty selection): o = 0, lse = -inf (reading R8).
 * sel_ids [B][Hkv][ksel] (global page ids), sel_count [B][Hkv].
 * o [B][Hq][d], lse [B][Hq] (nullable).
 * ---------------------------------------------------------------------------------- */
int or_sparse_attn(const or_layout *L, const void *q, const void *k_pool, const void *v_pool,
                   const int32_t *page_table, const int32_t *seq_lens, const int32_t *sel_ids,
                   const int32_t *sel_count, int ksel, double scale, double *o, double *lse,
                   int threads) {
    const int B = L->batch, Hq = L->num_q_heads, H = L->num_kv_heads, d = L->head_dim,
              S = L->page_size;
    const int G = Hq / H;
    set_threads(threads);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < Hq; ++h) {
            const int g = h / G;
            const int t_len = seq_lens[b];
            const int nsel = sel_count[(size_t)b * H + g];
            const int32_t *ids = sel_ids + ((size_t)b * H + g) * ksel;
            double qd[256];
            for (int i = 0; i < d; ++i) qd[i] = widen(q, L->dtype, ((size_t)b * Hq + h) * d + i);
            /* Step 3: gather (blk, slot) of the attended tokens */
            int ntok = 0;
            int *tb = (int *)malloc(sizeof(int) * ((size_t)nsel * S + 1));
            int *ts = (int *)malloc(sizeof(int) * ((size_t)nsel * S + 1));
            for (int u = 0; u < nsel; ++u) {
                const int j = ids[u];
                const int blk = page_table[(size_t)b * L->max_pages + j];
                for (int s = 0; s < S; ++s)
                    if (j * S + s < t_len) { tb[ntok] = blk; ts[ntok] = s; ++ntok; }
            }
            double *oh = o + ((size_t)b * Hq + h) * d;
            if (ntok == 0) {
                for (int i = 0; i < d; ++i) oh[i] = 0.0;
                if (lse) lse[(size_t)b * Hq + h] = -INFINITY;
                free(tb); free(ts);
                continue;
            }
            /* Step 4: a_t = scale q.k_t ; softmax ; o = sum alpha v */
            double *a = (double *)malloc(sizeof(double) * ntok);
            double amax = -INFINITY;
            for (int u = 0; u < ntok; ++u) {
                double dot = 0.0;
                for (int i = 0; i < d; ++i)
                    dot += qd[i] * widen(k_pool, L->dtype, pool_idx(L, tb[u], g, ts[u], i));
                a[u] = scale * dot;
                if (a[u] > amax) amax = a[u];
            }
            double l = 0.0;
            for (int u = 0; u < ntok; ++u) { a[u] = exp(a[u] - amax); l += a[u]; }
            for (int i = 0; i < d; ++i) oh[i] = 0.0;
            for (int u = 0; u < ntok; ++u) {
                const double alpha = a[u] / l;
                for (int i = 0; i < d; ++i)
                    oh[i] += alpha * widen(v_pool, L->dtype, pool_idx(L, tb[u], g, ts[u], i));
            }
            if (lse) lse[(size_t)b * Hq + h] = amax + log(l);
            free(a); free(tb); free(ts);
        }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Whole decode step (Alg. 1, in the paper's step order):
 * metadata (recomputed from K) -> scores -> top-K with K_b = min(P_b, max(1, budget/S))
 * (reading R4/R5) -> sparse attention.  sel_ids_out [B][Hkv][kmax], kmax = max(1, budget/S).
 * Workspace is allocated here (the oracle is not the product).
 * ---------------------------------------------------------------------------------- */
int or_decode_step(const or_layout *L, const void *q, const void *k_pool, const void *v_pool,
                   const int32_t *page_table, const int32_t *seq_lens, int budget_tokens,
                   double scale, double *o, double *lse, int32_t *sel_ids_out,
                   int32_t *sel_count_out, double *scores_out, int threads) {
    const int B = L->batch, H = L->num_kv_heads, d = L->head_dim, S = L->page_size;
    const int mp = L->max_pages;
    if (budget_tokens < 1 || S < 1 || d < 1) return 1;
    const int kmax = budget_tokens / S > 1 ? budget_tokens / S : 1;
    const size_t nmeta = (size_t)B * H * mp * d;
    double *mmin = (double *)calloc(nmeta ? nmeta : 1, sizeof(double));
    double *mmax = (double *)calloc(nmeta ? nmeta : 1, sizeof(double));
    double *sc = scores_out ? scores_out : (double *)malloc(sizeof(double) * (size_t)B * H * mp);
    int32_t *rl = (int32_t *)malloc(sizeof(int32_t) * (size_t)B * H);
    or_meta_build(L, k_pool, page_table, seq_lens, mmin, mmax, threads);
    or_score_pages(L, q, mmin, mmax, seq_lens, sc, threads);
    for (int b = 0; b < B; ++b)
        for (int g = 0; g < H; ++g) rl[b * H + g] = num_pages(seq_lens[b], S);
    or_select_topk(sc, B * H, mp, rl, NULL, kmax, sel_ids_out, NULL, sel_count_out, threads);
    or_sparse_attn(L, q, k_pool, v_pool, page_table, seq_lens, sel_ids_out, sel_count_out, kmax,
                   scale, o, lse, threads);
    free(mmin); free(mmax); free(rl);
    if (!scores_out) free(sc);
    return 0;
}

/* ------------------------------------------------------------------------------------
 * LSE merge of partial attentions over disjoint token sets (split-K / multi-GPU,
 * DESIGN.md §6; not in the paper).  With lse_p = m_p + ln l_p of part p:
 *     lse = ln sum_p exp(lse_p),  o = sum_p exp(lse_p - lse) o_p.
 * Parts with lse = -inf contribute nothing; all -inf -> o = 0, lse = -inf.
 * o_parts [parts][rows][d], lse_parts [parts][rows].
 * ---------------------------------------------------------------------------------- */
int or_lse_merge(int parts, int rows, int d, const double *o_parts, const double *lse_parts,
                 double *o, double *lse) {
    for (int r = 0; r < rows; ++r) {
        double mx = -INFINITY;
        for (int p = 0; p < parts; ++p)
            if (lse_parts[(size_t)p * rows + r] > mx) mx = lse_parts[(size_t)p * rows + r];
        double *orow = o + (size_t)r * d;
        for (int i = 0; i < d; ++i) orow[i] = 0.0;
        if (mx == -INFINITY) { if (lse) lse[r] = -INFINITY; continue; }
        double l = 0.0;
        for (int p = 0; p < parts; ++p) l += exp(lse_parts[(size_t)p * rows + r] - mx);
        const double total = mx + log(l);
        for (int p = 0; p < parts; ++p) {
            const double w = exp(lse_parts[(size_t)p * rows + r] - total);
            for (int i = 0; i < d; ++i) orow[i] += w * o_parts[((size_t)p * rows + r) * d + i];
        }
        if (lse) lse[r] = total;
    }
    return 0;
}

/* ------------------------------------------------------------------------------------
 * FP8 KV storage ("FP16/INT8 KV formats").  Reading
 * R21: every stored K or V row (one token, one kv head, d channels) is
 *     x_i = c_i * 2^e,   c_i an OCP FP8 E4M3 value (1 sign, 4 exponent bits with bias 7,
 *                        3 mantissa bits; largest finite 448, no infinities),
 *                        e an integer in [-64, 64] chosen per row:
 *     e = the smallest integer in [-64, 64] with max_i |x_i| <= 448 * 2^e,
 *     c_i = the E4M3 value nearest to x_i * 2^-e (ties to the even mantissa; magnitudes
 *           beyond 448 saturate to 448).
 * Because 2^e is a power of two, every dequantised value c_i * 2^e (4 significant bits,
 * |e| <= 64) is exactly a bf16 / fp32 number, so the page metadata built over the
 * dequantised keys (Eq. 1) stays exact and r (Eq. 2) stays an upper bound.
 * ---------------------------------------------------------------------------------- */

/* Value of an E4M3 code (the format definition written out). */
double or_e4m3_value(uint8_t c) {
    const int s = c >> 7, E = (c >> 3) & 15, m = c & 7;
    double v;
    if (E == 15 && m == 7) return NAN;                 /* the only NaN encodings */
    if (E == 0) v = ldexp((double)m / 8.0, -6);        /* subnormal: m/8 * 2^(1-7) */
    else v = ldexp(1.0 + (double)m / 8.0, E - 7);      /* normal: 1.m * 2^(E-7) */
    return s ? -v : v;
}

/* Nearest E4M3 code to x, ties to the even code (mantissa LSB 0), |x| > 448 saturates; the
 * sign bit is x's.  The non-negative finite codes 0..126 have increasing values, so the
 * answer is the lower or the upper neighbour of |x| among them (found by bisection). */
uint8_t or_e4m3_round(double x) {
    const double a = fabs(x);
    int best;
    if (a >= 448.0) {
        best = 126;                                    /* saturate (0x7e = 448) */
    } else {
        int lo = 0, hi = 126;                          /* value(lo) <= a < value(hi) */
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if (or_e4m3_value((uint8_t)mid) <= a) lo = mid; else hi = mid;
        }
        const double dl = a - or_e4m3_value((uint8_t)lo), dh = or_e4m3_value((uint8_t)hi) - a;
        best = (dl < dh || (dl == dh && (lo & 1) == 0)) ? lo : hi;
    }
    return (uint8_t)(best | (signbit(x) ? 0x80 : 0));
}

/* The row exponent: smallest e in [-64, 64] with amax <= 448 * 2^e. */
int or_kv_exponent(double amax) {
    int e = -64;
    while (e < 64 && amax > ldexp(448.0, e)) ++e;
    return e;
}

/* Quantise `rows` bf16 rows of d channels (src [rows][d] bf16 bits) into codes [rows][d]
 * and exponents [rows]. */
void or_kv_quantize(long long rows, int d, const uint16_t *src, uint8_t *codes, int8_t *exps) {
    for (long long r = 0; r < rows; ++r) {
        double amax = 0.0;
        for (int i = 0; i < d; ++i) {
            const double x = fabs(widen(src, 1, (size_t)r * d + i));
            if (x > amax) amax = x;
        }
        const int e = or_kv_exponent(amax);
        exps[r] = (int8_t)e;
        for (int i = 0; i < d; ++i)
            codes[(size_t)r * d + i] = or_e4m3_round(ldexp(widen(src, 1, (size_t)r * d + i), -e));
    }
}

/* Dequantise to fp32 (exact): out[r][i] = value(codes[r][i]) * 2^exps[r]. */
void or_kv_dequantize(long long rows, int d, const uint8_t *codes, const int8_t *exps, float *out) {
    for (long long r = 0; r < rows; ++r)
        for (int i = 0; i < d; ++i)
            out[(size_t)r * d + i] = (float)ldexp(or_e4m3_value(codes[(size_t)r * d + i]), exps[r]);
}
