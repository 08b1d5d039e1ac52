// select.cuh — top-K page selection (Alg. 1 Step 2 "shared heap or radix
// select").  Block-level radix select on orderable uint32 keys of the fp32
// scores (score_key: -0.0 == +0.0, larger score <-> larger key):
//   3 passes with digits of 11, 11 and 10 bits; pass p histograms the digit of the keys
//   whose higher digits equal the prefix found so far and picks the digit holding the
//   rem-th largest key.  If that digit's whole bin is needed (count == rem) the search
//   stops early and every key in the bin is taken.
// After the passes T (= prefix, compared under the prefix mask) is the K-th largest key
// and need_eq = how many keys equal to T to take.  Ties at T go to the lower id
// (reading R6): for affine ids (id = i*id_stride + id_offset, monotone in i) this is index
// order, done by two block scans that also emit the selected ids in ascending order with no
// sort.  With explicit ids_in (candidate merge) tie ranks and output
// positions are counted over the >= T candidates (O(C^2), C ~ K).
// Exact: only integer comparisons.  Deterministic.
#pragma once
#include "common.cuh"
#include "score_select.cuh"  // cta_topk

namespace ts {

constexpr int kSelThreads = 512;  // standalone select kernel
constexpr int kHistBins = 2048;

struct SelectParams {
    const float *scores;
    int rows, stride;         // entries per row (= parts * kp)
    const int *row_len;       // nullable
    const int *ids_in;        // nullable
    int id_stride, id_offset, k;
    int kp;                   // entries per row per part (== stride when parts == 1)
    long long part_stride;    // elements between parts (candidate merge)
    int *sel_ids;
    float *sel_scores;        // nullable
    int *sel_count;
};

// Shared scratch of select_row (static size).
template <int NT>
struct SelectSmem {
    int hist[kHistBins];
    int wsum[NT / 32 + 1];
    int bc[4];
    int red[64];        // cta_topk scratch
    uint32_t cand[128];  // cta_topk candidate slots
};

// Block-wide exclusive scan of one int per thread (NT threads); returns the exclusive
// prefix and writes the total to *total.
template <int NT>
TS_DEV int block_excl_scan(int v, int *wsum, int *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        constexpr int NW = NT / 32;
        int s = lane < NW ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < NW) wsum[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    const int before = (warp ? wsum[warp - 1] : 0) + x - v;
    *total = wsum[NT / 32 - 1];
    __syncthreads();
    return before;
}

// Radix search for the kk-th largest key among keys[0..len).  Returns (prefix, pmask,
// rem): the selected set is {key & pmask > prefix} plus the first `rem` (lowest id) keys
// with key & pmask == prefix.
template <int NT>
TS_DEV void radix_threshold(const uint32_t *keys, int len, int kk, SelectSmem<NT> &S,
                            uint32_t &prefix_out, uint32_t &pmask_out, int &rem_out) {
    constexpr int BPT = kHistBins / NT;  // bins per thread
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t prefix = 0, pmask = 0;
    int rem = kk;
#pragma unroll 1
    for (int ps = 0; ps < 3; ++ps) {
        const int shift = ps == 0 ? 21 : (ps == 1 ? 10 : 0);
        const uint32_t dmask = ps == 2 ? 0x3ffu : 0x7ffu;
        for (int i = tid; i < kHistBins; i += NT) S.hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < len; i += NT) {
            const uint32_t key = keys[i];
            if ((key & pmask) == prefix) atomicAdd(&S.hist[(key >> shift) & dmask], 1);
        }
        __syncthreads();
        // block suffix scan over bins: thread tid owns bins [tid*BPT, tid*BPT + BPT)
        int c[BPT], s = 0;
#pragma unroll
        for (int e = BPT - 1; e >= 0; --e) { c[e] = S.hist[tid * BPT + e]; s += c[e]; }
        int suf = s;  // inclusive suffix within the warp
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_down_sync(0xffffffffu, suf, o);
            if (lane + o < 32) suf += y;
        }
        if (lane == 0) S.wsum[warp] = suf;  // warp total
        __syncthreads();
        int after = 0;  // keys in the warps above mine
        for (int w = warp + 1; w < NT / 32; ++w) after += S.wsum[w];
        suf += after;
        const int above = suf - s;
        if (suf >= rem && above < rem) {  // exactly one thread
            int acc = above, d = tid * BPT, cd = 0;
#pragma unroll
            for (int e = BPT - 1; e >= 0; --e) {
                if (acc + c[e] >= rem) { d = tid * BPT + e; cd = c[e]; break; }
                acc += c[e];
            }
            S.bc[0] = d;
            S.bc[1] = acc;
            S.bc[2] = cd;
        }
        __syncthreads();
        prefix |= uint32_t(S.bc[0]) << shift;
        pmask |= dmask << shift;
        rem -= S.bc[1];
        const bool done = S.bc[2] == rem;  // the whole bin is taken
        __syncthreads();
        if (done) break;
    }
    prefix_out = prefix;
    pmask_out = pmask;
    rem_out = rem;
}

// Selection of row r by the whole CTA (NT threads).  keys: smem [stride] (+ ids, flags
// [stride] each if ids_in).  Scores are read with ld.global.cg (they may have been written
// by other CTAs of the same grid).
template <int NT>
TS_DEV void select_row(const SelectParams &p, int r, uint32_t *keys, SelectSmem<NT> &S) {
    int *ids = reinterpret_cast<int *>(keys + p.stride);
    const int tid = threadIdx.x;
    const int len = p.row_len ? min(p.row_len[r], p.stride) : p.stride;

    int nvalid = 0;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
    const int lenp = p.ids_in ? len : ((len + 3) & ~3);  // affine: zero-padded to 4 (uint4 scans)
    for (int i = tid; i < lenp; i += NT) {
        // entry i of row r = element (part i / kp, row r, column i % kp)
        uint32_t key = 0u;
        if (i < len) {
            const size_t at = (size_t)(i / p.kp) * p.part_stride + (size_t)r * p.kp + (i % p.kp);
            key = score_key(__ldcg(p.scores + at));
            if (p.ids_in) ids[i] = p.ids_in[at];
            if (key != kKeyNegInf) {
                ++nvalid;
                kmin = min(kmin, key);
                kmax = max(kmax, key);
            }
        }
        // affine ids: -inf ("no page") -> 0, below every live key (cta_topk convention)
        keys[i] = (!p.ids_in && key == kKeyNegInf) ? 0u : key;
    }
    int tot;
    block_excl_scan<NT>(nvalid, S.wsum, &tot);
    const int kk = min(p.k, tot);
    int *out_ids = p.sel_ids + (size_t)r * p.k;
    float *out_sc = p.sel_scores ? p.sel_scores + (size_t)r * p.k : nullptr;
    for (int i = kk + tid; i < p.k; i += NT) {
        out_ids[i] = -1;
        if (out_sc) out_sc[i] = kNegInf;
    }
    if (tid == 0) p.sel_count[r] = kk;
    if (kk == 0) return;

    if (!p.ids_in) {
        // ---- affine ids (ascending id == ascending index): the adaptive radix top-K of the
        // fused kernels (score_select.cuh)
        block_minmax<NT, 0>(kmin, kmax, S.red);
        for (int i = tid; i < kHistBins; i += NT) S.hist[i] = 0;
        __syncthreads();
        cta_topk<NT, 0, 11>(keys, len, p.k, kmin, kmax, S.hist, S.red, S.cand,
                            [&](int pos, int i) {
                                out_ids[pos] = i * p.id_stride + p.id_offset;
                                if (out_sc) out_sc[pos] = key_score(keys[i]);
                            },
                            nullptr, false, tot);
        return;
    }
    uint32_t T = kKeyNegInf, pmask = 0xffffffffu;
    int need_eq = 0;  // kk == tot: every candidate (key > key(-inf)) is selected
    if (kk < tot) radix_threshold<NT>(keys, len, kk, S, T, pmask, need_eq);

    {
        // ---- explicit ids: compact candidates (masked key >= T) then rank by id.  Requires
        // per-thread segments of <= 16 entries (stride <= 16 * NT, host-checked).
        int *flg = ids + p.stride;
        int mine = 0;
        const int per = (len + NT - 1) / NT;
        const int lo = tid * per, hi = min(len, lo + per);
        uint32_t kbuf[16];
        int ibuf[16];
        for (int i = lo; i < hi; ++i)
            if ((keys[i] & pmask) >= T && keys[i] != kKeyNegInf) {
                kbuf[mine] = keys[i];
                ibuf[mine] = ids[i];
                ++mine;
            }
        const int pos = block_excl_scan<NT>(mine, S.wsum, &tot);  // (contains __syncthreads)
        const int C = tot;
        for (int x = 0; x < mine; ++x) { keys[pos + x] = kbuf[x]; ids[pos + x] = ibuf[x]; }
        __syncthreads();
        // selected: masked key > T, or == T with fewer than need_eq tied ids below it
        for (int c = tid; c < C; c += NT) {
            const uint32_t kc = keys[c] & pmask;
            bool sel = kc > T;
            if (kc == T) {
                int below = 0;
                for (int x = 0; x < C; ++x) below += ((keys[x] & pmask) == T) && (ids[x] < ids[c]);
                sel = below < need_eq;
            }
            flg[c] = sel;
        }
        __syncthreads();
        for (int c = tid; c < C; c += NT) {
            if (!flg[c]) continue;
            int rank = 0;
            for (int x = 0; x < C; ++x) rank += flg[x] && (ids[x] < ids[c]);
            out_ids[rank] = ids[c];
            if (out_sc) out_sc[rank] = key_score(keys[c]);
        }
    }
}

__global__ void __launch_bounds__(kSelThreads) select_topk_kernel(SelectParams p) {
    extern __shared__ uint32_t sm[];
    __shared__ SelectSmem<kSelThreads> S;
    pdl_launch_dependents();
    pdl_wait();
    select_row<kSelThreads>(p, blockIdx.x, sm, S);
}

}  // namespace ts
