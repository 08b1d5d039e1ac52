// select.cuh — top-K page selection (Alg. 1 Step 2 "shared heap or radix
// select").  One CTA per row, block-level radix select on orderable
// uint32 keys of the fp32 scores (score_key: -0.0 == +0.0), 4 passes of 8 bits:
//   pass p: histogram the digit of the keys whose higher digits match the prefix found so
//   far, then find the digit that holds the rem-th largest key.
// After 4 passes T is the exact K-th largest key and need_eq = how many keys == T to take.
// Ties at T go to the lower id (reading R6): for affine ids (id = i*id_stride + id_offset,
// monotone in i) this is index order, done by two block scans that also emit the selected
// ids in ascending order with no sort.  With explicit ids_in (candidate merge)
// tie ranks and output positions are counted over the >= T candidates (O(C^2), C ~ K).
// Exact: only integer comparisons.  Deterministic.
#pragma once
#include "common.cuh"

namespace ts {

constexpr int kSelThreads = 512;

struct SelectParams {
    const float *scores;
    int rows, stride;         // entries per row (= parts * kp)
    const int *row_len;       // nullable
    const int *ids_in;        // nullable
    int id_stride, id_offset, k;
    int kp;                   // entries per row per part (== stride when parts == 1)
    long long part_stride;    // elements between parts (candidate merge)
    int *sel_ids;
    float *sel_scores;    // nullable
    int *sel_count;
};

// Block-wide exclusive scan of one int per thread (kSelThreads threads); returns the
// exclusive prefix and writes the total to *total.  `wsum` is smem[kSelThreads/32 + 1].
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
        constexpr int NW = kSelThreads / 32;
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
    *total = wsum[kSelThreads / 32 - 1];
    __syncthreads();
    return before;
}

__global__ void __launch_bounds__(kSelThreads) select_topk_kernel(SelectParams p) {
    extern __shared__ uint32_t sm[];  // keys [stride] (+ ids, flags [stride] if ids_in)
    __shared__ int hist[256];
    __shared__ int wsum[kSelThreads / 32 + 1];
    __shared__ int bc[4];
    uint32_t *keys = sm;
    int *ids = reinterpret_cast<int *>(sm + p.stride);
    const int r = blockIdx.x;
    const int tid = threadIdx.x;
    const int len = p.row_len ? min(p.row_len[r], p.stride) : p.stride;
    int nvalid = 0;
    for (int i = tid; i < len; i += kSelThreads) {
        // entry i of row r = element (part i / kp, row r, column i % kp)
        const size_t at = (size_t)(i / p.kp) * p.part_stride + (size_t)r * p.kp + (i % p.kp);
        const uint32_t key = score_key(p.scores[at]);
        keys[i] = key;
        if (p.ids_in) ids[i] = p.ids_in[at];
        nvalid += key != kKeyNegInf;
    }
    int tot;
    block_excl_scan(nvalid, wsum, &tot);
    const int kk = min(p.k, tot);
    int *out_ids = p.sel_ids + (size_t)r * p.k;
    float *out_sc = p.sel_scores ? p.sel_scores + (size_t)r * p.k : nullptr;
    for (int i = kk + tid; i < p.k; i += kSelThreads) {
        out_ids[i] = -1;
        if (out_sc) out_sc[i] = kNegInf;
    }
    if (tid == 0) p.sel_count[r] = kk;
    if (kk == 0) return;

    // ---- radix select: find T = kk-th largest key, need_eq
    uint32_t prefix = 0, pmask = 0;
    int rem = kk;
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += kSelThreads) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < len; i += kSelThreads) {
            const uint32_t key = keys[i];
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns bins [8l, 8l+8); suffix sums from the top bin down
            int c[8], s = 0;
#pragma unroll
            for (int e = 7; e >= 0; --e) { c[e] = hist[tid * 8 + e]; s += c[e]; }
            int suf = s;  // inclusive suffix over lanes >= tid
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf, o);
                if (tid + o < 32) suf += y;
            }
            const int above = suf - s;  // keys in bins of higher lanes
            const unsigned ball = __ballot_sync(0xffffffffu, suf >= rem && above < rem);
            const int L = 31 - __clz(ball);  // exactly one lane qualifies
            if (tid == L) {
                int acc = above, d = 8 * L + 7;
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    if (acc + c[e] >= rem) { d = 8 * L + e; break; }
                    acc += c[e];
                }
                bc[0] = d;
                bc[1] = acc;  // keys strictly above digit d (within the prefix)
            }
        }
        __syncthreads();
        prefix |= uint32_t(bc[0]) << shift;
        pmask |= 0xffu << shift;
        rem -= bc[1];
        __syncthreads();
    }
    const uint32_t T = prefix;
    const int need_eq = rem;  // >= 1

    if (!p.ids_in) {
        // ---- affine ids: ascending id == ascending index.  Contiguous segment per thread.
        const int per = (len + kSelThreads - 1) / kSelThreads;
        const int lo = tid * per, hi = min(len, lo + per);
        int n_gt = 0, n_eq = 0;
        for (int i = lo; i < hi; ++i) {
            const uint32_t key = keys[i];
            n_gt += key > T;
            n_eq += key == T;
        }
        const int eq_before = block_excl_scan(n_eq, wsum, &tot);
        const int take_eq = max(0, min(n_eq, need_eq - eq_before));
        int pos = block_excl_scan(n_gt + take_eq, wsum, &tot);
        int eq_seen = 0;
        for (int i = lo; i < hi; ++i) {
            const uint32_t key = keys[i];
            bool sel = key > T;
            if (key == T) { sel = eq_seen < take_eq; ++eq_seen; }
            if (sel) {
                out_ids[pos] = i * p.id_stride + p.id_offset;
                if (out_sc) out_sc[pos] = key_score(key);
                ++pos;
            }
        }
    } else {
        // ---- explicit ids: compact candidates (key >= T) then rank by id.  Requires
        // per-thread segments of <= 16 entries (stride <= 16 * kSelThreads, host-checked).
        int *flg = ids + p.stride;
        int mine = 0;
        const int per = (len + kSelThreads - 1) / kSelThreads;
        const int lo = tid * per, hi = min(len, lo + per);
        uint32_t kbuf[16];
        int ibuf[16];
        for (int i = lo; i < hi; ++i)
            if (keys[i] >= T) { kbuf[mine] = keys[i]; ibuf[mine] = ids[i]; ++mine; }
        const int pos = block_excl_scan(mine, wsum, &tot);  // (contains __syncthreads)
        const int C = tot;
        for (int x = 0; x < mine; ++x) { keys[pos + x] = kbuf[x]; ids[pos + x] = ibuf[x]; }
        __syncthreads();
        // selected: key > T, or key == T with fewer than need_eq tied ids below it
        for (int c = tid; c < C; c += kSelThreads) {
            bool sel = keys[c] > T;
            if (keys[c] == T) {
                int below = 0;
                for (int x = 0; x < C; ++x) below += (keys[x] == T) && (ids[x] < ids[c]);
                sel = below < need_eq;
            }
            flg[c] = sel;
        }
        __syncthreads();
        for (int c = tid; c < C; c += kSelThreads) {
            if (!flg[c]) continue;
            int rank = 0;
            for (int x = 0; x < C; ++x) rank += flg[x] && (ids[x] < ids[c]);
            out_ids[rank] = ids[c];
            if (out_sc) out_sc[rank] = key_score(keys[c]);
        }
    }
}

}  // namespace ts
