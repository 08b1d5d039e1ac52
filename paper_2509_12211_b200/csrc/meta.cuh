// meta.cuh — page metadata maintenance (Eq. 1).
//   ts_meta_append: fused K/V slot write + running min/max of the page
//   ts_meta_build : min/max over the valid keys of every page
// Both are exact in every dtype (compare/select only).  One thread per 16-byte chunk of a
// (page, kv-head) record: 128-bit loads/stores, coalesced along head_dim.  Metadata lives in
// the LOGICAL layout [B][Hkv][max_pages][2][D] (row (b, g) contiguous, page order), so that
// scoring is one contiguous stream per row with no page-table indirection.
#pragma once
#include "common.cuh"

namespace ts {

struct MetaParams {
    int B, Hkv, D, S, max_pages, stride, offset, num_blocks;
};

template <typename T>
struct Vec16;  // 16-byte chunk ops for a dtype
template <>
struct Vec16<uint16_t> {  // bf16
    static constexpr int kElems = 8;
    TS_DEV static uint4 vmin(uint4 a, uint4 b) {
        return make_uint4(bf16x2_min(a.x, b.x), bf16x2_min(a.y, b.y), bf16x2_min(a.z, b.z),
                          bf16x2_min(a.w, b.w));
    }
    TS_DEV static uint4 vmax(uint4 a, uint4 b) {
        return make_uint4(bf16x2_max(a.x, b.x), bf16x2_max(a.y, b.y), bf16x2_max(a.z, b.z),
                          bf16x2_max(a.w, b.w));
    }
};
template <>
struct Vec16<float> {
    static constexpr int kElems = 4;
    TS_DEV static uint32_t fmn(uint32_t a, uint32_t b) {
        return __float_as_uint(fminf(__uint_as_float(a), __uint_as_float(b)));
    }
    TS_DEV static uint32_t fmx(uint32_t a, uint32_t b) {
        return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b)));
    }
    TS_DEV static uint4 vmin(uint4 a, uint4 b) {
        return make_uint4(fmn(a.x, b.x), fmn(a.y, b.y), fmn(a.z, b.z), fmn(a.w, b.w));
    }
    TS_DEV static uint4 vmax(uint4 a, uint4 b) {
        return make_uint4(fmx(a.x, b.x), fmx(a.y, b.y), fmx(a.z, b.z), fmx(a.w, b.w));
    }
};

// grid.x = B, block = Hkv * chunks_per_row threads (chunks_per_row = D / elems_per_chunk).
template <typename T>
__global__ void meta_append_kernel(MetaParams p, const T *__restrict__ k_new,
                                   const T *__restrict__ v_new, int *__restrict__ seq_lens,
                                   int advance, const int *__restrict__ page_table,
                                   T *__restrict__ k_pool, T *__restrict__ v_pool,
                                   T *__restrict__ meta) {
    pdl_launch_dependents();
    pdl_wait();
    using V = Vec16<T>;
    const int cpr = p.D / V::kElems;
    const int b = blockIdx.x;
    const int h = threadIdx.x / cpr, c = threadIdx.x % cpr;
    // advance < 0 (internal, ts_decode_step_append fallback): seq_lens already counts the
    // new token, which goes to slot t = seq_len - 1
    const int t = seq_lens[b] + (advance < 0 ? -1 : 0);
    // capacity of the sequence: global pages j < max_pages * stride (the last rank's local
    // row may be one page short; that page has no slot and is rejected below).  A token past
    // the capacity is dropped AND the length is not advanced, so no later step sees a
    // P_b beyond the page-table row (the oracle's or_meta_append reports a shape error here).
    const long long cap = (long long)p.max_pages * p.stride * p.S;
    if (advance > 0) {  // every thread has read t; then one thread publishes t + 1
        __syncthreads();
        if (threadIdx.x == 0 && t + 1LL <= cap) seq_lens[b] = t + 1;
    }
    if (h >= p.Hkv || t < 0 || t >= cap) return;
    const int j = t / p.S, slot = t % p.S;
    if (j % p.stride != p.offset) return;  // page owned by another rank
    const int jl = j / p.stride;
    if (jl >= p.max_pages) return;
    const int blk = checked_block(page_table[(size_t)b * p.max_pages + jl], p.num_blocks);
    const size_t src = ((size_t)b * p.Hkv + h) * p.D + c * V::kElems;
    const uint4 k = *reinterpret_cast<const uint4 *>(k_new + src);
    const uint4 v = *reinterpret_cast<const uint4 *>(v_new + src);
    const size_t dst = (((size_t)blk * p.Hkv + h) * p.S + slot) * p.D + c * V::kElems;
    *reinterpret_cast<uint4 *>(k_pool + dst) = k;
    *reinterpret_cast<uint4 *>(v_pool + dst) = v;
    // logical metadata layout [B][Hkv][max_pages][2][D]
    T *mrec = meta + (((size_t)b * p.Hkv + h) * p.max_pages + jl) * 2 * p.D + c * V::kElems;
    uint4 *mn = reinterpret_cast<uint4 *>(mrec);
    uint4 *mx = reinterpret_cast<uint4 *>(mrec + p.D);
    if (slot == 0) {  // first key of a page: m = M = k
        *mn = k;
        *mx = k;
    } else {
        *mn = V::vmin(*mn, k);
        *mx = V::vmax(*mx, k);
    }
}

// One thread per (b, local page, kv head, chunk).  grid-stride over all of them.
template <typename T>
__global__ void meta_build_kernel(MetaParams p, const T *__restrict__ k_pool,
                                  const int *__restrict__ page_table,
                                  const int *__restrict__ seq_lens, T *__restrict__ meta) {
    pdl_launch_dependents();
    pdl_wait();
    using V = Vec16<T>;
    const int cpr = p.D / V::kElems;
    const long long total = (long long)p.B * p.max_pages * p.Hkv * cpr;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total;
         w += (long long)gridDim.x * blockDim.x) {
        const int c = int(w % cpr);
        long long r = w / cpr;
        const int h = int(r % p.Hkv);
        r /= p.Hkv;
        const int jl = int(r % p.max_pages);
        const int b = int(r / p.max_pages);
        const int L = seq_lens[b];
        debug_flag(L < 0 || L > (long long)p.max_pages * p.stride * p.S, kDbgSeqLen);
        const long long j = (long long)jl * p.stride + p.offset;  // global page id
        const long long nvalid = (long long)L - j * p.S;
        if (nvalid <= 0) continue;
        const int n = nvalid < p.S ? int(nvalid) : p.S;
        const int blk = checked_block(page_table[(size_t)b * p.max_pages + jl], p.num_blocks);
        const T *src = k_pool + ((size_t)blk * p.Hkv + h) * p.S * p.D + c * V::kElems;
        uint4 lo = *reinterpret_cast<const uint4 *>(src);
        uint4 hi = lo;
        for (int s = 1; s < n; ++s) {
            const uint4 x = *reinterpret_cast<const uint4 *>(src + (size_t)s * p.D);
            lo = V::vmin(lo, x);
            hi = V::vmax(hi, x);
        }
        T *mrec = meta + (((size_t)b * p.Hkv + h) * p.max_pages + jl) * 2 * p.D + c * V::kElems;
        *reinterpret_cast<uint4 *>(mrec) = lo;
        *reinterpret_cast<uint4 *>(mrec + p.D) = hi;
    }
}

}  // namespace ts
