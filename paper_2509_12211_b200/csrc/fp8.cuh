// fp8.cuh — FP8 KV storage ("FP16/INT8 KV formats").
//
// Reading R21: every stored K or V row (one token, one kv head, 64 channels)
// is 64 OCP E4M3 codes c_i plus one power-of-two scale 2^e (an int8 exponent):
//     e = the smallest integer in [-64, 64] with max_i |x_i| <= 448 * 2^e,
//     c_i = E4M3 nearest to x_i * 2^-e (round to nearest even, saturating at 448).
// Dequantised values c_i * 2^e are exact bf16 numbers, so the metadata (bf16, Eq. 1) over
// the dequantised keys is exact and r (Eq. 2) remains an upper bound of q.k.
//
// Pool layout (include/tinyserve.h): an FP8 pool is [NB][Hkv][S][64] codes followed by
// [NB][Hkv][S] int8 exponents (one byte per row), i.e. NB*Hkv*S*65 bytes.
//
//   kv_quantize_kernel     bf16 rows -> codes + exponents (prefill / cache import)
//   meta_append_f8_kernel  the append (Eq. 1 maintenance) of a bf16 token into an FP8 cache
//   meta_build_f8_kernel   metadata over the dequantised keys of every page
#pragma once
#include "common.cuh"
#include "meta.cuh"

namespace ts {

constexpr int kF8MinExp = -64, kF8MaxExp = 64;

// 2^e as an fp32 (|e| <= 126)
TS_DEV float pow2i(int e) { return __uint_as_float(uint32_t(127 + e) << 23); }

// Row exponent from the row's max |x| (reading R21).  amax = 1.f * 2^E (normal fp32):
// amax <= 1.75 * 2^(8 + e)  <=>  e >= E - 8 when f <= 1.75, else e >= E - 7.
TS_DEV int f8_row_exp(float amax) {
    const uint32_t u = __float_as_uint(amax);
    const int bexp = int(u >> 23);
    int e = bexp == 0 ? kF8MinExp : (bexp - 127) - 8 + ((u & 0x7fffffu) > 0x600000u ? 1 : 0);
    return min(max(e, kF8MinExp), kF8MaxExp);
}

// four fp32 -> four E4M3 codes (byte k = element k), round to nearest even, saturating
TS_DEV uint32_t f8x4_pack(float a, float b, float c, float d) {
    uint16_t lo, hi;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return uint32_t(lo) | (uint32_t(hi) << 16);
}

// two E4M3 codes (low byte = element 0) -> f16x2 (exact)
TS_DEV uint32_t f8x2_to_f16x2(uint32_t two) {
    uint32_t r;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(r) : "h"((uint16_t)two));
    return r;
}

// four codes -> their values times 2^e as packed bf16x2 (exact: 4 significant bits)
TS_DEV uint2 f8x4_dequant_bf16(uint32_t w, float sc) {
    const uint32_t h01 = f8x2_to_f16x2(w & 0xffffu), h23 = f8x2_to_f16x2(w >> 16);
    const __half2 a = *reinterpret_cast<const __half2 *>(&h01), b = *reinterpret_cast<const __half2 *>(&h23);
    const float2 fa = __half22float2(a), fb = __half22float2(b);
    uint32_t r0, r1;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r0) : "f"(fa.y * sc), "f"(fa.x * sc));
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r1) : "f"(fb.y * sc), "f"(fb.x * sc));
    return make_uint2(r0, r1);
}

// Quantise 8 bf16 channels (one lane of an aligned group of 8 lanes holding a 64-channel
// row): returns the 8 codes and the row exponent (same in all 8 lanes).
TS_DEV uint2 f8_quantize8(uint4 x, int &e_out) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    float f[8];
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16lo_to_f32(w[i]);
        f[2 * i + 1] = bf16hi_to_f32(w[i]);
        amax = fmaxf(amax, fmaxf(fabsf(f[2 * i]), fabsf(f[2 * i + 1])));
    }
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 2));
    amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, 4));
    const int e = f8_row_exp(amax);
    const float s = pow2i(-e);  // exact scaling
    e_out = e;
    return make_uint2(f8x4_pack(f[0] * s, f[1] * s, f[2] * s, f[3] * s),
                      f8x4_pack(f[4] * s, f[5] * s, f[6] * s, f[7] * s));
}

// ts_kv_quantize: rows of 64 bf16 -> codes [rows][64] + exps [rows]; 8 lanes per row.
__global__ void kv_quantize_kernel(long long rows, const uint16_t *__restrict__ src,
                                   uint8_t *__restrict__ codes, int8_t *__restrict__ exps) {
    pdl_launch_dependents();
    pdl_wait();
    const long long nthr = rows * 8;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w - (threadIdx.x & 31) < nthr;
         w += (long long)gridDim.x * blockDim.x) {
        const bool live = w < nthr;  // whole warps iterate (the shuffles span 8 lanes)
        const long long r = w >> 3;
        const int c = int(w & 7);
        const uint4 x = live ? *reinterpret_cast<const uint4 *>(src + r * 64 + c * 8) : make_uint4(0, 0, 0, 0);
        int e;
        const uint2 q = f8_quantize8(x, e);
        if (live) {
            *reinterpret_cast<uint2 *>(codes + r * 64 + c * 8) = q;
            if (c == 0) exps[r] = (int8_t)e;
        }
    }
}

// The append into an FP8 cache (meta_append_kernel's contract, Eq. 1 over the DEQUANTISED
// key): grid.x = B, block = Hkv * 8 threads (8 lanes per kv head, 8 channels each).
__global__ void meta_append_f8_kernel(MetaParams p, const uint16_t *__restrict__ k_new,
                                      const uint16_t *__restrict__ v_new, int *__restrict__ seq_lens,
                                      int advance, const int *__restrict__ page_table,
                                      uint8_t *__restrict__ k_pool, uint8_t *__restrict__ v_pool,
                                      int8_t *__restrict__ k_exp, int8_t *__restrict__ v_exp,
                                      uint16_t *__restrict__ meta) {
    pdl_launch_dependents();
    pdl_wait();
    const int b = blockIdx.x;
    const int h = threadIdx.x >> 3, c = threadIdx.x & 7;
    const int t = seq_lens[b] + (advance < 0 ? -1 : 0);
    const long long cap = (long long)p.max_pages * p.stride * p.S;
    if (advance > 0) {
        __syncthreads();
        if (threadIdx.x == 0 && t + 1LL <= cap) seq_lens[b] = t + 1;
    }
    // warp-uniform exits only (8-lane groups shuffle): every condition below is per block
    if (t < 0 || t >= cap) return;
    const int j = t / p.S, slot = t % p.S;
    if (j % p.stride != p.offset) return;
    const int jl = j / p.stride;
    if (jl >= p.max_pages) return;
    const bool live = h < p.Hkv;
    const int hh = live ? h : 0;
    const int blk = checked_block(page_table[(size_t)b * p.max_pages + jl], p.num_blocks);
    const size_t src = ((size_t)b * p.Hkv + hh) * 64 + c * 8;
    const uint4 k = *reinterpret_cast<const uint4 *>(k_new + src);
    const uint4 v = *reinterpret_cast<const uint4 *>(v_new + src);
    int ek, ev;
    const uint2 kq = f8_quantize8(k, ek);
    const uint2 vq = f8_quantize8(v, ev);
    if (!live) return;
    const size_t row = ((size_t)blk * p.Hkv + h) * p.S + slot;
    *reinterpret_cast<uint2 *>(k_pool + row * 64 + c * 8) = kq;
    *reinterpret_cast<uint2 *>(v_pool + row * 64 + c * 8) = vq;
    if (c == 0) {
        k_exp[row] = (int8_t)ek;
        v_exp[row] = (int8_t)ev;
    }
    // metadata over the dequantised key (exact bf16)
    const float sc = pow2i(ek);
    const uint2 d0 = f8x4_dequant_bf16(kq.x, sc), d1 = f8x4_dequant_bf16(kq.y, sc);
    const uint4 kd = make_uint4(d0.x, d0.y, d1.x, d1.y);
    uint16_t *mrec = meta + (((size_t)b * p.Hkv + h) * p.max_pages + jl) * 2 * 64 + c * 8;
    uint4 *mn = reinterpret_cast<uint4 *>(mrec);
    uint4 *mx = reinterpret_cast<uint4 *>(mrec + 64);
    if (slot == 0) {
        *mn = kd;
        *mx = kd;
    } else {
        *mn = Vec16<uint16_t>::vmin(*mn, kd);
        *mx = Vec16<uint16_t>::vmax(*mx, kd);
    }
}

// Metadata over the dequantised keys: one thread per (b, local page, kv head, 8 channels).
__global__ void meta_build_f8_kernel(MetaParams p, const uint8_t *__restrict__ k_pool,
                                     const int8_t *__restrict__ k_exp,
                                     const int *__restrict__ page_table,
                                     const int *__restrict__ seq_lens, uint16_t *__restrict__ meta) {
    pdl_launch_dependents();
    pdl_wait();
    const long long total = (long long)p.B * p.max_pages * p.Hkv * 8;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < total;
         w += (long long)gridDim.x * blockDim.x) {
        const int c = int(w & 7);
        long long r = w >> 3;
        const int h = int(r % p.Hkv);
        r /= p.Hkv;
        const int jl = int(r % p.max_pages);
        const int b = int(r / p.max_pages);
        const long long j = (long long)jl * p.stride + p.offset;
        const long long nvalid = (long long)seq_lens[b] - j * p.S;
        if (nvalid <= 0) continue;
        const int n = nvalid < p.S ? int(nvalid) : p.S;
        const int blk = checked_block(page_table[(size_t)b * p.max_pages + jl], p.num_blocks);
        const size_t row0 = ((size_t)blk * p.Hkv + h) * p.S;
        uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
        for (int s = 0; s < n; ++s) {
            const uint2 q = *reinterpret_cast<const uint2 *>(k_pool + (row0 + s) * 64 + c * 8);
            const float sc = pow2i(k_exp[row0 + s]);
            const uint2 d0 = f8x4_dequant_bf16(q.x, sc), d1 = f8x4_dequant_bf16(q.y, sc);
            const uint4 x = make_uint4(d0.x, d0.y, d1.x, d1.y);
            lo = s ? Vec16<uint16_t>::vmin(lo, x) : x;
            hi = s ? Vec16<uint16_t>::vmax(hi, x) : x;
        }
        uint16_t *mrec = meta + (((size_t)b * p.Hkv + h) * p.max_pages + jl) * 2 * 64 + c * 8;
        *reinterpret_cast<uint4 *>(mrec) = lo;
        *reinterpret_cast<uint4 *>(mrec + 64) = hi;
    }
}

}  // namespace ts
