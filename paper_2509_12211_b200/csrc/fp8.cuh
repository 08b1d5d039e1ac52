// fp8.cuh — FP8 KV storage ("FP16/INT8 KV formats").
//
// Reading R21: every stored K or V row (one token, one kv head, 64 channels)
// is 64 OCP E4M3 codes c_i plus one power-of-two scale 2^e (an int8 exponent):
//     e = the smallest integer in [-64, 64] with max_i |x_i| <= 448 * 2^e,
//     c_i = E4M3 nearest to x_i * 2^-e (round to nearest even, saturating at 448).
// Dequantised values c_i * 2^e are exact bf16 numbers, so the metadata (bf16, Eq. 1) over
// the dequantised keys is exact and r (Eq. 2) remains an upper bound of q.k.
//
// Pool layout (include/tinyserve.h): an FP8 pool is a sequence of 1040-byte SUB-PAGE RECORDS,
// one per 16 consecutive rows (token, kv head) of [NB][Hkv][S] (S a multiple of 16): the 16
// rows' codes [16][64] then their 16 exponent bytes.  A 16-token attention tile and its scales
// are one contiguous 1040-byte bulk copy; NB*Hkv*S*65 bytes in total.
//
//   kv_quantize_kernel     bf16 rows -> codes + exponents (prefill / cache import)
//   meta_append_f8_kernel  the append (Eq. 1 maintenance) of a bf16 token into an FP8 cache
//   meta_build_f8_kernel   metadata over the dequantised keys of every page
#pragma once
#include "attn.cuh"
#include "common.cuh"
#include "meta.cuh"

namespace ts {

constexpr int kF8MinExp = -64, kF8MaxExp = 64;
constexpr int kF8Rec = 16 * 64 + 16;  // one sub-page record: 16 rows of codes + 16 exponents
// byte offsets of row r's codes / exponent in an FP8 pool
TS_DEV size_t f8_code_off(size_t r) { return (r >> 4) * kF8Rec + (r & 15) * 64; }
TS_DEV size_t f8_exp_off(size_t r) { return (r >> 4) * kF8Rec + 16 * 64 + (r & 15); }

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
// row): returns the 8 codes and the row exponent (same in all 8 lanes).  `mask`: the lanes
// executing the call (each aligned group of 8 complete).
TS_DEV uint2 f8_quantize8(uint4 x, int &e_out, unsigned mask = 0xffffffffu) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    float f[8];
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16lo_to_f32(w[i]);
        f[2 * i + 1] = bf16hi_to_f32(w[i]);
        amax = fmaxf(amax, fmaxf(fabsf(f[2 * i]), fabsf(f[2 * i + 1])));
    }
    amax = fmaxf(amax, __shfl_xor_sync(mask, amax, 1));
    amax = fmaxf(amax, __shfl_xor_sync(mask, amax, 2));
    amax = fmaxf(amax, __shfl_xor_sync(mask, amax, 4));
    const int e = f8_row_exp(amax);
    const float s = pow2i(-e);  // exact scaling
    e_out = e;
    return make_uint2(f8x4_pack(f[0] * s, f[1] * s, f[2] * s, f[3] * s),
                      f8x4_pack(f[4] * s, f[5] * s, f[6] * s, f[7] * s));
}

// ts_kv_quantize: rows of 64 bf16 -> an FP8 pool (sub-page records); 8 lanes per row.
__global__ void kv_quantize_kernel(long long rows, const uint16_t *__restrict__ src,
                                   uint8_t *__restrict__ pool) {
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
            *reinterpret_cast<uint2 *>(pool + f8_code_off(r) + c * 8) = q;
            if (c == 0) pool[f8_exp_off(r)] = (uint8_t)(int8_t)e;
        }
    }
}

// The append into an FP8 cache (meta_append_kernel's contract, Eq. 1 over the DEQUANTISED
// key): grid.x = B, block = Hkv * 8 threads (8 lanes per kv head, 8 channels each).
__global__ void meta_append_f8_kernel(MetaParams p, const uint16_t *__restrict__ k_new,
                                      const uint16_t *__restrict__ v_new, int *__restrict__ seq_lens,
                                      int advance, const int *__restrict__ page_table,
                                      uint8_t *__restrict__ k_pool, uint8_t *__restrict__ v_pool,
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
    *reinterpret_cast<uint2 *>(k_pool + f8_code_off(row) + c * 8) = kq;
    *reinterpret_cast<uint2 *>(v_pool + f8_code_off(row) + c * 8) = vq;
    if (c == 0) {
        k_pool[f8_exp_off(row)] = (uint8_t)(int8_t)ek;
        v_pool[f8_exp_off(row)] = (uint8_t)(int8_t)ev;
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
            const uint2 q = *reinterpret_cast<const uint2 *>(k_pool + f8_code_off(row0 + s) + c * 8);
            const float sc = pow2i((int8_t)k_pool[f8_exp_off(row0 + s)]);
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

// ---------------------------------------------------------------------------------------
// The FP8 attention consumer (reading R21), shared by decode_cluster_kernel (F8) and
// sparse_attn_tma_kernel (F8).  Per 16-token tile, lane (gid, t):
//  S = Q'·K_code^T on mma.m16n8k16 f16 (E4M3 widens exactly to f16; q' = q * 2^-sq per head,
//  |q'| in [2^14, 2^15), so bf16 q is exact in f16), times 2^(e_k + sq) per token; the online
//  softmax keeps the V accumulator relative to (running max, running max V exponent E), so
//  P' = P * 2^(e_v - E) <= 1 enters O^T += V_code^T P'^T as a hi + lo f16 pair; 2^E is applied
//  when the partial is stored.  Token order in each 8-token MMA group: f8_tok (the two 64-byte
//  K rows read by each 8-lane phase of a 128-bit shared load have different parity: no bank
//  conflicts without a swizzle).
TS_DEV int f8_tok(int n) { return ((n ^ (n >> 1)) & 1) | ((n & 1) << 1) | (n & 4); }

struct F8Q {
    uint32_t qh[8];  // f16x2 of q' channels 16t + {2i, 2i+1} (head gid)
    float qsc;       // softmax scale * log2(e) * 2^sq
};
// x0, x1: the lane's 32 bytes of q (bf16 channels 16t .. 16t + 15 of head gid; zero if gid >= G)
TS_DEV F8Q f8_q_prep(uint4 x0, uint4 x1, float sl2) {
    F8Q f;
    const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    float am = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) am = fmaxf(am, fmaxf(fabsf(bf16lo_to_f32(w[i])), fabsf(bf16hi_to_f32(w[i]))));
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 1));
    am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 2));
    const int ea = int(__float_as_uint(am) >> 23) - 127;  // floor(log2 am) for normal am
    const int sq = am > 0.f ? min(max(ea - 14, -100), 100) : 0;
    const float s = pow2i(-sq);
#pragma unroll
    for (int i = 0; i < 8; ++i) f.qh[i] = f16x2_pack(bf16lo_to_f32(w[i]) * s, bf16hi_to_f32(w[i]) * s);
    f.qsc = sl2 * pow2i(sq);
    return f;
}

struct F8Acc {
    float m = kNegInf, lp = 0.f;
    int E = -128;  // running max V exponent of the attended tokens (-128: none yet)
    float oacc[4][4];  // O^T: channels (8 gid + 2 db, + 1) x heads (2t, 2t+1)
    TS_DEV F8Acc() {
#pragma unroll
        for (int j = 0; j < 4; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
    }
};

// One 16-token tile: the K and V sub-page records at kb / vb (codes [16][64] bytes, then the 16
// exponent bytes at +1024); tokens tok0 + r, valid while < L.
TS_DEV void f8_attend_tile(F8Acc &a, const F8Q &q, uint32_t kb, uint32_t vb, int tok0, int L, int gid, int t) {
    int trow[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) trow[nt][q2] = nt * 8 + f8_tok(2 * t + q2);
    float sacc[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
        sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
        const int r = nt * 8 + f8_tok(gid);  // B column gid = this K row
        const uint4 k = lds_v4(kb + r * 64 + (t << 4));
        const uint32_t kw[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
        for (int kc = 0; kc < 4; ++kc)
            mma_f16_16816(sacc[nt], q.qh[2 * kc], 0u, q.qh[2 * kc + 1], 0u, f8x2_to_f16x2(kw[kc] & 0xffffu),
                          f8x2_to_f16x2(kw[kc] >> 16));
    }
    float x[2][2];
    bool ok[2][2];
    int ev[2][2];
    float tmax = kNegInf;
    int evmax = -128;
    // row exponents: 8-byte reads per 8-token group, the lane's bytes picked with PRMT
    const uint2 ke0 = lds_v2(kb + 1024), ke1 = lds_v2(kb + 1032), ve0 = lds_v2(vb + 1024), ve1 = lds_v2(vb + 1032);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
            const int r = trow[nt][q2];
            ok[nt][q2] = tok0 + r < L;
            const uint2 kw = nt ? ke1 : ke0, vw = nt ? ve1 : ve0;
            const int sb_ = r & 7;
            const int ek = int(__byte_perm(kw.x, kw.y, sb_) << 24) >> 24;
            ev[nt][q2] = int(__byte_perm(vw.x, vw.y, sb_) << 24) >> 24;
            x[nt][q2] = ok[nt][q2] ? sacc[nt][q2] * q.qsc * pow2i(ek) : kNegInf;
            tmax = fmaxf(tmax, x[nt][q2]);
            if (ok[nt][q2]) evmax = max(evmax, ev[nt][q2]);
        }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    evmax = max(evmax, __shfl_xor_sync(0xffffffffu, evmax, 1));
    evmax = max(evmax, __shfl_xor_sync(0xffffffffu, evmax, 2));
    const int En = max(a.E, evmax);
    const float mnew = fmaxf(a.m, tmax);
    const float mref = mnew == kNegInf ? 0.f : mnew;
    const float corr = exp2f(a.m - mref);
    const float corr_o = corr * exp2f((float)(a.E - En));
    a.m = mnew;
    a.E = En;
    float pr[2][2];
    float psum = 0.f;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
            const float pw = exp2f(x[nt][q2] - mref);
            psum += pw;
            const int de = ev[nt][q2] - a.E;  // <= 0 for attended tokens
            pr[nt][q2] = ok[nt][q2] && de >= -126 ? pw * pow2i(de) : 0.f;
        }
    a.lp = a.lp * corr + psum;
    ot_rescale(a.oacc, corr_o, t);
    // B = P'^T (k = this lane's tokens, n = head gid), hi + lo f16 parts
    const uint32_t ah0 = f16x2_pack(pr[0][0], pr[0][1]), ah2 = f16x2_pack(pr[1][0], pr[1][1]);
    const float2 h0 = __half22float2(*reinterpret_cast<const __half2 *>(&ah0));
    const float2 h2 = __half22float2(*reinterpret_cast<const __half2 *>(&ah2));
    const uint32_t al0 = f16x2_pack(pr[0][0] - h0.x, pr[0][1] - h0.y);
    const uint32_t al2 = f16x2_pack(pr[1][0] - h2.x, pr[1][1] - h2.y);
    // A = V^T: channels 8 gid .. 8 gid + 7 (8 code bytes) of this lane's 4 token rows
    uint2 vr[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
            const uint2 v = lds_v2(vb + trow[nt][q2] * 64 + gid * 8);
            vr[nt][q2] = ok[nt][q2] ? v : make_uint2(0, 0);  // past seq_len: may be anything
        }
#pragma unroll
    for (int db = 0; db < 4; ++db) {  // channels 8 gid + 2 db (A rows gid) and + 1 (rows gid + 8)
        const uint32_t sel_ = (db & 1) ? 0x7362u : 0x5140u;
        const uint32_t p0 = __byte_perm(db < 2 ? vr[0][0].x : vr[0][0].y, db < 2 ? vr[0][1].x : vr[0][1].y, sel_);
        const uint32_t p1 = __byte_perm(db < 2 ? vr[1][0].x : vr[1][0].y, db < 2 ? vr[1][1].x : vr[1][1].y, sel_);
        const uint32_t a0 = f8x2_to_f16x2(p0 & 0xffffu), a1 = f8x2_to_f16x2(p0 >> 16);
        const uint32_t a2 = f8x2_to_f16x2(p1 & 0xffffu), a3 = f8x2_to_f16x2(p1 >> 16);
        mma_f16_16816(a.oacc[db], a0, a1, a2, a3, ah0, ah2);
        mma_f16_16816(a.oacc[db], a0, a1, a2, a3, al0, al2);
    }
}

// the warp's partial: O^T rows of heads 2t, 2t+1 (x 2^E) and (m, l) of head gid
TS_DEV void f8_store_partial(float *wpart_warp, int ld, F8Acc &a, int gid, int t, int G) {
    a.lp += __shfl_xor_sync(0xffffffffu, a.lp, 1);
    a.lp += __shfl_xor_sync(0xffffffffu, a.lp, 2);
    const float s2e = a.E > -128 ? pow2i(a.E) : 1.f;  // back from the V-exponent reference
    ot_store(wpart_warp, ld, a.oacc, gid, t, G, s2e);
    if (gid < G && t == 0) {
        wpart_warp[gid * ld + kAttnD] = a.m;
        wpart_warp[gid * ld + kAttnD + 1] = a.lp;
    }
}

}  // namespace ts
