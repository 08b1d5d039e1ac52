// score.cuh — bounding-box page scoring (Eq. 2; Alg. 1 Step 1, 217-224).
//
//   s[b][g][jl] = max_{h in group g} sum_i max(q_hi * m_i, q_hi * M_i)
//              = max_h ( q_h^+ . M + q_h^- . m )            (m <= M; reading R3)
//
// This is a streaming read of the metadata: one 2*d-element record per (page, kv head), in
// the logical layout [B][Hkv][max_pages][2][d], so a row is one contiguous run.
//  * bf16, G <= 8: the record row [m | M] (K = 2d) times the coefficient matrix
//    [q^- ; q^+] (2d x G) is a 16-page x 2d x 8-head product per warp tile, run on the
//    tensor cores with mma.sync.m16n8k16 (bf16 x bf16 products are exact in fp32).  The
//    metadata goes global -> registers with coalesced 128-bit loads straight into the
//    A-fragments under a fixed k-permutation (the same permutation is applied to the
//    coefficients), so no shared-memory staging is needed.  Why tensor cores: at G = 8 the
//    CUDA-core form needs 4 FMA per metadata byte, ~26 T FMA/s at HBM rate — more than
//    the FFMA budget of 148 SMs.
//  * fp32 (any G) and bf16 with G > 8: CUDA-core FFMA, a group of lanes per record with a
//    fixed shuffle tree (SIMT path).
// A page's score is a pure function of (q, its record): fixed lane/fragment assignment and
// reduction order, independent of grid position or sharding.  -0.0 is written as +0.0.
#pragma once
#include "common.cuh"

namespace ts {

struct ScoreParams {
    int B, Hq, Hkv, G, D, S, max_pages, stride, offset;
};


// ------------------------------------------------------------------ tensor-core path
// D = 64 or 128 (bf16).  CTA = 4 warps, each warp 2 tiles of 16 pages -> 128 pages/CTA.
// grid = (ceil(max_pages / 128), B * Hkv).
constexpr int kScoreWarps = 4;
constexpr int kScoreTilesPerWarp = 2;
constexpr int kScorePagesPerCta = kScoreWarps * kScoreTilesPerWarp * 16;

// Scores of pages [chunk * 128, chunk * 128 + 128) of row `row` by one 4-warp CTA.
template <int D>
TS_DEV void score_mma_block(const ScoreParams &p, const uint16_t *__restrict__ q,
                            const uint16_t *__restrict__ meta, const int *__restrict__ page_table,
                            const int *__restrict__ seq_lens, float *__restrict__ scores, int row,
                            int chunk) {
    constexpr int CH = 2 * D / 8;    // 16-byte chunks per record (16 for d = 64)
    constexpr int CPT = CH / 4;      // chunks per thread per record row
    constexpr int STEPS = CH / 2;    // k16 steps per record
    const int b = row / p.Hkv, g = row % p.Hkv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, t = lane & 3;
    const int P = local_pages(clamp_len(seq_lens[b], p.max_pages, p.stride, p.S), p.S, p.stride, p.offset);
    const int cta_base = chunk * kScorePagesPerCta;
    float *srow = scores + (size_t)row * p.max_pages;

    if (cta_base >= P) {  // nothing to score: fill -inf for this CTA's slice
        for (int j = cta_base + threadIdx.x; j < min(cta_base + kScorePagesPerCta, p.max_pages);
             j += blockDim.x)
            srow[j] = kNegInf;
        return;
    }

    // ---- metadata loads first (all tiles, all chunks): 2 * 2 * CPT 128-bit loads/thread
    uint4 a[kScoreTilesPerWarp][2][CPT];
    const int warp_base = cta_base + warp * kScoreTilesPerWarp * 16;
#pragma unroll
    for (int tt = 0; tt < kScoreTilesPerWarp; ++tt)
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            const int jl = warp_base + tt * 16 + gid + hr * 8;
            if (jl < P) {
                const uint16_t *rec = meta + ((size_t)row * p.max_pages + jl) * 2 * D;
#pragma unroll
                for (int i = 0; i < CPT; ++i) a[tt][hr][i] = ldg_nc_v4(rec + (t + 4 * i) * 8);
            } else {
#pragma unroll
                for (int i = 0; i < CPT; ++i) a[tt][hr][i] = make_uint4(0, 0, 0, 0);
            }
        }

    // ---- coefficients (B fragment): column n = gid <-> q head g*G + gid.
    // Thread chunk i covers record elements 8(t+4i) .. +7: min part (coef q^-) for
    // t+4i < CH/2, max part (coef q^+) otherwise; both use q channels 8(t + 4(i mod CPT/2)).
    uint32_t bq[CPT][4];
    {
        const bool live = gid < p.G;
        const uint16_t *qh = q + ((size_t)b * p.Hq + g * p.G + (live ? gid : 0)) * D;
#pragma unroll
        for (int i = 0; i < CPT / 2; ++i) {
            uint4 v = live ? ldg_v4(qh + 8 * (t + 4 * i)) : make_uint4(0, 0, 0, 0);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                bq[i][e] = bf16x2_min0(w[e]);            // q^- for the min part
                bq[i + CPT / 2][e] = bf16x2_max0(w[e]);  // q^+ for the max part
            }
        }
    }

#pragma unroll
    for (int tt = 0; tt < kScoreTilesPerWarp; ++tt) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < STEPS; ++s) {
            const int i = s >> 1, h2 = (s & 1) * 2;  // chunk i, pairs h2 and h2+1
            const uint4 &lo = a[tt][0][i];
            const uint4 &hi = a[tt][1][i];
            const uint32_t lo0 = h2 ? lo.z : lo.x, lo1 = h2 ? lo.w : lo.y;
            const uint32_t hi0 = h2 ? hi.z : hi.x, hi1 = h2 ? hi.w : hi.y;
            mma_bf16_16816(acc, lo0, hi0, lo1, hi1, bq[i][h2], bq[i][h2 + 1]);
        }
        // acc: (page gid, heads 2t,2t+1), (page gid+8, heads 2t, 2t+1)
        const bool c0 = 2 * t < p.G, c1 = 2 * t + 1 < p.G;
        float m0 = fmaxf(c0 ? acc[0] : kNegInf, c1 ? acc[1] : kNegInf);
        float m1 = fmaxf(c0 ? acc[2] : kNegInf, c1 ? acc[3] : kNegInf);
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
        if (t < 2) {
            const int jl = warp_base + tt * 16 + gid + t * 8;
            if (jl < p.max_pages) srow[jl] = jl < P ? (t ? m1 : m0) + 0.0f : kNegInf;
        }
    }
}

template <int D>
__global__ void __launch_bounds__(kScoreWarps * 32)
    score_mma_kernel(ScoreParams p, const uint16_t *__restrict__ q,
                     const uint16_t *__restrict__ meta, const int *__restrict__ page_table,
                     const int *__restrict__ seq_lens, float *__restrict__ scores) {
    pdl_launch_dependents();  // PDL: the next call's prologue may overlap this kernel
    pdl_wait();               // inputs may come from the previous call in the stream
    score_mma_block<D>(p, q, meta, page_table, seq_lens, scores, blockIdx.y, blockIdx.x);
}

// ------------------------------------------------------------------ SIMT path
// Record = 2*D elements of T; LPR lanes per record (16-byte chunk each, CPL chunks per
// lane).  q of the group staged in smem as fp32 [G][D].  grid = (ceil(max_pages/PPC), rows).
constexpr int kSimtWarps = 4;
constexpr int kSimtPagesPerCta = 64;

template <typename T, int D>
__global__ void __launch_bounds__(kSimtWarps * 32)
    score_simt_kernel(ScoreParams p, const T *__restrict__ q, const T *__restrict__ meta,
                      const int *__restrict__ page_table, const int *__restrict__ seq_lens,
                      float *__restrict__ scores) {
    constexpr int EPC = 16 / sizeof(T);               // elements per chunk
    constexpr int CH = 2 * D / EPC;                   // chunks per record
    constexpr int LPR = CH < 32 ? CH : 32;            // lanes per record
    constexpr int CPL = CH / LPR;                     // chunks per lane
    constexpr int RPW = 32 / LPR;                     // records per warp pass
    extern __shared__ float qs[];                     // [G][D]: q^- then q^+ as one row of 2D
    pdl_launch_dependents();
    pdl_wait();
    const int row = blockIdx.y;
    const int b = row / p.Hkv, g = row % p.Hkv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int P = local_pages(clamp_len(seq_lens[b], p.max_pages, p.stride, p.S), p.S, p.stride, p.offset);
    float *srow = scores + (size_t)row * p.max_pages;
    const int base = blockIdx.x * kSimtPagesPerCta;
    // coefficient rows [G][2D]: [q^- | q^+]
    for (int x = threadIdx.x; x < p.G * D; x += blockDim.x) {
        const int hh = x / D, i = x % D;
        const T qv = q[((size_t)b * p.Hq + g * p.G + hh) * D + i];
        float f;
        if constexpr (sizeof(T) == 2) f = bf16_to_f32(qv); else f = qv;
        qs[hh * 2 * D + i] = fminf(f, 0.f);
        qs[hh * 2 * D + D + i] = fmaxf(f, 0.f);
    }
    __syncthreads();
    const int sub = lane / LPR, sl = lane % LPR;
    for (int j0 = base + warp * RPW; j0 < min(base + kSimtPagesPerCta, p.max_pages);
         j0 += kSimtWarps * RPW) {
        const int jl = j0 + sub;
        const bool live = jl < P && jl < min(base + kSimtPagesPerCta, p.max_pages);
        float e[CPL][EPC];
        if (live) {
            const T *rec = meta + ((size_t)row * p.max_pages + jl) * 2 * D;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const T *src = rec + (sl + c * LPR) * EPC;
#pragma unroll
                for (int k = 0; k < EPC; ++k) {
                    if constexpr (sizeof(T) == 2) e[c][k] = bf16_to_f32(src[k]); else e[c][k] = src[k];
                }
            }
        } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int k = 0; k < EPC; ++k) e[c][k] = 0.f;
        }
        float best = kNegInf;
        for (int hh = 0; hh < p.G; ++hh) {
            float part = 0.f;
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int k = 0; k < EPC; ++k)
                    part = fmaf(qs[hh * 2 * D + (sl + c * LPR) * EPC + k], e[c][k], part);
#pragma unroll
            for (int o = LPR / 2; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            best = fmaxf(best, part);
        }
        if (sl == 0 && jl < min(base + kSimtPagesPerCta, p.max_pages))
            srow[jl] = live ? best + 0.0f : kNegInf;
    }
}

}  // namespace ts
