// fused_step.cuh — the bf16 decode step (Alg. 1: score, select, gather,
// attend; "in a single pass") as ONE cooperative persistent kernel for batches
// with many (sequence, kv head) rows.
//
// The grid is split statically into two roles that run at the same time (cooperative
// launch: every CTA is resident, so the spin-waits below cannot deadlock):
//  * CTAs [0, NS): score + select (score_select_role, score_select.cuh): row r is scored
//    and selected by CTA r mod NS; its flag ready[r] is released when the selection (page
//    ids + physical blocks + count) is in global memory;
//  * CTAs [NS, NS + NA): attention (attention_role below): CTA NS + a attends rows a,
//    a + NA, ... in the selector's order, so it starts on a row as soon as the row is
//    released, while later rows are still being scored — the metadata stream and the K/V
//    stream overlap on HBM without a kernel boundary or a PDL launch gap.
// attention_role: a producer warp waits for the row's flag, resolves the owned selected
// pages and streams [16 x 64] K / V tiles (2-D TMA, 128-byte swizzle, L2 evict-first) into
// an R-stage ring; W consumer warps run S = Q K^T (mma.m16n8k16 bf16), the fp32 online
// softmax (exp2) and O += P V (mma.m16n8k8, tf32 P — reading R10) per tile, then merge the
// warp partials and write o (fp32) and lse.  The producer runs ahead into the next row.
#pragma once
#include "attn.cuh"
#include "common.cuh"
#include "score_select.cuh"
#include "sparse_attn.cuh"

namespace ts {

template <int W, int R>
struct AttnRoleSmem {
    static constexpr int kTile = 16 * kRowBytes;                   // 2 KB
    static constexpr int kStage = 2 * kTile;                       // K + V
    static constexpr int kRing = 0;                                // 1024-aligned (swizzle)
    static constexpr int kWarpPart = kRing + R * kStage;           // [W][8][kSaPart] fp32
    static constexpr int kQ = kWarpPart + W * 8 * kSaPart * 4;     // [2][8][64] bf16
    static constexpr int kInfo = kQ + 2 * 8 * kRowBytes;           // [R] int token0
    static constexpr int kRowInfo = kInfo + R * 4;                 // [2] int4 (tile0, ntile, row, -)
    static constexpr int kBars = (kRowInfo + 32 + 7) / 8 * 8;      // full, empty [R]; rowfull, rowempty [2]
    static constexpr int kPages = kBars + (2 * R + 4) * 8;         // [sel_stride] int2 (row0, tok0)
    static size_t bytes(int sel_stride) { return kPages + (size_t)sel_stride * 8; }
};

template <int W, int R>
TS_DEV void attention_role(const CUtensorMap *tmK, const CUtensorMap *tmV, const AttnParams &p,
                           int unit, int nunits, uint8_t *smem) {
    using SM = AttnRoleSmem<W, R>;
    static_assert(R % W == 0, "stage -> consumer warp must be fixed");
    const uint32_t sb = smem_u32(smem);
    const uint32_t full0 = sb + SM::kBars, empty0 = full0 + 8 * R;
    const uint32_t rowfull0 = empty0 + 8 * R, rowempty0 = rowfull0 + 16;
    float *wpart = reinterpret_cast<float *>(smem + SM::kWarpPart);
    int *info = reinterpret_cast<int *>(smem + SM::kInfo);
    int4 *rowinfo = reinterpret_cast<int4 *>(smem + SM::kRowInfo);
    int2 *pages = reinterpret_cast<int2 *>(smem + SM::kPages);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rows = p.B * p.Hkv;
    unsigned long long *dts = p.dbg && unit < 2048 ? p.dbg + unit * 8 : nullptr;
    if (dts && threadIdx.x == 0) dts[0] = globaltimer();
    if (threadIdx.x == 0) {
        prefetch_tmap(tmK);
        prefetch_tmap(tmV);
        for (int i = 0; i < R; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(rowfull0 + 8 * i, 1);
            mbar_init(rowempty0 + 8 * i, 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int tpp = p.S >> 4;  // tiles per page
    const int qbytes = p.G * kRowBytes;

    if (warp == W) {
        // ================================ producer ================================
        const uint64_t pol = l2_policy_evict_first();
        int gt = 0;
        for (int it = 0;; ++it) {
            const int row = unit + it * nunits;
            if (row >= rows) break;
            const int b = row / p.Hkv, g = row % p.Hkv;
            const int rs = it & 1;
            if (lane == 0) {
                mbar_wait(rowempty0 + 8 * rs, ((it >> 1) & 1) ^ 1);
                // q of the row's group -> qbuf[rs] (counted on rowfull)
                mbar_expect_tx(rowfull0 + 8 * rs, qbytes);  // the arrive comes with rowinfo
                bulk_load(sb + SM::kQ + rs * 8 * kRowBytes,
                          static_cast<const uint16_t *>(p.q) + ((size_t)b * p.Hq + g * p.G) * kAttnD,
                          qbytes, rowfull0 + 8 * rs);
                while (ld_relaxed_u32(p.ready + row) == 0u) nanosleep_ns(64);
                fence_acquire_gpu();
                if (dts && it == 0) dts[1] = globaltimer();
            }
            __syncwarp();
            const int cnt = __ldcg(p.sel_count + row);
            const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
            const int *blks = p.sel_blk + (size_t)row * p.sel_stride;
            int n = 0;
            for (int u0 = 0; u0 < cnt; u0 += 32) {
                const int u = u0 + lane;
                const bool own = u < cnt;
                const unsigned m = __ballot_sync(0xffffffffu, own);
                if (own) pages[n + lane] = make_int2((__ldcg(blks + u) * p.Hkv + g) * p.S, __ldcg(ids + u) * p.S);
                n += __popc(m);
            }
            __syncwarp();
            const int ntile = n * tpp;
            if (lane == 0) {
                p.ready[row] = 0u;  // this CTA is the row's only reader; re-armed for the next step
                rowinfo[rs] = make_int4(gt, ntile, row, 0);
                mbar_arrive(rowfull0 + 8 * rs);
                for (int i = 0; i < ntile; ++i, ++gt) {
                    const int st = gt % R;
                    mbar_wait(empty0 + 8 * st, ((gt / R) & 1) ^ 1);
                    const int u = i / tpp, sub = i - u * tpp;
                    const int2 pg = pages[u];
                    info[st] = pg.y + 16 * sub;
                    mbar_arrive_expect_tx(full0 + 8 * st, SM::kStage);
                    const uint32_t dst = sb + SM::kRing + st * SM::kStage;
                    tma_load_2d(dst, tmK, 0, pg.x + 16 * sub, full0 + 8 * st, pol);
                    tma_load_2d(dst + SM::kTile, tmV, 0, pg.x + 16 * sub, full0 + 8 * st, pol);
                }
            } else {
                gt += ntile;
            }
            __syncwarp();
        }
        return;
    }
    if (warp > W) return;  // spare warp of the shared CTA shape

    // ================================ consumers ===============================
    const int gid = lane >> 2, t = lane & 3;
    const float sl2 = p.scale * kLog2e;
    for (int it = 0;; ++it) {
        const int row = unit + it * nunits;
        if (row >= rows) break;
        const int b = row / p.Hkv, g = row % p.Hkv;
        const int rs = it & 1;
        const int L = p.seq_lens[b];
        mbar_wait(rowfull0 + 8 * rs, (it >> 1) & 1);
        const int4 ri = rowinfo[rs];
        const int g0 = ri.x, ntile = ri.y;
        uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (gid < p.G) {
            const uint32_t qrow = sb + SM::kQ + rs * 8 * kRowBytes + gid * kRowBytes + 32 * t;
            const uint4 x0 = lds_v4(qrow), x1 = lds_v4(qrow + 16);
            qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
            qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
        }
        float m = kNegInf, lp = 0.f;
        float oacc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
        for (int gl = g0 + (warp - g0 % W + W) % W; gl < g0 + ntile; gl += W) {
            const int st = gl % R;
            mbar_wait(full0 + 8 * st, (gl / R) & 1);
            const int tok0 = info[st];
            const uint32_t kb = sb + SM::kRing + st * SM::kStage, vb = kb + SM::kTile;
            float sacc[2][4];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
                const int r = nt * 8 + gid;
                const uint32_t ra = kb + r * kRowBytes;
                const uint4 k0 = lds_v4(ra + (((2 * t) ^ (r & 7)) << 4));
                const uint4 k1 = lds_v4(ra + (((2 * t + 1) ^ (r & 7)) << 4));
                mma_bf16_16816(sacc[nt], qa[0], 0u, qa[1], 0u, k0.x, k0.y);
                mma_bf16_16816(sacc[nt], qa[2], 0u, qa[3], 0u, k0.z, k0.w);
                mma_bf16_16816(sacc[nt], qa[4], 0u, qa[5], 0u, k1.x, k1.y);
                mma_bf16_16816(sacc[nt], qa[6], 0u, qa[7], 0u, k1.z, k1.w);
            }
            float x[2][2];
            float tmax = kNegInf;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    const bool ok = tok0 + nt * 8 + 2 * t + q2 < L;
                    x[nt][q2] = ok ? sacc[nt][q2] * sl2 : kNegInf;
                    tmax = fmaxf(tmax, x[nt][q2]);
                }
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
            const float mnew = fmaxf(m, tmax);
            const float mref = mnew == kNegInf ? 0.f : mnew;
            const float corr = exp2f(m - mref);
            m = mnew;
            float pr[2][2];
            float psum = 0.f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    pr[nt][q2] = exp2f(x[nt][q2] - mref);
                    psum += pr[nt][q2];
                }
            lp = lp * corr + psum;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                oacc[j][0] *= corr;
                oacc[j][1] *= corr;
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int q0 = nt * 8 + 2 * t, q1 = q0 + 1;
                uint4 v0 = lds_v4(vb + q0 * kRowBytes + ((gid ^ (q0 & 7)) << 4));
                uint4 v1 = lds_v4(vb + q1 * kRowBytes + ((gid ^ (q1 & 7)) << 4));
                if (tok0 + q0 >= L) v0 = make_uint4(0, 0, 0, 0);  // past seq_len: may be anything
                if (tok0 + q1 >= L) v1 = make_uint4(0, 0, 0, 0);
                const uint32_t a0 = f32_to_tf32(pr[nt][0]), a2 = f32_to_tf32(pr[nt][1]);
                const uint32_t w0[4] = {v0.x, v0.y, v0.z, v0.w};
                const uint32_t w1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t b0 = (j & 1) ? (w0[j >> 1] & 0xffff0000u) : (w0[j >> 1] << 16);
                    const uint32_t b1 = (j & 1) ? (w1[j >> 1] & 0xffff0000u) : (w1[j >> 1] << 16);
                    mma_tf32_1688(oacc[j], a0, 0u, a2, 0u, b0, b1);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * st);
        }
        // ---- warp partial: head gid, channels 16t + j (c0) and 16t + 8 + j (c1)
        lp += __shfl_xor_sync(0xffffffffu, lp, 1);
        lp += __shfl_xor_sync(0xffffffffu, lp, 2);
        if (gid < p.G) {
            float *wr = wpart + (warp * 8 + gid) * kSaPart;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                wr[16 * t + j] = oacc[j][0];
                wr[16 * t + 8 + j] = oacc[j][1];
            }
            if (t == 0) {
                wr[kAttnD] = m;
                wr[kAttnD + 1] = lp;
            }
        }
        named_bar_sync(2, W * 32);
        if (threadIdx.x == 0) mbar_arrive(rowempty0 + 8 * rs);  // rowinfo / q slot reusable
        // ---- merge the W warp partials, write o and lse
        for (int x = threadIdx.x; x < p.G * 16; x += W * 32) {
            const int h = x >> 4, d0 = (x & 15) * 4;
            float M = kNegInf;
#pragma unroll
            for (int w = 0; w < W; ++w) M = fmaxf(M, wpart[(w * 8 + h) * kSaPart + kAttnD]);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            float l = 0.f;
            if (M != kNegInf) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    const float *wr = wpart + (w * 8 + h) * kSaPart;
                    const float mw = wr[kAttnD];
                    const float f = mw == kNegInf ? 0.f : exp2f(mw - M);
                    l += wr[kAttnD + 1] * f;
                    const float4 v = *reinterpret_cast<const float4 *>(wr + d0);
                    acc.x += v.x * f; acc.y += v.y * f; acc.z += v.z * f; acc.w += v.w * f;
                }
            }
            const size_t oh = (size_t)b * p.Hq + g * p.G + h;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
            if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
        }
        named_bar_sync(2, W * 32);  // wpart reusable
        if (dts && threadIdx.x == 0 && it == 0) dts[3] = globaltimer();
    }
}

// One launch, two roles (see the header).  blockDim = (W + 2) * 32 for both.
template <int W, int R1, int R2, int KPL>
__global__ void __launch_bounds__((W + 2) * 32) decode_fused_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
    ScoreSelParams sp, AttnParams ap, int pt_pref, int ns) {
    extern __shared__ uint8_t fs_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(fs_raw) + 1023) &
                                                ~uintptr_t(1023));
    if ((int)blockIdx.x < ns)
        score_select_role<W, R1, KPL>(sp, pt_pref, blockIdx.x, ns, smem);
    else
        attention_role<W, R2>(&tmK, &tmV, ap, blockIdx.x - ns, gridDim.x - ns, smem);
}

}  // namespace ts
