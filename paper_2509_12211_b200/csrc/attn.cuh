// attn.cuh — sparse gather + masked softmax attention over the selected pages
// (SparseAttn PAPER.md:169-172; Alg. 1 Steps 3-4).
//
// bf16 path (attn_mma_kernel), split-K flash-decode:
//  * work item = (row (b, kv head g), split); persistent CTAs walk items with a fixed
//    stride.  Each item covers a contiguous range of the row's selected-page tiles
//    (TT = min(S, 16) tokens per tile).
//  * Step 3 (gather): every warp owns a private STAGES-deep ring of shared-memory tile
//    buffers filled by TMA tile loads (cp.async.bulk.tensor.2d, 128-byte swizzle, L2
//    evict-first) of K and V rows [TT x 64] of one page of one kv head, completing on a
//    per-stage mbarrier.  No block-wide barrier inside the streaming loop.
//  * Step 4 (attention) on the tensor cores, entirely from the swizzled smem tiles:
//      S^T = Q K^T  : mma.m16n8k16 bf16, A = the G query heads of the group (rows), B = K^T
//                     (8 tokens); conflict-free 128-bit smem reads thanks to the swizzle.
//      O  += P V    : mma.m16n8k8 tf32 with A = P (fp32 probabilities rounded to tf32,
//                     straight from the S accumulators), B = V (bf16 widened exactly);
//                     the k (token) order is permuted so no transpose is needed.
//    fp32 online softmax in the log2 domain (exp2), masking of tokens >= seq_len by
//    selection (partial V rows zeroed in smem so 0 * garbage cannot make NaN).
//  * merge: warps -> CTA through smem; CTAs of a row through an fp32 (o, m, l) partial
//    in the workspace, merged by the last CTA to finish the row (atomic ticket), which
//    also re-arms the ticket.  Output o fp32, lse = ln sum exp (natural log).
// fp32 path (attn_simt_kernel): CUDA-core FFMA, one warp per q head, lane-parallel dot
// products with a fixed shuffle tree (no tf32 anywhere; reading R10).
#pragma once
#include "common.cuh"

namespace ts {

struct AttnParams {
    const void *q;
    const int *page_table;
    const int *seq_lens;
    const int *sel_ids;
    const int *sel_count;
    int sel_stride;
    int B, Hq, Hkv, G, D, S, max_pages, stride, offset;
    float scale;       // softmax scale (reading R1)
    float *o;
    float *lse;        // nullable
    float *part;       // [rows][splits][8][kPS]
    unsigned *tickets; // [rows]
    int splits, items;
};

constexpr int kAttnD = 64;        // head_dim of the tensor-core path
constexpr int kRowBytes = kAttnD * 2;
constexpr int kPS = kAttnD + 4;   // floats per (split, head) partial: o[D], m, l, pad (16 B aligned)

template <int TT, int NW, int STAGES>
struct AttnSmem {
    static constexpr int kTileBytes = TT * kRowBytes;                  // one K or V tile
    static constexpr int kStageBytes = 2 * kTileBytes;
    static constexpr int kRingBytes = NW * STAGES * kStageBytes;
    static constexpr int kScratchBytes = NW * 8 * (kAttnD + 2) * 4;     // warp partials
    static constexpr int kBufBytes = kRingBytes > kScratchBytes ? kRingBytes : kScratchBytes;
    static constexpr int kBarOff = kBufBytes;                           // mbarriers
    static constexpr int kListOff = kBarOff + NW * STAGES * 8 + 16;     // page list
    static size_t bytes(int sel_stride) { return 1024 + kListOff + (size_t)sel_stride * 8; }
};

// Compact the row's OWNED selected pages (global id j with j % stride == offset) into
// list[] as (physical block, valid tokens).  Order preserved.  Returns the count.
TS_DEV int build_page_list(const AttnParams &p, int row, int b, int L, int2 *list, int *wtot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int cnt = p.sel_count[row];
    const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
    int base = 0;
    for (int u0 = 0; u0 < cnt; u0 += blockDim.x) {
        const int u = u0 + threadIdx.x;
        int j = u < cnt ? ids[u] : -1;
        const bool own = j >= 0 && (j % p.stride) == p.offset;
        const unsigned ball = __ballot_sync(0xffffffffu, own);
        if (lane == 0) wtot[warp] = __popc(ball);
        __syncthreads();
        int before = base;
        for (int w = 0; w < warp; ++w) before += wtot[w];
        int total = 0;
        for (int w = 0; w < nw; ++w) total += wtot[w];
        if (own) {
            const int jl = j / p.stride;
            const int blk = p.page_table[(size_t)b * p.max_pages + jl];
            const int nv = min(p.S, L - j * p.S);
            list[before + __popc(ball & ((1u << lane) - 1))] = make_int2(blk, nv);
        }
        base += total;
        __syncthreads();
    }
    return base;
}

template <int TT, int NW, int STAGES>
__global__ void __launch_bounds__(NW * 32)
    attn_mma_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                    AttnParams p) {
    using SM = AttnSmem<TT, NW, STAGES>;
    constexpr int NT = TT / 8;  // 8-token sub-tiles per tile
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + SM::kBarOff;
    int2 *list = reinterpret_cast<int2 *>(smem + SM::kListOff);
    float *scratch = reinterpret_cast<float *>(smem);  // aliases the rings (used after drain)
    __shared__ int wtot[32];
    __shared__ int flag;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, t = lane & 3;
    if (threadIdx.x == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
        for (int i = 0; i < NW * STAGES; ++i) mbar_init(bar0 + 8 * i, 1);
        fence_mbar_init();
    }
    __syncthreads();
    const uint64_t pol = l2_policy_evict_first();
    const uint32_t ring = sbase + warp * STAGES * SM::kStageBytes;
    const uint32_t wbar = bar0 + warp * STAGES * 8;
    const int TPP = p.S / TT;
    const float sl2 = p.scale * kLog2e;
    uint32_t it = 0;  // tiles consumed by this warp so far (ring position / phase)

    for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        const int row = item / p.splits, split = item % p.splits;
        const int b = row / p.Hkv, g = row % p.Hkv;
        const int L = p.seq_lens[b];
        const int npages = build_page_list(p, row, b, L, list, wtot);
        const int ntiles = npages * TPP;
        const int t0 = (int)((long long)split * ntiles / p.splits);
        const int t1 = (int)((long long)(split + 1) * ntiles / p.splits);
        const int n = t1 - t0 > warp ? (t1 - t0 - warp + NW - 1) / NW : 0;  // my tiles

        // Q fragments: row gid <-> q head g*G + gid; k-slot permutation d = 16t + 4s + {0..3}
        uint32_t qa[8];
        {
            const bool live = gid < p.G;
            const uint16_t *qh = static_cast<const uint16_t *>(p.q) +
                                 ((size_t)b * p.Hq + g * p.G + (live ? gid : 0)) * kAttnD + 16 * t;
            const uint4 x0 = live ? ldg_v4(qh) : make_uint4(0, 0, 0, 0);
            const uint4 x1 = live ? ldg_v4(qh + 8) : make_uint4(0, 0, 0, 0);
            qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
            qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
        }

        auto issue = [&](int jt) {  // lane 0 only: TMA for my jt-th tile of this item
            const int tau = t0 + warp + jt * NW;
            const int2 pg = list[tau / TPP];
            const int y = (pg.x * p.Hkv + g) * p.S + (tau % TPP) * TT;
            const uint32_t slot = (it + jt) % STAGES;
            const uint32_t dst = ring + slot * SM::kStageBytes;
            const uint32_t bar = wbar + 8 * slot;
            fence_proxy_async();
            mbar_arrive_expect_tx(bar, SM::kStageBytes);
            tma_load_2d(dst, &tmK, 0, y, bar, pol);
            tma_load_2d(dst + SM::kTileBytes, &tmV, 0, y, bar, pol);
        };
        if (lane == 0)
            for (int jt = 0; jt < min(n, STAGES); ++jt) issue(jt);

        float m = kNegInf;  // running max (log2 domain) of head gid
        float lpart = 0.f;  // this thread's share of the softmax denominator
        float oacc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;

        for (int jt = 0; jt < n; ++jt) {
            const uint32_t slot = (it + jt) % STAGES;
            const uint32_t kb = ring + slot * SM::kStageBytes, vb = kb + SM::kTileBytes;
            mbar_wait(wbar + 8 * slot, ((it + jt) / STAGES) & 1);
            const int tau = t0 + warp + jt * NW;
            const int nv = min(TT, list[tau / TPP].y - (tau % TPP) * TT);  // valid tokens
            if (nv > 0) {
                if (nv < TT) {  // zero V rows past seq_len (their p is 0, but 0*NaN = NaN)
                    for (int c = lane; c < (TT - nv) * 8; c += 32)
                        sts_v4(vb + nv * kRowBytes + c * 16, make_uint4(0, 0, 0, 0));
                    __syncwarp();
                }
                // ---- S^T[head gid][token] = q . k  (bf16 MMA, fp32 accumulate)
                float sacc[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
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
                // ---- online softmax (log2 domain) over tokens nt*8 + 2t + {0,1}
                float x[NT][2];
                float tmax = kNegInf;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int tok = nt * 8 + 2 * t + e;
                        x[nt][e] = tok < nv ? sacc[nt][e] * sl2 : kNegInf;
                        tmax = fmaxf(tmax, x[nt][e]);
                    }
                tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
                tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
                const float mnew = fmaxf(m, tmax);  // finite: nv > 0 valid tokens
                const float corr = exp2f(m - mnew);
                m = mnew;
                float pr[NT][2];
                float psum = 0.f;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        pr[nt][e] = exp2f(x[nt][e] - mnew);
                        psum += pr[nt][e];
                    }
                lpart = lpart * corr + psum;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    oacc[j][0] *= corr;
                    oacc[j][1] *= corr;
                }
                // ---- O[head gid][d] += P . V  (tf32 MMA; k slot t <-> token 2t, t+4 <-> 2t+1)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int r0 = nt * 8 + 2 * t, r1 = r0 + 1;
                    const uint4 v0 = lds_v4(vb + r0 * kRowBytes + ((gid ^ (r0 & 7)) << 4));
                    const uint4 v1 = lds_v4(vb + r1 * kRowBytes + ((gid ^ (r1 & 7)) << 4));
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
            }
            __syncwarp();
            if (lane == 0 && jt + STAGES < n) issue(jt + STAGES);
        }
        it += n;

        // ---- warp partials -> CTA (scratch aliases the rings: all warps must be done)
        const float lrow = lpart + __shfl_xor_sync(0xffffffffu, lpart, 1);
        const float lsum = lrow + __shfl_xor_sync(0xffffffffu, lrow, 2);
        __syncthreads();
        float *ws = scratch + warp * 8 * (kAttnD + 2);  // [8 heads][D + 2]
        if (gid < p.G) {
            float *wr = ws + gid * (kAttnD + 2);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                wr[16 * t + j] = oacc[j][0];
                wr[16 * t + 8 + j] = oacc[j][1];
            }
            if (t == 0) {
                wr[kAttnD] = m;
                wr[kAttnD + 1] = lsum;
            }
        }
        __syncthreads();
        // combine the NW warps: thread -> (head h, 4 channels)
        const bool single = p.splits == 1;
        float *prow = p.part + ((size_t)row * p.splits + split) * 8 * kPS;
        for (int x = threadIdx.x; x < p.G * (kAttnD / 4); x += NW * 32) {
            const int h = x / (kAttnD / 4), d0 = (x % (kAttnD / 4)) * 4;
            float M = kNegInf;
            for (int w = 0; w < NW; ++w) M = fmaxf(M, scratch[(w * 8 + h) * (kAttnD + 2) + kAttnD]);
            float acc[4] = {0.f, 0.f, 0.f, 0.f}, l = 0.f;
            if (M != kNegInf) {
                for (int w = 0; w < NW; ++w) {
                    const float *wr = scratch + (w * 8 + h) * (kAttnD + 2);
                    const float mw = wr[kAttnD];
                    if (mw == kNegInf) continue;
                    const float f = exp2f(mw - M);
                    l += wr[kAttnD + 1] * f;
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[e] += wr[d0 + e] * f;
                }
            }
            if (single) {
                const size_t oh = (size_t)b * p.Hq + g * p.G + h;
                const float inv = l > 0.f ? 1.f / l : 0.f;
                *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                    make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
                if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
            } else {
                float *pr = prow + h * kPS;
                *reinterpret_cast<float4 *>(pr + d0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
                if (d0 == 0) {
                    pr[kAttnD] = M;
                    pr[kAttnD + 1] = l;
                }
            }
        }
        if (!single) {
            // ---- last CTA of the row merges the splits and re-arms the ticket
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) flag = atomicAdd(p.tickets + row, 1u) == unsigned(p.splits - 1);
            __syncthreads();
            if (flag) {
                __threadfence();
                const float *pbase = p.part + (size_t)row * p.splits * 8 * kPS;
                for (int x = threadIdx.x; x < p.G * (kAttnD / 4); x += NW * 32) {
                    const int h = x / (kAttnD / 4), d0 = (x % (kAttnD / 4)) * 4;
                    float M = kNegInf;
                    for (int s = 0; s < p.splits; ++s)
                        M = fmaxf(M, __ldcg(pbase + (s * 8 + h) * kPS + kAttnD));
                    float acc[4] = {0.f, 0.f, 0.f, 0.f}, l = 0.f;
                    if (M != kNegInf) {
                        for (int s = 0; s < p.splits; ++s) {
                            const float *pr = pbase + (s * 8 + h) * kPS;
                            const float ms = __ldcg(pr + kAttnD);
                            if (ms == kNegInf) continue;
                            const float f = exp2f(ms - M);
                            l += __ldcg(pr + kAttnD + 1) * f;
                            const float4 v = __ldcg(reinterpret_cast<const float4 *>(pr + d0));
                            acc[0] += v.x * f; acc[1] += v.y * f; acc[2] += v.z * f; acc[3] += v.w * f;
                        }
                    }
                    const size_t oh = (size_t)b * p.Hq + g * p.G + h;
                    const float inv = l > 0.f ? 1.f / l : 0.f;
                    *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                        make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
                    if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
                }
                if (threadIdx.x == 0) p.tickets[row] = 0u;
            }
        }
        __syncthreads();  // scratch / list reuse by the next item
    }
}

// ------------------------------------------------------------------ fp32 CUDA-core path
// grid = rows (b, g); block = 32 * min(G, 8) threads; warp w handles q heads w, w+8, ...
template <int D>
__global__ void __launch_bounds__(256) attn_simt_kernel(AttnParams p, const float *__restrict__ k_pool,
                                                        const float *__restrict__ v_pool) {
    constexpr int E = D / 32;  // elements per lane: d = lane + 32 e
    const int row = blockIdx.x;
    const int b = row / p.Hkv, g = row % p.Hkv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int L = p.seq_lens[b];
    const int cnt = p.sel_count[row];
    const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
    const float *q = static_cast<const float *>(p.q);
    for (int hh = warp; hh < p.G; hh += nwarps) {
        const size_t oh = (size_t)b * p.Hq + g * p.G + hh;
        float qv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) qv[e] = q[oh * D + lane + 32 * e];
        float m = kNegInf, l = 0.f, acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.f;
        for (int u = 0; u < cnt; ++u) {
            const int j = ids[u];
            if (j < 0 || j % p.stride != p.offset) continue;
            const int blk = p.page_table[(size_t)b * p.max_pages + j / p.stride];
            const int nv = min(p.S, L - j * p.S);
            for (int s = 0; s < nv; ++s) {
                const size_t base = (((size_t)blk * p.Hkv + g) * p.S + s) * D;
                float dot = 0.f;
#pragma unroll
                for (int e = 0; e < E; ++e) dot = fmaf(qv[e], k_pool[base + lane + 32 * e], dot);
                dot = warp_sum(dot);  // fixed tree: identical on all lanes
                const float a = dot * p.scale;
                const float mn = fmaxf(m, a);
                const float corr = expf(m - mn);
                const float pw = expf(a - mn);
                l = l * corr + pw;
#pragma unroll
                for (int e = 0; e < E; ++e) acc[e] = fmaf(pw, v_pool[base + lane + 32 * e], acc[e] * corr);
                m = mn;
            }
        }
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) p.o[oh * D + lane + 32 * e] = acc[e] * inv;
        if (p.lse && lane == 0) p.lse[oh] = l > 0.f ? m + logf(l) : kNegInf;
    }
}

// ------------------------------------------------------------------ LSE merge (API)
// part q of o_parts starts at q * so, of lse_parts at q * sl (elements).
__global__ void lse_merge_kernel(int parts, int rows, int d, const float *__restrict__ o_parts,
                                 const float *__restrict__ lse_parts, long long so, long long sl,
                                 float *__restrict__ o, float *__restrict__ lse) {
    const int r = blockIdx.x;
    float M = kNegInf;
    for (int q = 0; q < parts; ++q) M = fmaxf(M, lse_parts[q * sl + r]);
    float l = 0.f;
    if (M != kNegInf)
        for (int q = 0; q < parts; ++q) l += expf(lse_parts[q * sl + r] - M);
    const float tot = M != kNegInf ? M + logf(l) : kNegInf;
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
        float acc = 0.f;
        if (M != kNegInf)
            for (int q = 0; q < parts; ++q) {
                const float lp = lse_parts[q * sl + r];
                if (lp == kNegInf) continue;
                acc += expf(lp - tot) * o_parts[q * so + (size_t)r * d + i];
            }
        o[(size_t)r * d + i] = acc;
    }
    if (threadIdx.x == 0 && lse) lse[r] = tot;
}

}  // namespace ts
