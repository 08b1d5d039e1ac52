// sparse_attn.cuh — masked softmax attention over the selected pages (SparseAttn,
// PAPER.md:169-172; Alg. 1 Steps 3-4 "gather K/V of the selected pages, attention",
// PAPER.md:231-244), bf16 KV, head_dim 64, GQA group G <= 8.
//
// Split-K flash-decode with the split merged inside a thread-block cluster:
//  * grid = rows x C CTAs, cluster = the C CTAs of one row (b, kv head g); the row's
//    OWNED selected pages (global ids, sharding filter) are cut into 8-token "octets" and
//    the octets are dealt out in contiguous ranges to the C x W warps of the cluster;
//  * every warp streams its octets global -> registers with 128-bit loads, DP octets in
//    flight (software pipeline, no shared-memory staging, no cross-warp synchronisation
//    in the main loop): per octet a lane loads 32 B of K (token gid, channels
//    [16t, 16t+16)) and 2 x 16 B of V (tokens 2t, 2t+1, channels [8 gid, 8 gid + 8));
//  * S = Q K^T on mma.m16n8k16 (bf16 in, fp32 out; A rows = the G q heads, rows >= G
//    zero; channel permutation d = 16t + 4s + {0..3} so the 32 B of K feed all four
//    k-steps), fp32 online softmax in exp2, O^T += V^T P^T on mma.m16n8k8 with a hi + lo
//    bf16 P (reading R10; attn.cuh: the lane's two P values are its B fragment and its V
//    rows, the same tokens, form the A fragment by PRMT);
//  * tokens t >= seq_len are masked (score -inf, V zeroed: the tail of a partial page may
//    hold anything — reading R7);
//  * warp partials (o, m, l) merge in shared memory, CTA partials across the cluster
//    through distributed shared memory; the cluster writes o (fp32) and lse.
// With PDL (the fused step) everything up to the first read of the selection overlaps
// the tail of the score/select kernel: griddepcontrol.wait sits just before it.
#pragma once

#include <type_traits>

#include "attn.cuh"
#include "common.cuh"
#include "fp8.cuh"           // the FP8 tile consumer (F8 instantiation)
#include "score_select.cuh"  // cta_topk, block_scan (the candidate merge of ts_shard_attend)

namespace ts {

constexpr int kSsHistM = 2048;  // radix bins of the candidate merge



constexpr int kSaPart = 68;  // floats per (head) partial in smem: o[64], m, l, pad

template <int W>
struct SaSmem {
    // warp partials [W][8 heads][kSaPart] then the CTA partial [8][kSaPart]; page lists
    // (block element base, first token) follow dynamically.
    static constexpr int kWarpPart = 0;
    static constexpr int kCtaPart = W * 8 * kSaPart * 4;
    static constexpr int kPages = kCtaPart + 8 * kSaPart * 4;
    static size_t bytes(int max_pages) { return kPages + (size_t)max_pages * 8; }
};

template <int W, int DP>
__global__ void __launch_bounds__(W * 32, 512 / (W * 32)) sparse_attn_kernel(AttnParams p, int C) {
    using SM = SaSmem<W>;
    extern __shared__ __align__(16) uint8_t sa_smem[];
    float *wpart = reinterpret_cast<float *>(sa_smem + SM::kWarpPart);
    float *cpart = reinterpret_cast<float *>(sa_smem + SM::kCtaPart);
    int *s_base = reinterpret_cast<int *>(sa_smem + SM::kPages);  // [n_own] element base / 64
    int *s_tok = s_base + p.sel_stride;                             // [n_own] first token
    __shared__ int s_nown;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, t = lane & 3;
    const int rank = blockIdx.x % C, ncl = gridDim.x / C;
    const int rows = p.B * p.Hkv;
    // persistent over rows: cluster x handles rows x, x + clusters, ... (row order = the
    // selector's order, so the first rows it releases are the first ones attended)
    for (int row = blockIdx.x / C; row < rows; row += ncl) {
    unsigned long long *dts = p.dbg && blockIdx.x < 2048 && row < ncl ? p.dbg + blockIdx.x * 8 : nullptr;
#define SA_STAMP(e) \
    if (dts && threadIdx.x == 0) dts[e] = globaltimer();
    SA_STAMP(0);
    const int b = row / p.Hkv, g = row % p.Hkv;
    const int L = clamp_len(p.seq_lens[b], p.max_pages, p.stride, p.S);

    // ---- Q fragments (independent of the selection): q heads g*G + gid, channels [16t, +16)
    uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (gid < p.G) {
        const uint16_t *qr =
            static_cast<const uint16_t *>(p.q) + ((size_t)b * p.Hq + g * p.G + gid) * kAttnD + 16 * t;
        const uint4 x0 = ldg_nc_v4(qr), x1 = ldg_nc_v4(qr + 8);
        qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
        qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
    }
    if (dts && threadIdx.x == 0) dts[1] = globaltimer() + (qa[0] & 0u);  // q arrived
    pdl_wait();  // the selection may come from the previous kernel (two-kernel step)

    // ---- owned selected pages of the row -> (block base, first token), in id order
    const int cnt = __ldcg(p.sel_count + row);
    const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
    if (p.sel_blk) {  // fused step: the selector already resolved the blocks
        const int *blks = p.sel_blk + (size_t)row * p.sel_stride;
        for (int u = threadIdx.x; u < cnt; u += blockDim.x) {
            s_base[u] = (checked_block(__ldcg(blks + u), p.num_blocks) * p.Hkv + g) * p.S;
            s_tok[u] = __ldcg(ids + u) * p.S;
        }
        if (threadIdx.x == 0) s_nown = cnt;
    } else if (p.stride == 1) {
        for (int u = threadIdx.x; u < cnt; u += blockDim.x) {
            const int j = __ldg(ids + u);
            const int blk = checked_block(__ldg(p.page_table + (size_t)b * p.max_pages + j), p.num_blocks);
            s_base[u] = (blk * p.Hkv + g) * p.S;  // in 64-channel rows
            s_tok[u] = j * p.S;
        }
        if (threadIdx.x == 0) s_nown = cnt;
    } else {  // sequence sharding: keep the pages this rank owns (warp 0 compacts in order)
        if (warp == 0) {
            int n = 0;
            for (int u0 = 0; u0 < cnt; u0 += 32) {
                const int u = u0 + lane;
                const int j = u < cnt ? __ldg(ids + u) : -1;
                const bool own = j >= 0 && j % p.stride == p.offset;
                const unsigned m = __ballot_sync(0xffffffffu, own);
                if (own) {
                    const int pos = n + __popc(m & ((1u << lane) - 1u));
                    const int blk = checked_block(__ldg(p.page_table + (size_t)b * p.max_pages + j / p.stride), p.num_blocks);
                    s_base[pos] = (blk * p.Hkv + g) * p.S;
                    s_tok[pos] = j * p.S;
                }
                n += __popc(m);
            }
            if (lane == 0) s_nown = n;
        }
    }
    __syncthreads();
    SA_STAMP(2);
    const int n_own = s_nown;
    // octets per page; a page of S = 4 tokens is one half-filled octet (rows >= 4 of it
    // belong to other (block, head) runs: never loaded, masked like tokens past seq_len)
    const int ops = p.S >= 8 ? p.S >> 3 : 1;
    const int orows = p.S >= 8 ? 8 : p.S;  // token rows per octet
    const int n_oct = n_own * ops;
    const int nw = C * W, wg = rank * W + warp;
    const int o0 = (int)((long long)n_oct * wg / nw), o1 = (int)((long long)n_oct * (wg + 1) / nw);

    const uint16_t *kp = static_cast<const uint16_t *>(p.k_pool);
    const uint16_t *vp = static_cast<const uint16_t *>(p.v_pool);
    const float sl2 = p.scale * kLog2e;
    float m = kNegInf, lp = 0.f;
    float oacc[4][4];  // O^T: channels (8 gid + 2 db, + 1) x heads (2t, 2t + 1) (attn.cuh)
#pragma unroll
    for (int j = 0; j < 4; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;

    // octet o -> element offset of its first token row, and its first global token
    auto octet_addr = [&](int o, int &tok0) -> size_t {
        const int u = o / ops, sub = o - u * ops;
        tok0 = s_tok[u] + 8 * sub;
        return ((size_t)s_base[u] + 8 * sub) * kAttnD;
    };
    uint4 kb[DP][2], vb[DP][2];
    int tk[DP];
    auto issue = [&](int j, int o) {
        if (o < o1) {
            const size_t e = octet_addr(o, tk[j]);
            const uint16_t *kr = kp + e + gid * kAttnD + 16 * t;
            kb[j][0] = gid < orows ? ldg_nc_v4(kr) : make_uint4(0, 0, 0, 0);
            kb[j][1] = gid < orows ? ldg_nc_v4(kr + 8) : make_uint4(0, 0, 0, 0);
            const uint16_t *vr = vp + e + (2 * t) * kAttnD + 8 * gid;
            vb[j][0] = 2 * t < orows ? ldg_nc_v4(vr) : make_uint4(0, 0, 0, 0);
            vb[j][1] = 2 * t + 1 < orows ? ldg_nc_v4(vr + kAttnD) : make_uint4(0, 0, 0, 0);
        }
    };
#pragma unroll
    for (int j = 0; j < DP; ++j) issue(j, o0 + j);

    for (int ob = o0; ob < o1; ob += DP) {
#pragma unroll
        for (int j = 0; j < DP; ++j) {
            const int o = ob + j;
            if (o >= o1) break;
            // ---- S^T tile: heads (rows gid) x tokens (2t, 2t+1) of the octet
            float s[4] = {0.f, 0.f, 0.f, 0.f};
            mma_bf16_16816(s, qa[0], 0u, qa[1], 0u, kb[j][0].x, kb[j][0].y);
            mma_bf16_16816(s, qa[2], 0u, qa[3], 0u, kb[j][0].z, kb[j][0].w);
            mma_bf16_16816(s, qa[4], 0u, qa[5], 0u, kb[j][1].x, kb[j][1].y);
            mma_bf16_16816(s, qa[6], 0u, qa[7], 0u, kb[j][1].z, kb[j][1].w);
            const int tok = tk[j] + 2 * t;
            const bool ok0 = tok < L && 2 * t < orows, ok1 = tok + 1 < L && 2 * t + 1 < orows;
            const float x0 = ok0 ? s[0] * sl2 : kNegInf;
            const float x1 = ok1 ? s[1] * sl2 : kNegInf;
            float tmax = fmaxf(x0, x1);
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
            const float mnew = fmaxf(m, tmax);
            // an octet past seq_len (tail of a partial page) has no valid token: keep the
            // exponents finite (mref) so it contributes exactly nothing
            const float mref = mnew == kNegInf ? 0.f : mnew;
            const float corr = exp2f(m - mref);  // m = -inf -> 0
            m = mnew;
            const float p0 = exp2f(x0 - mref), p1 = exp2f(x1 - mref);
            lp = lp * corr + p0 + p1;
            const uint4 v0 = ok0 ? vb[j][0] : make_uint4(0, 0, 0, 0);
            const uint4 v1 = ok1 ? vb[j][1] : make_uint4(0, 0, 0, 0);
            issue(j, o + DP);  // refill this slot while the tensor cores work
            ot_rescale(oacc, corr, t);
            ot_pv_octet_bf16(oacc, v0, v1, p0, p1);
        }
    }

    if (dts && threadIdx.x == 0) dts[3] = globaltimer() + (__float_as_uint(oacc[0][0]) & 0u);
    // ---- warp partial -> smem: heads 2t, 2t+1 x channels 8 gid + {0..7}; m, l of head gid
    lp += __shfl_xor_sync(0xffffffffu, lp, 1);
    lp += __shfl_xor_sync(0xffffffffu, lp, 2);
    ot_store(wpart + warp * 8 * kSaPart, kSaPart, oacc, gid, t, p.G);
    if (gid < p.G && t == 0) {
        float *wr = wpart + (warp * 8 + gid) * kSaPart;
        wr[kAttnD] = m;
        wr[kAttnD + 1] = lp;
    }
    __syncthreads();
    // ---- CTA merge: thread -> (head, 4 channels)
    for (int x = threadIdx.x; x < p.G * 16; x += blockDim.x) {
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
        float *cr = cpart + h * kSaPart;
        *reinterpret_cast<float4 *>(cr + d0) = acc;
        if (d0 == 0) {
            cr[kAttnD] = M;
            cr[kAttnD + 1] = l;
        }
    }
    // ---- cluster merge through DSMEM: CTA `rank` finalises outputs x = rank, rank + C, ...
    cg::cluster_group cl = cg::this_cluster();
    SA_STAMP(4);
    if (C > 1) cl.sync(); else __syncthreads();
    SA_STAMP(5);
    for (int x = rank * blockDim.x + threadIdx.x; x < p.G * 16; x += C * blockDim.x) {
        const int h = x >> 4, d0 = (x & 15) * 4;
        float M = kNegInf;
        for (int r = 0; r < C; ++r) {
            const float *cr = C > 1 ? cl.map_shared_rank(cpart, r) : cpart;
            M = fmaxf(M, cr[h * kSaPart + kAttnD]);
        }
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float l = 0.f;
        if (M != kNegInf)
            for (int r = 0; r < C; ++r) {
                const float *cr = (C > 1 ? cl.map_shared_rank(cpart, r) : cpart) + h * kSaPart;
                const float mr = cr[kAttnD];
                const float f = mr == kNegInf ? 0.f : exp2f(mr - M);
                l += cr[kAttnD + 1] * f;
                const float4 v = *reinterpret_cast<const float4 *>(cr + d0);
                acc.x += v.x * f; acc.y += v.y * f; acc.z += v.z * f; acc.w += v.w * f;
            }
        const size_t oh = (size_t)b * p.Hq + g * p.G + h;
        const float inv = l > 0.f ? 1.f / l : 0.f;
        *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
            make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
    }
    SA_STAMP(6);
    if (C > 1) cl.sync(); else __syncthreads();  // partials / page lists free for the next row
    SA_STAMP(7);
    }  // row loop
}

// ---------------------------------------------------------------------------------------
// TMA variant (S a multiple of 16): one (row, split) per CTA.  A producer warp resolves the
// CTA's pages and streams [16 x 64] K and V tiles (2-D tensor maps over the pools, 128-byte
// swizzle, L2 evict-first) into an R-stage shared-memory ring; W consumer warps take tiles
// round-robin (S = Q K^T on m16n8k16, online softmax, O^T += V^T P^T on m16n8k16, hi + lo bf16 P) reading
// the swizzled rows conflict-free; partials merge as in sparse_attn_kernel.  Bytes in
// flight are bounded by shared memory (R x 4 KB per CTA), not by registers.
template <int W, int R>
struct SatSmem {
    static constexpr int kTile = 16 * kRowBytes;                  // 2 KB
    static constexpr int kStage = 2 * kTile;                      // K + V (FP8: SatSmemF8)
    static constexpr int kRing = 0;
    static constexpr int kWarpPart = kRing + R * kStage;          // [W][8][kSaPart] fp32
    static constexpr int kCtaPart = kWarpPart + W * 8 * kSaPart * 4;
    static constexpr int kInfo = kCtaPart + 8 * kSaPart * 4;      // [R] int2 (token0, valid)
    static constexpr int kBars = kInfo + R * 8;
    static constexpr int kPages = kBars + 2 * R * 8;              // [sel_stride] int2 (row0, tok0)
    static size_t bytes(int sel_stride) { return 1024 + kPages + (size_t)sel_stride * 8; }
};

// FP8 stages: the K and V sub-page records (2 x 1040 B), so twice the stages fit the bytes
template <int W, int R>
struct SatSmemF8 : SatSmem<W, R> {
    static constexpr int kStage = 2 * kF8Rec;
    static constexpr int kRing = 0;
    static constexpr int kWarpPart = kRing + R * kStage;
    static constexpr int kCtaPart = kWarpPart + W * 8 * kSaPart * 4;
    static constexpr int kInfo = kCtaPart + 8 * kSaPart * 4;
    static constexpr int kBars = kInfo + R * 8;
    static constexpr int kPages = kBars + 2 * R * 8;
    static size_t bytes(int sel_stride) { return 1024 + kPages + (size_t)sel_stride * 8; }
};
template <int W, int R, bool F8>
using SatSmemT = typename std::conditional<F8, SatSmemF8<W, R>, SatSmem<W, R>>::type;

// F8: FP8 KV (reading R21) — a stage holds the tile's K and V sub-page records (codes +
// exponents, 1040 B each, 1-D bulk copies), consumed by f8_attend_tile (fp8.cuh).
template <int W, int R, bool F8 = false>
__global__ void __launch_bounds__((W + 1) * 32, W >= 8 ? 2 : 4) sparse_attn_tma_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, AttnParams p,
    int C) {
    using SM = SatSmemT<W, R, F8>;
    static_assert(R % W == 0, "stage -> consumer warp must be fixed");
    extern __shared__ uint8_t sat_raw[];
    // 1024-byte aligned (TMA swizzle atoms) by pointer arithmetic on the __shared__ array
    // itself, so the compiler keeps the shared state space (LDS / ATOMS, not generic LD / ATOM)
    uint8_t *smem = sat_raw + ((1024u - (smem_u32(sat_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(smem);
    const uint32_t full0 = sb + SM::kBars, empty0 = full0 + 8 * R;
    float *wpart = reinterpret_cast<float *>(smem + SM::kWarpPart);
    float *cpart = reinterpret_cast<float *>(smem + SM::kCtaPart);
    int2 *info = reinterpret_cast<int2 *>(smem + SM::kInfo);
    int2 *pages = reinterpret_cast<int2 *>(smem + SM::kPages);
    __shared__ int s_nown;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row = blockIdx.x / C, rank = blockIdx.x % C;
    const int b = row / p.Hkv, g = row % p.Hkv;
    unsigned long long *dts = p.dbg && blockIdx.x < 2048 ? p.dbg + blockIdx.x * 8 : nullptr;
    if (dts && threadIdx.x == 0) dts[0] = globaltimer();
    pdl_launch_dependents();  // the next step's selector may start its prologue
    if (threadIdx.x == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
        for (int i = 0; i < R; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        fence_mbar_init();
    }
    const int L = clamp_len(p.seq_lens[b], p.max_pages, p.stride, p.S);
    // ---- Q fragments (consumers; independent of the selection)
    const int gid = lane >> 2, t = lane & 3;
    uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (warp < W && gid < p.G) {
        const uint16_t *qr =
            static_cast<const uint16_t *>(p.q) + ((size_t)b * p.Hq + g * p.G + gid) * kAttnD + 16 * t;
        const uint4 x0 = ldg_nc_v4(qr), x1 = ldg_nc_v4(qr + 8);
        qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
        qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
    }
    // ---- wait for the selection (PDL), then resolve the pages this CTA attends
    pdl_wait();
    __syncthreads();
    if (dts && threadIdx.x == 0) dts[1] = globaltimer();
    if (p.dense) {
        // FullCache baseline (dense attention): every page
        // j < P_b of the row, in order, through the same gather + attention machinery
        const int P = (L + p.S - 1) / p.S;
        for (int u = threadIdx.x; u < P; u += blockDim.x) {
            const int blk = checked_block(__ldg(p.page_table + (size_t)b * p.max_pages + u), p.num_blocks);
            pages[u] = make_int2((blk * p.Hkv + g) * p.S, u * p.S);
        }
        if (threadIdx.x == 0) s_nown = P;
    } else if (p.cand_scores) {
        // ts_shard_attend: the global top-k over the ranks' candidates (the exchange step of
        // sequence sharding), merged here instead of by a separate kernel.
        // The candidates are placed in ascending GLOBAL page id order (a bitmap over the
        // row's pages + a prefix count: ids are unique), so cta_topk's lower-index tie-break
        // is the lower-global-id rule (reading R6) and the output comes out ascending.
        // Scratch lives in the TMA ring, which is idle until the producer starts.
        const int Pg = (L + p.S - 1) / p.S;  // global pages of the row
        const int nw = (Pg + 31) >> 5;
        const int ncand = p.cand_parts * p.cand_k;
        const int n4 = (ncand + 3) & ~3;
        uint32_t *mkeys = reinterpret_cast<uint32_t *>(smem + SM::kRing);
        int *mids = reinterpret_cast<int *>(mkeys + n4);
        const int nw4 = (nw + 3) & ~3;  // 16-byte aligned sub-arrays (cta_topk reads int4 / uint4)
        uint32_t *bits = reinterpret_cast<uint32_t *>(mids + n4);
        int *wpre = reinterpret_cast<int *>(bits + nw4);
        int *mhist = wpre + nw4;
        int *mred = mhist + kSsHistM;
        uint32_t *mcand = reinterpret_cast<uint32_t *>(mred + 64);
        int *msel = reinterpret_cast<int *>(mcand + 2 * 64);
        constexpr int NT = (W + 1) * 32;
        // the candidates are read from L2 once, all of a thread's loads in flight together, and
        // kept in registers for the placement below (up to kCpt per thread; more: two passes)
        constexpr int kCpt = 8;
        const bool inreg = ncand <= kCpt * NT;
        int rid[kCpt];
        float rsc[kCpt];
        if (inreg) {
#pragma unroll
            for (int j = 0; j < kCpt; ++j) {
                const int e = threadIdx.x + j * NT;
                rid[j] = -1;
                rsc[j] = kNegInf;
                if (e < ncand) {
                    const size_t at = (size_t)(e / p.cand_k) * p.cand_part_stride + (size_t)row * p.cand_k + e % p.cand_k;
                    rid[j] = __ldcg(p.cand_ids + at);
                    rsc[j] = __ldcg(p.cand_scores + at);
                }
            }
        }
        for (int i = threadIdx.x; i < nw; i += NT) bits[i] = 0u;
        for (int i = threadIdx.x; i < kSsHistM; i += NT) mhist[i] = 0;
        __syncthreads();
        if (inreg) {
#pragma unroll
            for (int j = 0; j < kCpt; ++j)
                if (rsc[j] != kNegInf && rid[j] >= 0 && rid[j] < Pg) atomicOr(&bits[rid[j] >> 5], 1u << (rid[j] & 31));
        } else {
            for (int e = threadIdx.x; e < ncand; e += NT) {
                const size_t at = (size_t)(e / p.cand_k) * p.cand_part_stride + (size_t)row * p.cand_k + e % p.cand_k;
                const int id = __ldcg(p.cand_ids + at);
                if (__ldcg(p.cand_scores + at) != kNegInf && id >= 0 && id < Pg) atomicOr(&bits[id >> 5], 1u << (id & 31));
            }
        }
        __syncthreads();
        {  // exclusive prefix of the word popcounts (contiguous runs of words per thread)
            const int per = (nw + NT - 1) / NT, w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
            int c = 0;
            for (int w = w0; w < w1; ++w) c += __popc(bits[w]);
            int tot;
            int before = block_scan<NT>(c, mred, &tot);
            for (int w = w0; w < w1; ++w) {
                wpre[w] = before;
                before += __popc(bits[w]);
            }
            if (threadIdx.x == 0) mred[63] = tot;
        }
        __syncthreads();
        const int nlive = mred[63];
        uint32_t kmn = 0xffffffffu, kmx = 0u;
        auto place = [&](int id, float sv) {
            if (sv != kNegInf && id >= 0 && id < Pg) {
                const int pos = wpre[id >> 5] + __popc(bits[id >> 5] & ((1u << (id & 31)) - 1u));
                const uint32_t key = score_key(sv);
                mkeys[pos] = key;
                mids[pos] = id;
                kmn = min(kmn, key);
                kmx = max(kmx, key);
            }
        };
        if (inreg) {
#pragma unroll
            for (int j = 0; j < kCpt; ++j) place(rid[j], rsc[j]);
        } else {
            for (int e = threadIdx.x; e < ncand; e += NT) {
                const size_t at = (size_t)(e / p.cand_k) * p.cand_part_stride + (size_t)row * p.cand_k + e % p.cand_k;
                place(__ldcg(p.cand_ids + at), __ldcg(p.cand_scores + at));
            }
        }
        for (int i = nlive + threadIdx.x; i < n4; i += NT) mkeys[i] = 0u;
        block_minmax<NT>(kmn, kmx, mred);  // (barriers inside)
        const int kk = cta_topk<NT, 0, 11>(mkeys, nlive, p.cand_k, kmn, kmx, mhist, mred, mcand,
                                           [&](int pos, int i) { msel[pos] = mids[i]; });
        __syncthreads();
        if (rank == 0) {  // the global selection (identical on every rank)
            int *out = p.sel_out ? p.sel_out + (size_t)row * p.cand_k : nullptr;
            for (int i = threadIdx.x; out && i < p.cand_k; i += NT) out[i] = i < kk ? msel[i] : -1;
            if (p.sel_cnt_out && threadIdx.x == 0) p.sel_cnt_out[row] = kk;
        }
        if (warp == W) {  // owned pages, compacted in id order (two rounds' page-table loads at once)
            int n = 0;
            for (int u0 = 0; u0 < kk; u0 += 64) {
                int j[2], blk[2];
                bool own[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u = u0 + 32 * h + lane;
                    j[h] = u < kk ? msel[u] : -1;
                    own[h] = j[h] >= 0 && j[h] % p.stride == p.offset;
                    blk[h] = own[h] ? __ldg(p.page_table + (size_t)b * p.max_pages + j[h] / p.stride) : 0;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const unsigned m = __ballot_sync(0xffffffffu, own[h]);
                    if (own[h])
                        pages[n + __popc(m & ((1u << lane) - 1u))] =
                            make_int2((checked_block(blk[h], p.num_blocks) * p.Hkv + g) * p.S, j[h] * p.S);
                    n += __popc(m);
                }
            }
            if (lane == 0) s_nown = n;
        }
        fence_proxy_async();  // every thread: its generic writes to the ring scratch precede the TMA fills
    } else if (p.stride == 1) {
        // every selected page is owned: all threads resolve entries in parallel (one load
        // round for the ids / blocks, one more for the page table when not pre-resolved)
        const int cnt = __ldcg(p.sel_count + row);
        const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
        const int *blks = p.sel_blk ? p.sel_blk + (size_t)row * p.sel_stride : nullptr;
        for (int u = threadIdx.x; u < cnt; u += blockDim.x) {
            const int j = __ldcg(ids + u);
            const int blk = checked_block(blks ? __ldcg(blks + u) : __ldg(p.page_table + (size_t)b * p.max_pages + j), p.num_blocks);
            pages[u] = make_int2((blk * p.Hkv + g) * p.S, j * p.S);
        }
        if (threadIdx.x == 0) s_nown = cnt;
    } else if (warp == W) {  // sequence sharding: owned pages, compacted in id order
        const int cnt = __ldcg(p.sel_count + row);
        const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
        int n = 0;
        for (int u0 = 0; u0 < cnt; u0 += 32) {
            const int u = u0 + lane;
            const int j = u < cnt ? __ldcg(ids + u) : -1;
            const bool own = j >= 0 && j % p.stride == p.offset;
            const unsigned m = __ballot_sync(0xffffffffu, own);
            if (own) {
                const int blk = checked_block(__ldg(p.page_table + (size_t)b * p.max_pages + j / p.stride), p.num_blocks);
                pages[n + __popc(m & ((1u << lane) - 1u))] = make_int2((blk * p.Hkv + g) * p.S, j * p.S);
            }
            n += __popc(m);
        }
        if (lane == 0) s_nown = n;
    }
    __syncthreads();
    const int tpp = p.S >> 4;                 // tiles per page
    const int ntile = s_nown * tpp;
    const int t0 = ntile * rank / C, t1 = ntile * (rank + 1) / C;  // < 2^31: check_layout bounds a row
    if (dts && threadIdx.x == 0) dts[2] = globaltimer();

    // stage i of this CTA's tiles -> slot i % R, consumed by warp i % W (R % W == 0), which
    // re-issues the slot with stage i + R right after consuming it: W issuing warps per CTA
    // (one issuing lane caps a CTA's gather of small tiles at ~20 GB/s: scripts/gatherbench.cu)
    const uint64_t pol = l2_policy_evict_first();
    const int ntl = t1 - t0;
    auto tok0_of = [&](int i) {
        const int tl = t0 + i, u = tl / tpp;
        return pages[u].y + 16 * (tl - u * tpp);
    };
    auto issue = [&](int i, int kv) {  // part kv (0 = K, 1 = V) of stage i
        const int st = i % R, tl = t0 + i, u = tl / tpp, sub = tl - u * tpp;
        const int2 pg = pages[u];
        const uint32_t dst = sb + SM::kRing + st * SM::kStage;
        if constexpr (F8) {  // the tile's K / V sub-page record (codes + exponents)
            const size_t rec = (size_t)(pg.x >> 4) + sub;
            bulk_load_hint(dst + kv * kF8Rec, static_cast<const uint8_t *>(kv ? p.v_pool : p.k_pool) + rec * kF8Rec,
                           kF8Rec, full0 + 8 * st, pol);
        } else {
            tma_load_2d(dst + kv * SM::kTile, kv ? &tmV : &tmK, 0, pg.x + 16 * sub, full0 + 8 * st, pol);
        }
    };
    if (warp == W) {
        // ================================ producer ================================
        // the first R stages, two lanes (K, V) per stage in parallel
        const int i = lane >> 1;
        if (i < R && i < ntl) {
            if ((lane & 1) == 0) mbar_arrive_expect_tx(full0 + 8 * i, SM::kStage);
            issue(i, lane & 1);
        }
    } else if constexpr (F8) {
        // ================================ consumers (FP8) ==========================
        uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
        if (gid < p.G) {
            const uint16_t *qr =
                static_cast<const uint16_t *>(p.q) + ((size_t)b * p.Hq + g * p.G + gid) * kAttnD + 16 * t;
            x0 = ldg_nc_v4(qr);
            x1 = ldg_nc_v4(qr + 8);
        }
        const F8Q fq = f8_q_prep(x0, x1, p.scale * kLog2e);
        F8Acc acc;
        for (int i = warp; i < ntl; i += W) {
            const int st = i % R;
            mbar_wait(full0 + 8 * st, (i / R) & 1);
            const uint32_t kb = sb + SM::kRing + st * SM::kStage;
            f8_attend_tile(acc, fq, kb, kb + kF8Rec, tok0_of(i), L, gid, t);
            __syncwarp();
            if (lane < 2 && i + R < ntl) {  // refill this warp's slot with stage i + R
                fence_proxy_async();
                if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * st, SM::kStage);
                issue(i + R, lane);
            }
        }
        f8_store_partial(wpart + warp * 8 * kSaPart, kSaPart, acc, gid, t, p.G);
    } else {
        // ================================ consumers ===============================
        const float sl2 = p.scale * kLog2e;
        float m = kNegInf, lp = 0.f;
        float oacc[4][4];  // O^T: channels (8 gid + 2 db, + 1) x heads (2t, 2t + 1) (attn.cuh)
#pragma unroll
        for (int j = 0; j < 4; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
        for (int i = warp; i < ntl; i += W) {
            const int st = i % R;
            const int tok0 = tok0_of(i);
            mbar_wait(full0 + 8 * st, (i / R) & 1);
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
            ot_rescale(oacc, corr, t);
            uint4 vr[2][2];
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    const int q = nt * 8 + 2 * t + q2;
                    const uint4 v = lds_v4(vb + q * kRowBytes + ((gid ^ (q & 7)) << 4));
                    vr[nt][q2] = tok0 + q < L ? v : make_uint4(0, 0, 0, 0);  // past seq_len: may be anything
                }
            ot_pv_tile_bf16(oacc, vr, pr);
            __syncwarp();
            if (lane < 2 && i + R < ntl) {  // refill this warp's slot with stage i + R
                fence_proxy_async();
                if (lane == 0) mbar_arrive_expect_tx(full0 + 8 * st, SM::kStage);
                issue(i + R, lane);
            }
        }
        // ---- warp partial: heads 2t, 2t+1 x channels 8 gid + {0..7}; m, l of head gid
        lp += __shfl_xor_sync(0xffffffffu, lp, 1);
        lp += __shfl_xor_sync(0xffffffffu, lp, 2);
        ot_store(wpart + warp * 8 * kSaPart, kSaPart, oacc, gid, t, p.G);
        if (gid < p.G && t == 0) {
            float *wr = wpart + (warp * 8 + gid) * kSaPart;
            wr[kAttnD] = m;
            wr[kAttnD + 1] = lp;
        }
    }
    __syncthreads();
    if (dts && threadIdx.x == 0) dts[3] = globaltimer();
    // ---- CTA merge of the W warp partials (C == 1: straight to o / lse)
    for (int x = threadIdx.x; x < p.G * 16; x += blockDim.x) {
        const int h = x >> 4, d0 = (x & 15) * 4;
        float mw[W];
#pragma unroll
        for (int w = 0; w < W; ++w) mw[w] = wpart[(w * 8 + h) * kSaPart + kAttnD];
        float M = kNegInf;
#pragma unroll
        for (int w = 0; w < W; ++w) M = fmaxf(M, mw[w]);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float l = 0.f;
        if (M != kNegInf) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const float *wr = wpart + (w * 8 + h) * kSaPart;
                const float f = mw[w] == kNegInf ? 0.f : exp2f(mw[w] - M);
                l += wr[kAttnD + 1] * f;
                const float4 v = *reinterpret_cast<const float4 *>(wr + d0);
                acc.x += v.x * f; acc.y += v.y * f; acc.z += v.z * f; acc.w += v.w * f;
            }
        }
        if (C == 1) {
            const size_t oh = (size_t)b * p.Hq + g * p.G + h;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
            if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
        } else {  // this CTA's partial -> global workspace [rows][C][8][kPS]
            float *pr = p.part + (((size_t)row * C + rank) * 8 + h) * kPS;
            *reinterpret_cast<float4 *>(pr + d0) = acc;
            if (d0 == 0) {
                pr[kAttnD] = M;
                pr[kAttnD + 1] = l;
            }
        }
    }
    if (C > 1) {
        // ---- split merge: the last CTA of the row (ticket) combines the C partials from L2
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0) s_last = atom_add_acq_rel_gpu(p.tickets + row, 1u) == unsigned(C - 1);
        __syncthreads();
        if (s_last) {
            constexpr int kMaxC = 16;
            const float *pb = p.part + (size_t)row * C * 8 * kPS;
            for (int x = threadIdx.x; x < p.G * 16; x += blockDim.x) {
                const int h = x >> 4, d0 = (x & 15) * 4;
                float mr[kMaxC];
#pragma unroll
                for (int r = 0; r < kMaxC; ++r)
                    mr[r] = r < C ? __ldcg(pb + (r * 8 + h) * kPS + kAttnD) : kNegInf;
                float M = kNegInf;
#pragma unroll
                for (int r = 0; r < kMaxC; ++r) M = fmaxf(M, mr[r]);
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                float l = 0.f;
                if (M != kNegInf) {
#pragma unroll
                    for (int r0 = 0; r0 < kMaxC; r0 += 4) {
                        if (r0 >= C) break;
                        float lq[4];
                        float4 vq[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float *pr = pb + ((r0 + e) * 8 + h) * kPS;
                            lq[e] = r0 + e < C ? __ldcg(pr + kAttnD + 1) : 0.f;
                            vq[e] = r0 + e < C ? __ldcg(reinterpret_cast<const float4 *>(pr + d0))
                                               : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float f = mr[r0 + e] == kNegInf ? 0.f : exp2f(mr[r0 + e] - M);
                            l += lq[e] * f;
                            acc.x += vq[e].x * f; acc.y += vq[e].y * f; acc.z += vq[e].z * f; acc.w += vq[e].w * f;
                        }
                    }
                }
                const size_t oh = (size_t)b * p.Hq + g * p.G + h;
                const float inv = l > 0.f ? 1.f / l : 0.f;
                *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                    make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
                if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
            }
            if (threadIdx.x == 0) p.tickets[row] = 0u;  // re-armed for the next launch
        }
    }
    if (dts && threadIdx.x == 0) dts[7] = globaltimer();
}

}  // namespace ts
