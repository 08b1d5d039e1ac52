// step_cluster.cuh — the bf16 decode step (Alg. 1; "integrates page
// scoring, sparse memory access, and masked attention in a single pass") as ONE
// kernel: a thread-block cluster of C CTAs per row (b, kv head g) does all four steps.
//
//  1. score (Eq. 2): each CTA streams a contiguous chunk of the row's metadata records with
//     1-D bulk copies into an 8 KB-stage mbarrier ring; 4 consumer warps compute the
//     [m | M] x [q^- ; q^+] products on mma.m16n8k16 and the group max (reading R9);
//  2. select (TopK): the chunk keys are all-gathered into every CTA's shared memory (DSMEM
//     remote stores, one cluster barrier); every CTA runs the same exact CTA-wide top-K
//     (cta_topk, score_select.cuh) and keeps only the (tile row, first token) entries of
//     its own share of the ascending selection — no list broadcast, no second barrier;
//  3. gather: each CTA's producer streams its share's [16 x 64] K and V tiles with 2-D TMA
//     (128-byte swizzle) into the SAME ring, now as 4 KB stages;
//  4. attend: consumers run S = Q K^T (mma.m16n8k16), the fp32 online softmax and
//     O^T += V^T P^T (mma.m16n8k16, hi + lo bf16 P — R10; attn.cuh) per tile, with the q fragments already in
//     shared memory from step 1; warp partials merge in smem, the C CTA partials of a row
//     in the cluster leader's shared memory (DSM instantiation: DSMEM stores, one cluster
//     arrive / wait) or through an L2 workspace (last CTA by atomic ticket).
// No kernel boundary, no PDL gap, no second page-list lookup: the step is one launch.
#pragma once
#include "attn.cuh"
#include "common.cuh"
#include "fp8.cuh"
#include "score_select.cuh"
#include "sparse_attn.cuh"

namespace ts {

template <int W, int R>
struct ScSmem {
    static constexpr int NT = (W + 1) * 32;
    static constexpr int kRing = 0;                                 // R x 8 KB = 2R x 4 KB
    static constexpr int kQ = kRing + R * kSsStageBytes;           // [8][64] bf16
    static constexpr int kHist = kQ + 8 * kRowBytes;                // [2048] int
    static constexpr int kRed = kHist + kSsHist * 4;                // [64] int
    static constexpr int kWarpPart = kRed + 64 * 4;                 // [W][8][kSaPart] fp32
    static constexpr int kBars = (kWarpPart + W * 8 * kSaPart * 4 + 7) / 8 * 8;  // mfull,mempty[R]; afull,aempty[2R]; q; pt
    static constexpr int kSel = (kBars + (6 * R + 2) * 8 + 15) / 16 * 16;  // [kmax] int2
    __host__ __device__ static size_t scores_off(int kmax) { return ((size_t)kSel + (size_t)kmax * 8 + 127) / 128 * 128; }
    // scores [cap] fp32 (cap = the row, or only this CTA's chunk for the two-level select,
    // flag bit 1), then the page-table row [mp4] (flag bit 0), then the two-level candidates
    // [C * kmax] keys + ids (flag bit 1)
    __host__ __device__ static int score_cap(int max_pages, int flags, int chunk) {
        return (flags & 2) ? ((chunk + 3) & ~3) : ((max_pages + 3) & ~3);
    }
    // ... then the leader's merge area for the C CTA partials [C][8][kPS] fp32 (flag bit 2)
    static size_t bytes(int kmax, int max_pages, int flags, int C, int chunk) {
        const size_t mp4 = (max_pages + 3) & ~3;
        return scores_off(kmax) + (size_t)score_cap(max_pages, flags, chunk) * 4 +
               ((flags & 1) ? mp4 * 4 : 0) + ((flags & 2) ? (size_t)C * kmax * 8 : 0) +
               ((flags & 4) && C > 1 ? (size_t)C * 8 * kPS * 4 : 0) + 16;
    }
};

// FP8 KV (F8, reading R21): an attention stage holds the tile's K and V sub-page records
// (16 code rows + 16 exponent bytes each, 1040 B, one 1-D bulk copy apiece).
constexpr int kF8Stage = 2 * kF8Rec;

template <int W, int R, bool DSM, bool APP, bool F8 = false>
__global__ void __launch_bounds__((W + 1) * 32, 4) decode_cluster_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
    ScoreSelParams p, AttnParams ap) {
    using SM = ScSmem<W, R>;
    constexpr int NT = SM::NT;
    // attention stages: 4 KB (bf16) / kF8Stage (FP8) slots over the scoring ring's bytes
    // (FP8: at most 6 stages per consumer warp — 8 measured slower on C3)
    constexpr int RA = F8 ? ((R * kSsStageBytes / kF8Stage) / W * W < 6 * W ? (R * kSsStageBytes / kF8Stage) / W * W : 6 * W) : 2 * R;
    static_assert(!F8 || RA <= 4 * R, "FP8 stage barriers must fit the afull / aempty slots");
    static_assert(R % W == 0 && RA % W == 0, "stage -> consumer warp must be fixed");
    extern __shared__ uint8_t sc_raw[];
    // 1024-byte aligned (TMA swizzle atoms) by pointer arithmetic on the __shared__ array
    // itself, so the compiler keeps the shared state space (LDS / ATOMS, not generic LD / ATOM)
    uint8_t *smem = sc_raw + ((1024u - (smem_u32(sc_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(smem);
    const uint32_t mfull0 = sb + SM::kBars, mempty0 = mfull0 + 8 * R;
    // barrier slots (6R + 2): mfull[R], mempty[R], afull[2R], aempty[2R], q, pt; the FP8
    // attention stages (RA <= 4R) use the afull and (otherwise unused) aempty slots
    const uint32_t afull0 = mempty0 + 8 * R, aempty0 = afull0 + 8 * 2 * R;
    const uint32_t qbar = aempty0 + 8 * 2 * R, ptbar = qbar + 8;
    const int mp4 = (p.max_pages + 3) & ~3;
    float *sc = reinterpret_cast<float *>(smem + SM::scores_off(p.kmax));
    const bool pt_bulk = p.flags & 1, two = (p.flags & 2) && p.C > 1;
    const int scap = SM::score_cap(p.max_pages, p.flags, p.chunk);
    int *pt_s = reinterpret_cast<int *>(sc) + scap;
    uint32_t *ckey = reinterpret_cast<uint32_t *>(pt_s + (pt_bulk ? mp4 : 0));  // [C * kmax]
    int *cid = reinterpret_cast<int *>(ckey) + p.C * p.kmax;
    float *mrg = reinterpret_cast<float *>(ckey + ((p.flags & 2) ? 2 * p.C * p.kmax : 0));  // DSM: [C][8][kPS]
    int *hist = reinterpret_cast<int *>(smem + SM::kHist);
    int *red = reinterpret_cast<int *>(smem + SM::kRed);
    float *wpart = reinterpret_cast<float *>(smem + SM::kWarpPart);
    int2 *sel = reinterpret_cast<int2 *>(smem + SM::kSel);
    unsigned *s_kmin = reinterpret_cast<unsigned *>(red + 60), *s_kmax = s_kmin + 1;
    __shared__ int s_last;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = p.C;
    const int row = blockIdx.x / C, rank = blockIdx.x % C;
    const int b = row / p.Hkv, g = row % p.Hkv;
    unsigned long long *dts = p.dbg && blockIdx.x < 4096 ? p.dbg + blockIdx.x * 8 : nullptr;
#ifdef TS_SEL_PROF  // select-internal stamps (the final select) at +4096*8
    unsigned long long *dsel = dts ? dts + 4096 * 8 : nullptr;
#else
    unsigned long long *dsel = nullptr;
#endif
#define SC_STAMP(e) \
    if (dts && tid == 0) dts[e] = globaltimer();
    SC_STAMP(0);
    // the next kernel in the stream (the next layer / step) may be scheduled as our CTAs
    // retire: its prologue overlaps our tail; it waits for our completion before any read
    if (p.flags & 8) pdl_launch_dependents();  // early trigger (dev knob; host default: bit 4)
    if (warp == 0) {  // the 6R + 2 consecutive mbarriers (all count 1), one per lane
        for (int i = lane; i < 6 * R + 2; i += 32) mbar_init(mfull0 + 8 * i, 1);
        fence_mbar_init();
        if (lane == 0) {
            *s_kmin = 0xffffffffu;
            *s_kmax = 0u;
        }
    } else if (warp == 1 && lane < 2) {
        prefetch_tmap(lane ? &tmV : &tmK);
    }
    for (int i = tid; i < kSsHist / 4; i += NT) reinterpret_cast<int4 *>(hist)[i] = make_int4(0, 0, 0, 0);
    __syncthreads();
    // "this CTA is running" (before any DSMEM access); release: its initialised counters
    // and histogram are visible to the remote updates that follow the matching wait
    if (C > 1) cluster_arrive_release();
    pdl_wait();  // inputs may come from the previous kernel in the stream

    // The first copies leave before the row length is known (its load is a global round trip):
    // q (independent of it; the consumers need it with the first stage) and the first R
    // metadata stages of the chunk's storage, full (pages past P_b are scored -inf and read
    // only when a row is shorter than its chunk's first R stages; every issued stage is consumed)
    const int j0 = rank * p.chunk;
    const int cstore = max(0, min(p.chunk, p.max_pages - j0));  // the chunk's pages in storage
    const int nspec = min(R, (cstore + kSsStagePages - 1) / kSsStagePages);
    if (warp == W) {
        if (lane == R) {
            mbar_arrive_expect_tx(qbar, p.G * kRowBytes);
            bulk_load(sb + SM::kQ, p.q + ((size_t)b * p.Hq + g * p.G) * kAttnD, p.G * kRowBytes, qbar);
        }
        if (lane < nspec) {
            const uint32_t bytes = min(kSsStagePages, cstore - lane * kSsStagePages) * 2 * kRowBytes;
            mbar_arrive_expect_tx(mfull0 + 8 * lane, bytes);
            bulk_load_hint(sb + lane * kSsStageBytes,
                           p.meta + ((size_t)row * p.max_pages + j0 + (size_t)lane * kSsStagePages) * 2 * kAttnD,
                           bytes, mfull0 + 8 * lane, l2_policy_evict_first());
        }
    }
    const int L = clamp_len(p.seq_lens[b], p.max_pages, 1, p.S);
    const int P = (L + p.S - 1) / p.S;
    const int nloc = max(0, min(P - j0, p.chunk));
    const int sb0 = two ? 0 : j0;  // index of this CTA's first page in sc[]
    // fused append (ts_decode_step_append, Eq. 1 / SPEC.md:56-59): the row's newest token
    // t = L - 1 goes into its K/V slot and into the min/max record of its page before that
    // page is scored; the CTA whose chunk holds the page does both
    const bool app = APP && L > 0;  // APP instantiation: p.k_new / p.v_new are set
    const int ja = app ? (L - 1) / p.S : -1, aslot = app ? (L - 1) - ja * p.S : 0;
    const bool own = app && ja >= j0 && ja < j0 + nloc;
    const int nst = (nloc + kSsStagePages - 1) / kSsStagePages;
    const int gid = lane >> 2, t = lane & 3;

    // ===================================== 1. score =====================================
    if (warp == W) {
        // (q and the first nspec stages are in flight, above; the consumer warp that owns a
        // slot refills it as it drains)
        if (lane == R + 1 && P > 0 && pt_bulk) {  // every CTA: it maps its own share of the selection
            const uint32_t ptb = min(((uint32_t)P * 4 + 15) & ~15u, (uint32_t)mp4 * 4);
            mbar_arrive_expect_tx(ptbar, ptb);
            bulk_load(smem_u32(pt_s), p.page_table + (size_t)b * p.max_pages, ptb, ptbar);
        }
        if (own && lane >= 16 && lane < 24) {  // the new token's K and V rows (16 B per lane)
            const int c = lane - 16;
            const int blk = checked_block(p.page_table[(size_t)b * p.max_pages + max(ja, 0)], ap.num_blocks);  // (ja >= 0 when own)
            const size_t src = ((size_t)b * p.Hkv + g) * kAttnD + c * 8;
            const size_t prow = ((size_t)blk * p.Hkv + g) * p.S + aslot;  // pool row of the token
            const uint4 kx = *reinterpret_cast<const uint4 *>(p.k_new + src);
            const uint4 vx = *reinterpret_cast<const uint4 *>(p.v_new + src);
            if constexpr (F8) {  // quantise (reading R21): codes + one exponent byte per row
                int ek, ev;
                const uint2 kq = f8_quantize8(kx, ek, 0x00ff0000u), vq = f8_quantize8(vx, ev, 0x00ff0000u);
                uint8_t *kp = const_cast<uint8_t *>(static_cast<const uint8_t *>(ap.k_pool));
                uint8_t *vp = const_cast<uint8_t *>(static_cast<const uint8_t *>(ap.v_pool));
                *reinterpret_cast<uint2 *>(kp + f8_code_off(prow) + c * 8) = kq;
                *reinterpret_cast<uint2 *>(vp + f8_code_off(prow) + c * 8) = vq;
                if (c == 0) {
                    kp[f8_exp_off(prow)] = (uint8_t)(int8_t)ek;
                    vp[f8_exp_off(prow)] = (uint8_t)(int8_t)ev;
                }
            } else {
                uint16_t *kp = const_cast<uint16_t *>(static_cast<const uint16_t *>(ap.k_pool));
                uint16_t *vp = const_cast<uint16_t *>(static_cast<const uint16_t *>(ap.v_pool));
                *reinterpret_cast<uint4 *>(kp + prow * kAttnD + c * 8) = kx;
                *reinterpret_cast<uint4 *>(vp + prow * kAttnD + c * 8) = vx;
            }
            fence_proxy_async_all();  // before the attention phase's TMA reads of this page
        }
        // refills: the consumer warp that owns a slot (stage i -> warp i % W, slot i % R,
        // R % W == 0) re-issues it right after consuming it — no producer round trip
        if (p.prev_ids) {
            // cross-step reuse (NEXT-2; "prefetching selected pages", the rho
            // term of PAPER.md:263-271): this CTA's slice of the PREVIOUS step's selection of
            // the row is staged in sel[] now (block rows; -1 = skip) and its K / V blocks are
            // prefetched into L2 by the whole CTA as soon as the chunk is scored, i.e. during
            // the select.  A hint only: entries outside [0, P_b) are skipped, results do not
            // depend on it.  Read here, before the cluster barrier that precedes every CTA's
            // writes of the new ids.  (Measured: issuing at kernel start, or with an
            // evict_last policy, is slower.)
            const int kp = max(0, min(p.prev_count[row], p.kmax));
            const int a0 = kp * rank / C, a1 = kp * (rank + 1) / C;
            for (int e = lane; e < a1 - a0; e += 32) {
                const int pg = p.prev_ids[(size_t)row * p.kmax + a0 + e];
                sel[e] = make_int2((pg >= 0 && pg < P) ? p.page_table[(size_t)b * p.max_pages + pg] * p.Hkv + g : -1, 0);
            }
        }
    } else {
        mbar_wait(qbar, 0);
        uint32_t qa[8], qp[8];
        {
            const bool live = gid < p.G;
            const uint32_t qrow = sb + SM::kQ + gid * kRowBytes;
            const uint4 x0 = live ? lds_v4(qrow + 16 * t) : make_uint4(0, 0, 0, 0);
            const uint4 x1 = live ? lds_v4(qrow + 16 * (t + 4)) : make_uint4(0, 0, 0, 0);
            const uint32_t w0[4] = {x0.x, x0.y, x0.z, x0.w}, w1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                qa[e] = bf16x2_min0(w0[e]);
                qa[4 + e] = bf16x2_min0(w1[e]);
                qp[e] = bf16x2_max0(w0[e]);
                qp[4 + e] = bf16x2_max0(w1[e]);
            }
        }
        const bool c0 = 2 * t < p.G, c1 = 2 * t + 1 < p.G;
        uint32_t kmn = 0xffffffffu, kmx = 0u;
        const int apl = own ? ja - j0 : -1;  // the appended page, chunk-local
        uint4 kn = make_uint4(0, 0, 0, 0);
        if (own && lane < 16 && (apl / kSsStagePages) % W == warp) {
            kn = *reinterpret_cast<const uint4 *>(p.k_new + ((size_t)b * p.Hkv + g) * kAttnD + (lane & 7) * 8);
            if constexpr (F8) {  // Eq. 1 over the DEQUANTISED key (exact bf16; reading R21)
                int ek;
                const uint2 kq = f8_quantize8(kn, ek, 0x0000ffffu);
                const float sc = pow2i(ek);
                const uint2 d0 = f8x4_dequant_bf16(kq.x, sc), d1 = f8x4_dequant_bf16(kq.y, sc);
                kn = make_uint4(d0.x, d0.y, d1.x, d1.y);
            }
        }
        for (int i = warp; i < max(nst, nspec); i += W) {
            const int st = i % R;
            mbar_wait(mfull0 + 8 * st, (i / R) & 1);
            const uint32_t kb = sb + st * kSsStageBytes;
            if (apl >= i * kSsStagePages && apl < (i + 1) * kSsStagePages) {  // warp-uniform
                if (lane < 16) {  // lanes 0-7: the m row, 8-15: the M row (16 B each)
                    const uint32_t a = kb + (apl - i * kSsStagePages) * 2 * kRowBytes + (lane >> 3) * kRowBytes +
                                       (lane & 7) * 16;
                    uint4 v = lds_v4(a);
                    if (aslot == 0) {  // first key of the page: m = M = k
                        v = kn;
                    } else if (lane < 8) {
                        v = make_uint4(bf16x2_min(v.x, kn.x), bf16x2_min(v.y, kn.y), bf16x2_min(v.z, kn.z),
                                       bf16x2_min(v.w, kn.w));
                    } else {
                        v = make_uint4(bf16x2_max(v.x, kn.x), bf16x2_max(v.y, kn.y), bf16x2_max(v.z, kn.z),
                                       bf16x2_max(v.w, kn.w));
                    }
                    sts_v4(a, v);
                    uint16_t *mrec = const_cast<uint16_t *>(p.meta) + ((size_t)row * p.max_pages + max(ja, 0)) * 2 * kAttnD +
                                     (lane >> 3) * kAttnD + (lane & 7) * 8;
                    *reinterpret_cast<uint4 *>(mrec) = v;  // the cache's record (logical layout)
                    fence_proxy_async();  // generic smem write before the stage's next TMA fill
                }
                __syncwarp();
            }
#pragma unroll
            for (int tile = 0; tile < 2; ++tile) {
                const uint32_t tb = kb + tile * 16 * 2 * kRowBytes;
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int ci = 0; ci < 4; ++ci) {
                    const uint4 a = lds_v4(tb + gid * 2 * kRowBytes + 16 * (t + 4 * ci));
                    const uint4 h = lds_v4(tb + (gid + 8) * 2 * kRowBytes + 16 * (t + 4 * ci));
                    const uint32_t *cf = ci < 2 ? qa + 4 * ci : qp + 4 * (ci - 2);
                    mma_bf16_16816(acc, a.x, h.x, a.y, h.y, cf[0], cf[1]);
                    mma_bf16_16816(acc, a.z, h.z, a.w, h.w, cf[2], cf[3]);
                }
                float m0 = fmaxf(c0 ? acc[0] : kNegInf, c1 ? acc[1] : kNegInf);
                float m1 = fmaxf(c0 ? acc[2] : kNegInf, c1 ? acc[3] : kNegInf);
                m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
                m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
                m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
                m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
                if (t < 2) {
                    const int pg = i * kSsStagePages + tile * 16 + gid + 8 * t;
                    if (j0 + pg < p.max_pages && pg < p.chunk) {
                        const bool valid = pg < nloc;
                        const float v = valid ? (t ? m1 : m0) + 0.0f : kNegInf;
                        sc[sb0 + pg] = v;
                        if (valid) {
                            const uint32_t key = score_key(v);
                            kmn = min(kmn, key);
                            kmx = max(kmx, key);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0 && i + R < nst) {  // refill this warp's slot with stage i + R
                fence_proxy_async();  // this warp's generic reads (and APP patch) before the async write
                const int np = min(kSsStagePages, nloc - (i + R) * kSsStagePages);
                mbar_arrive_expect_tx(mfull0 + 8 * st, np * 2 * kRowBytes);
                bulk_load_hint(kb, p.meta + ((size_t)row * p.max_pages + j0 + (size_t)(i + R) * kSsStagePages) * 2 * kAttnD,
                               np * 2 * kRowBytes, mfull0 + 8 * st, l2_policy_evict_first());
            }
        }
        kmn = __reduce_min_sync(0xffffffffu, kmn);
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        if (lane == 0 && kmn <= kmx) {
            atomicMin(s_kmin, kmn);
            atomicMax(s_kmax, kmx);
        }
    }
    for (int pg = max(nst, nspec) * kSsStagePages + tid; pg < p.chunk; pg += NT)
        if (j0 + pg < p.max_pages) sc[sb0 + pg] = kNegInf;
    __syncthreads();
    SC_STAMP(1);
    if (p.prev_ids) {  // NEXT-2: the previous selection's K / V blocks -> L2 (list staged above)
        const int kp = max(0, min(p.prev_count[row], p.kmax));
        const int a0 = kp * rank / C, a1 = kp * (rank + 1) / C;
        for (int e = tid; e < 2 * (a1 - a0); e += NT) {
            const int brow = sel[e >> 1].x;
            if (brow >= 0) {
                if constexpr (F8)  // the block's S / 16 sub-page records are contiguous
                    prefetch_l2_bulk(reinterpret_cast<const uint8_t *>((e & 1) ? p.v_pool : p.k_pool) +
                                         (size_t)brow * (p.S >> 4) * kF8Rec, (uint32_t)(p.S >> 4) * kF8Rec);
                else
                    prefetch_l2_bulk(((e & 1) ? p.v_pool : p.k_pool) + (size_t)brow * p.S * kAttnD,
                                     (uint32_t)p.S * kRowBytes);
            }
        }
    }

    // ===================================== 2. select =====================================
    // Every CTA of the cluster ends up with the whole row's keys (one-level) or all C x K
    // chunk candidates (two-level) in its own shared memory — an all-gather through DSMEM
    // remote stores and ONE cluster barrier — and runs the same exact top-K redundantly.
    // Each CTA then keeps only its share of the ascending selection (the pages covering its
    // tiles [t0, t1)), so no selection list is broadcast and no second barrier is needed.
    // Two-level (rows much longer than C x K): every CTA first selects its chunk's top-K;
    // exact, as a page of the row's top-K is beaten by fewer than K pages of its own chunk
    // (same order: score, then lower id), so it is among its chunk's candidates.
    cg::cluster_group cl = cg::this_cluster();
    const int S = p.S, tpp = S >> 4, tps = __ffs(tpp) - 1;  // tiles per page (power of 2), log2
    const int kk = min(p.kmax, P);  // the selection size is known before the select
    const int ntile = kk * tpp;
    const int t0 = ntile * rank / C, t1 = ntile * (rank + 1) / C;  // < 2^31: check_layout bounds a row
    const int u0 = t0 / tpp, u1 = (t1 + tpp - 1) / tpp;     // pages of this CTA's tiles
    const int w0 = kk * rank / C, w1 = kk * (rank + 1) / C;  // sel_ids entries this CTA writes
    const int *ptrow = pt_bulk ? pt_s : p.page_table + (size_t)b * p.max_pages;
    int *out_id = p.sel_ids + (size_t)row * p.kmax;
    uint32_t *cand = reinterpret_cast<uint32_t *>(wpart);  // free until the attention ends
    auto emit_pg = [&](int pos, int pg) {
        if (pos >= u0 && pos < u1) sel[pos - u0] = make_int2((checked_block(ptrow[pg], ap.num_blocks) * p.Hkv + g) * S, pg * S);
        if (pos >= w0 && pos < w1) out_id[pos] = pg;
    };
    // attention tile i of this CTA (stage i -> warp i % W, slot i % RA): part kv (0 = K, 1 = V)
    // of its copy; arm_tile sets the slot's expected bytes (one lane per tile)
    auto issue_tile = [&](int i, int kv) {
        const int st = i % RA;
        const int tl = t0 + i, u = tl >> tps, sub = tl & (tpp - 1);
        const int2 pg = sel[u - u0];
        if constexpr (F8) {  // the tile's K / V sub-page record (codes + exponents)
            bulk_load_hint(sb + st * kF8Stage + kv * kF8Rec,
                           static_cast<const uint8_t *>(kv ? ap.v_pool : ap.k_pool) + (size_t)((pg.x >> 4) + sub) * kF8Rec,
                           kF8Rec, afull0 + 8 * st, l2_policy_evict_first());
        } else {
            tma_load_2d(sb + st * 2 * 16 * kRowBytes + kv * 16 * kRowBytes, kv ? &tmV : &tmK, 0, pg.x + 16 * sub,
                        afull0 + 8 * st, l2_policy_evict_first());
        }
    };
    auto arm_tile = [&](int i) { mbar_arrive_expect_tx(afull0 + 8 * (i % RA), F8 ? kF8Stage : 2 * 16 * kRowBytes); };
    // One-level rows: the first attention tiles leave DURING the select.  As soon as its first radix
    // pass has found the boundary bin, every key above the bin is known to be selected: those
    // pages go first in the attention order (ascending), their first RA tiles are issued at
    // once, and the rest of the select (boundary ranking, compaction) overlaps the copies; the
    // remaining selected pages follow in ascending order.  sel_ids stays ascending.
    int s_pre = 0;  // attention tiles [0, s_pre) already issued
    uint64_t pre_gm = 0;  // this thread's run of keys: which are "above the bin"
    int pre_cb = 0, pre_nc = 0;
    uint32_t pre_x = 0xffffffffu;
    bool pre_on = false;
    const int pn4 = (P + 3) >> 2, pper4 = (pn4 + NT - 1) / NT, pi0 = tid * pper4;  // cta_topk's compaction runs
    auto emit_att = [&](int q, int i) {  // attention-order entry q (this CTA keeps its share)
        if (q >= u0 && q < u1) sel[q - u0] = make_int2((checked_block(ptrow[i], ap.num_blocks) * p.Hkv + g) * S, i * S);
    };
    uint32_t *lkeys = reinterpret_cast<uint32_t *>(sc);  // scores -> orderable keys, in place
    if (!two) {
        // this CTA's slice of the row as keys (0 = no page, up to the 4-padded row length)
        const int e1 = min(j0 + p.chunk, (P + 3) & ~3);
        for (int i = j0 + tid; i < e1; i += NT) lkeys[i] = i < P ? score_key(sc[i]) : 0u;
        if (C > 1) {
            __syncthreads();
            cluster_wait();  // every CTA of the cluster is running
            const int n4 = max(0, e1 - j0) >> 2;  // j0 and e1 are multiples of 4: 16-byte stores
            const uint4 *src = reinterpret_cast<const uint4 *>(lkeys + j0);
            for (int x = tid; x < (C - 1) * n4; x += NT) {
                const int r = rank + 1 + x / n4, i = x % n4;
                reinterpret_cast<uint4 *>(cl.map_shared_rank(lkeys, r < C ? r : r - C) + j0)[i] = src[i];
            }
            if (tid >= 1 && tid < C && *s_kmin <= *s_kmax) {  // thread r: peer rank + r
                const int r = rank + tid, peer = r < C ? r : r - C;
                atomicMin(cl.map_shared_rank(s_kmin, peer), *s_kmin);
                atomicMax(cl.map_shared_rank(s_kmax, peer), *s_kmax);
            }
            cluster_arrive_release();
            cluster_wait();
        }
        SC_STAMP(5);
        if (P > 0 && pt_bulk) mbar_wait(ptbar, 0);
        __syncthreads();
        SC_STAMP(6);
        {
            auto pre = [&](uint32_t x, int nc) {  // every key > x is selected; nc of them
                // block-uniform; not for FP8 KV (measured 0.5 % slower there: its consumer,
                // not the first copies' latency, bounds the attention)
                if (F8 || pper4 > 16 || nc <= 0) return;
                const uint4 *k4 = reinterpret_cast<const uint4 *>(lkeys);
                const int pi1 = min(pn4, pi0 + pper4);
                uint64_t gm = 0;
                for (int i = pi0; i < pi1; ++i) {
                    const uint4 v = k4[i];
                    gm |= (uint64_t)((uint32_t)(v.x > x) | ((uint32_t)(v.y > x) << 1) | ((uint32_t)(v.z > x) << 2) |
                                     ((uint32_t)(v.w > x) << 3)) << (4 * (i - pi0));
                }
                int tot;
                const int before = block_scan<NT, 0>(__popcll(gm), red, &tot);
                int q = before;
                for (uint64_t sm = gm; sm; sm &= sm - 1) emit_att(q++, 4 * pi0 + __ffsll((long long)sm) - 1);
                pre_gm = gm;
                pre_cb = before;
                pre_nc = nc;
                pre_x = x;
                pre_on = true;
                __syncthreads();  // the first nc attention entries are in place
                s_pre = max(0, min(nc * tpp - t0, min(RA, t1 - t0)));  // this CTA's share of them
                if (warp < W) {
                    if constexpr (APP)
                        fence_proxy_async_all();  // the appended row (generic stores) may be gathered
                    else
                        fence_proxy_async();  // the ring was last accessed by the generic proxy
                    const int e = lane >> 1, i = warp + W * e;
                    if (e < RA / W && i < s_pre) {
                        if ((lane & 1) == 0) arm_tile(i);
                        issue_tile(i, lane & 1);
                    }
                }
            };
            cta_topk<NT, 0, 0>(lkeys, P, p.kmax, *s_kmin, *s_kmax, hist, red, cand,
                               [&](int pos, int i) {
                                   if (pos >= w0 && pos < w1) out_id[pos] = i;
                                   if (!pre_on) {
                                       emit_att(pos, i);
                                   } else if (lkeys[i] <= pre_x) {  // after the nc keys above the bin
                                       const int below = __popcll(pre_gm & ((1ull << (i - 4 * pi0)) - 1ull));
                                       emit_att(pre_nc + pos - (pre_cb + below), i);
                                   }
                               },
                               dsel, false, -1, 0, 0, pre);
        }
    } else {
        // two-level: ONE inlined cta_topk serves both levels (instruction-cache footprint: the
        // fused step's top stall is no_instruction; measured C5 22.4 -> 22.1 us): level 0 = this
        // chunk's top-K, level 1 = the top-K of the C x K gathered candidates
        uint32_t *myk = ckey + rank * p.kmax;
        int *myi = cid + rank * p.kmax;
        for (int i = tid; i < ((nloc + 3) & ~3); i += NT) lkeys[i] = i < nloc ? score_key(sc[i]) : 0u;
        __syncthreads();
        int lvl = 0;
#pragma unroll 1
        for (;;) {
            const uint32_t *skeys = lkeys;
            int sn = nloc, snlive = -1;
            uint32_t smn = *s_kmin, smx = *s_kmax;
            if (lvl == 1) {  // the C x K candidates: chunk-major, ids ascending inside a chunk
                sn = C * p.kmax;
                snlive = 0;  // live candidates: sum over chunks of min(K, chunk pages)
                for (int r = 0; r < C; ++r) snlive += min(p.kmax, max(0, min(P - r * p.chunk, p.chunk)));
                smn = 0xffffffffu;
                smx = 0u;
                for (int i = tid; i < sn; i += NT)
                    if (ckey[i]) {
                        smn = min(smn, ckey[i]);
                        smx = max(smx, ckey[i]);
                    }
                skeys = ckey;
                if (P > 0 && pt_bulk) mbar_wait(ptbar, 0);
                block_minmax<NT, 0>(smn, smx, red);
                SC_STAMP(6);
            }
            // entry order == page-id order at both levels: lower index wins ties (reading R6)
            const int kd = cta_topk<NT, 0, 0>(skeys, sn, p.kmax, smn, smx, hist, red, cand,
                                              [&](int pos, int i) {
                                                  if (lvl == 0) {
                                                      myk[pos] = lkeys[i];
                                                      myi[pos] = j0 + i;
                                                  } else {
                                                      emit_pg(pos, cid[i]);
                                                  }
                                              },
                                              lvl ? dsel : nullptr, false, snlive);
            if (lvl == 1) break;
            for (int i = kd + tid; i < p.kmax; i += NT) myk[i] = 0u;  // absent
            __syncthreads();
            cluster_wait();  // every CTA of the cluster is running
            // push this chunk's K candidates into every other CTA; reset the histogram meanwhile
            const int k4n = p.kmax >> 2;  // 16-byte remote stores (host: kmax % 4 == 0)
            for (int x = tid; x < (C - 1) * k4n; x += NT) {
                const int r = rank + 1 + x / k4n, u = x % k4n;
                const int peer = r < C ? r : r - C;
                reinterpret_cast<uint4 *>(cl.map_shared_rank(ckey, peer) + rank * p.kmax)[u] =
                    reinterpret_cast<const uint4 *>(myk)[u];
                reinterpret_cast<int4 *>(cl.map_shared_rank(cid, peer) + rank * p.kmax)[u] =
                    reinterpret_cast<const int4 *>(myi)[u];
            }
            for (int i = tid; i < kSsHist / 4; i += NT) reinterpret_cast<int4 *>(hist)[i] = make_int4(0, 0, 0, 0);
            cluster_arrive_release();
            cluster_wait();
            SC_STAMP(5);
            lvl = 1;
        }
    }
    if (rank == 0) {
        for (int i = kk + tid; i < p.kmax; i += NT) out_id[i] = -1;
        if (tid == 0) p.sel_count[row] = kk;
    }
    __syncthreads();
    if (dsel && tid == 0) dsel[7] = globaltimer();
    SC_STAMP(2);
    SC_STAMP(3);

    // ===================================== 3-4. gather + attend ==========================
    const float sl2 = ap.scale * kLog2e;
    if (warp == W) {
        // the producer's part ends with the metadata stream: the consumer warps gather their
        // own K / V tiles (stage i -> warp i % W, slot i % RA, RA % W == 0), so a slot is
        // re-issued by its owner right after it is consumed and a CTA has W issuing warps
        // (a single issuing lane caps a CTA's 2 KB-tile gather at ~21 GB/s: scripts/gatherbench.cu)
    } else if constexpr (F8) {
        // ---- FP8 KV (reading R21; fp8.cuh f8_attend_tile): per-head f16 q' fragments, each
        // tile's K and V sub-page records (codes + exponents) by one 1-D bulk copy apiece
        uint4 x0 = make_uint4(0, 0, 0, 0), x1 = x0;
        if (gid < p.G) {
            const uint32_t qrow = sb + SM::kQ + gid * kRowBytes + 32 * t;
            x0 = lds_v4(qrow);
            x1 = lds_v4(qrow + 16);
        }
        const F8Q fq = f8_q_prep(x0, x1, sl2);
        fence_proxy_async();  // the ring was last accessed by the generic proxy (scoring)
        const int ntl = t1 - t0;
        {  // lane 2e + kv issues the K (kv 0) or V (kv 1) record of the warp's e-th stage
            const int e = lane >> 1, i = warp + W * e;
            if (e < RA / W && i < ntl && i >= s_pre) {
                if ((lane & 1) == 0) arm_tile(i);
                issue_tile(i, lane & 1);
            }
        }
        F8Acc acc;
        for (int i = warp; i < ntl; i += W) {
            const int st = i % RA;
            const int tl = t0 + i, tu = tl >> tps;
            const int tok0 = sel[tu - u0].y + 16 * (tl & (tpp - 1));
            mbar_wait(afull0 + 8 * st, (i / RA) & 1);
            const uint32_t kb = sb + st * kF8Stage;
            f8_attend_tile(acc, fq, kb, kb + kF8Rec, tok0, L, gid, t);
            __syncwarp();
            if (lane < 2 && i + RA < ntl) {  // refill this warp's slot with stage i + RA
                fence_proxy_async();
                if (lane == 0) arm_tile(i + RA);
                issue_tile(i + RA, lane);
            }
        }
        f8_store_partial(wpart + warp * 8 * kSaPart, kSaPart, acc, gid, t, p.G);
    } else {
        uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (gid < p.G) {
            const uint32_t qrow = sb + SM::kQ + gid * kRowBytes + 32 * t;
            const uint4 x0 = lds_v4(qrow), x1 = lds_v4(qrow + 16);
            qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
            qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
        }
        // the ring was last accessed by the generic proxy (scoring); APP: the appended K/V
        // row (another CTA's generic stores, published by the cluster barrier) is read by TMA
        bool reads_app = false;  // does this CTA gather the appended page? (then a global proxy fence)
        if constexpr (APP) {
            for (int u = lane; app && u < u1 - u0; u += 32) reads_app |= sel[u].y == ja * p.S;
            reads_app = __any_sync(0xffffffffu, reads_app);
        }
        if (reads_app)
            fence_proxy_async_all();
        else
            fence_proxy_async();
        const int ntl = t1 - t0;
        {  // lane 2e + kv issues the K (kv 0) or V (kv 1) tile of this warp's e-th stage
            const int e = lane >> 1, i = warp + W * e;
            if (e < RA / W && i < ntl && i >= s_pre) {
                if ((lane & 1) == 0) arm_tile(i);
                issue_tile(i, lane & 1);
            }
        }
        float m = kNegInf, lp = 0.f;
        // O^T accumulators: oacc[db] = channels (8 gid + 2 db, 8 gid + 2 db + 1) x heads (2t, 2t+1)
        float oacc[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
        for (int i = warp; i < t1 - t0; i += W) {
            const int st = i % RA;
            // the tile's first token, from sel[] (complete before the barrier), ahead of the wait
            const int tl = t0 + i, tu = tl >> tps;
            const int tok0 = sel[tu - u0].y + 16 * (tl & (tpp - 1));
            mbar_wait(afull0 + 8 * st, (i / RA) & 1);
            const uint32_t kb = sb + st * 2 * 16 * kRowBytes, vb = kb + 16 * kRowBytes;
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
            // O^T += V^T P^T (attn.cuh): the lane's V rows (channels 8 gid .. + 7) of its tokens
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
            if (lane < 2 && i + RA < ntl) {  // refill this warp's slot with stage i + RA
                fence_proxy_async();
                if (lane == 0) arm_tile(i + RA);
                issue_tile(i + RA, lane);
            }
        }
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
    SC_STAMP(4);
    if (p.flags & 16) pdl_launch_dependents();  // late trigger: only the merge / tail remains
    // ---- CTA merge of the W warp partials (C == 1: straight to o / lse)
    for (int x = tid; x < p.G * 16; x += NT) {
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
            *reinterpret_cast<float4 *>(ap.o + oh * kAttnD + d0) =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
            if (ap.lse && d0 == 0) ap.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
        } else if constexpr (DSM) {  // into the leader's merge area (DSMEM stores)
            float *pr = cl.map_shared_rank(mrg, 0) + (rank * 8 + h) * kPS;
            *reinterpret_cast<float4 *>(pr + d0) = acc;
            if (d0 == 0) *reinterpret_cast<float2 *>(pr + kAttnD) = make_float2(M, l);
        } else {
            float *pr = ap.part + (((size_t)row * C + rank) * 8 + h) * kPS;
            *reinterpret_cast<float4 *>(pr + d0) = acc;
            if (d0 == 0) {
                pr[kAttnD] = M;
                pr[kAttnD + 1] = l;
            }
        }
    }
    if constexpr (DSM) {
        // one cluster arrive (release) publishes this CTA's partial; the leader alone waits
        // and merges the C partials from its own shared memory (no L2 round trips)
        if (C > 1) {
            cluster_arrive_release();
            if (rank == 0) {
                cluster_wait();
                for (int x = tid; x < p.G * 16; x += NT) {
                    const int h = x >> 4, d0 = (x & 15) * 4;
                    float M = kNegInf;
                    for (int r = 0; r < C; ++r) M = fmaxf(M, mrg[(r * 8 + h) * kPS + kAttnD]);
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    float l = 0.f;
                    if (M != kNegInf)
                        for (int r = 0; r < C; ++r) {
                            const float *pr = mrg + (r * 8 + h) * kPS;
                            const float f = pr[kAttnD] == kNegInf ? 0.f : exp2f(pr[kAttnD] - M);
                            l += pr[kAttnD + 1] * f;
                            const float4 v = *reinterpret_cast<const float4 *>(pr + d0);
                            acc.x += v.x * f; acc.y += v.y * f; acc.z += v.z * f; acc.w += v.w * f;
                        }
                    const size_t oh = (size_t)b * p.Hq + g * p.G + h;
                    const float inv = l > 0.f ? 1.f / l : 0.f;
                    *reinterpret_cast<float4 *>(ap.o + oh * kAttnD + d0) =
                        make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
                    if (ap.lse && d0 == 0) ap.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
                }
            }
        }
    } else if (C > 1) {
        __syncthreads();
        if (tid == 0) s_last = atom_add_acq_rel_gpu(ap.tickets + row, 1u) == unsigned(C - 1);
        __syncthreads();
        if (s_last) {
            constexpr int kMaxC = 16;
            const float *pb = ap.part + (size_t)row * C * 8 * kPS;
            for (int x = tid; x < p.G * 16; x += NT) {
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
                *reinterpret_cast<float4 *>(ap.o + oh * kAttnD + d0) =
                    make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
                if (ap.lse && d0 == 0) ap.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
            }
            if (tid == 0) ap.tickets[row] = 0u;  // re-armed for the next launch
        }
    }
    SC_STAMP(7);
}

}  // namespace ts
