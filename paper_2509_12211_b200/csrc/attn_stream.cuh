// attn_stream.cuh — persistent sparse decode attention (bf16, d = 64), Alg. 1 Steps 3-4
// as a warp-specialised TMA pipeline with dynamic work items.
//
// Work: row r = (b, kv head g) owns TPR = Kmax * (S / TT) tile slots (TT = min(S, 16) tokens
// of one selected page), cut into `ipr` items of <= IS slots.  Items are numbered row-major
// (the order in which the scoring grid releases rows) and grabbed dynamically by the
// persistent CTAs through a global counter, so rows are consumed as soon as they are
// selected and no CTA idles while work remains.
// CTA = NC consumer warps + 1 TMA warp + 1 scheduler warp + 1 merge warp:
//  * scheduler warp: grabs an item, waits for the row's selection (per-row ready flag,
//    released by score_select_kernel; none in standalone mode), resolves page id -> physical
//    block for the item's slots 32 at a time and appends tile descriptors (tensor-map row,
//    valid tokens, item flags) to a smem descriptor ring; the item is padded with empty
//    slots to a multiple of NC so every consumer sees every item.
//  * TMA warp: consumes descriptors in order; per item it loads the row's Q group (bulk
//    copy), per slot it issues the K and V tile loads ([TT x 64] bf16, 128-B swizzle, L2
//    evict-first) into a STAGES-deep ring; empty slots become empty stages.
//  * consumers: stage i goes to consumer i % NC.  Per tile: S^T = Q K^T on mma.m16n8k16
//    (bf16), fp32 online softmax (exp2), O += P V on mma.m16n8k8 (tf32 P, bf16 V widened
//    exactly) — fragment maps in attn.cuh.  At an item end each consumer drops its (o, m, l)
//    into a smem item slot and moves on.
//  * merge warp: merges the NC partials of each finished item (so merges never stall the
//    ring): a one-item row is finished in place, otherwise an item partial goes to the
//    workspace and the last item of the row (atomic ticket) merges them, re-arming the
//    ticket and the ready flag.  The last CTA to exit re-arms the work counter.
#pragma once
#include "attn.cuh"
#include "common.cuh"

namespace ts {

struct StreamParams {
    AttnParams a;              // shapes / pointers (a.part: [rows][ipr][8][kPS], a.tickets)
    unsigned *ready;           // [rows] selection released (decode-step mode) or nullptr
    unsigned *work;            // [2] global work counter + exit counter (self re-arming)
    int tpr;                   // tile slots per row
    int is;                    // slots per item (items of a row: ipr = ceil(tpr / is))
    int ipr;
    int n_items;               // rows * ipr
    int dbg;                   // development: bit 0 = consumers skip the math
    unsigned long long *dbg_ts;  // development: per-CTA event timestamps [grid][8] or nullptr
    const char *kpool_dbg, *vpool_dbg;  // development: raw pool pointers (dbg bit 1)
};

template <int NC, int STAGES>
struct StreamSmem {
    static constexpr int kTile = 16 * kRowBytes;                   // 2 KB (TT <= 16)
    static constexpr int kStage = 2 * kTile;                       // K + V
    static constexpr int kRing = STAGES * kStage;
    static constexpr int kQ = kRing;                               // 2 x [8][64] bf16
    static constexpr int kNSlot = 2;                               // item slots (partials)
    static constexpr int kScratch = kQ + 2 * 8 * kRowBytes;        // kNSlot x NC x 8 x kPS
    static constexpr int kDR = 256;                                // descriptor ring entries
    static constexpr int kDesc = kScratch + kNSlot * NC * 8 * kPS * 4;  // int4 descriptors
    static constexpr int kBars = kDesc + kDR * 16;
    static constexpr int kInfo = kBars + (2 * STAGES + 4) * 8;     // per-stage int2 info
    static constexpr int kItemRing = 64;                           // > items in flight
    static constexpr int kItems = kInfo + STAGES * 8;              // int4 item records
    static constexpr int kTotal = kItems + kItemRing * 16;
    static constexpr size_t bytes() { return 1024 + kTotal; }
};

template <int NC, int STAGES>
TS_DEV void stream_merge_warp(const StreamParams &sp, uint8_t *smem, int *s_arrive, int *s_merged,
                              const int *s_nitems);

// descriptor flags (bits above the 8-bit valid-token count)
constexpr int kFirst = 1 << 8, kLast = 1 << 9, kEnd = 1 << 10;

template <int TT, int NC, int STAGES>
__global__ void __launch_bounds__((NC + 3) * 32, 2)
    attn_stream_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       StreamParams sp) {
    using SM = StreamSmem<NC, STAGES>;
    constexpr int NT = TT / 8;
    constexpr int kStageTx = 2 * TT * kRowBytes;
    constexpr int DR = SM::kDR;
    const AttnParams &p = sp.a;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t full0 = sb + SM::kBars, empty0 = full0 + 8 * STAGES;
    const uint32_t qfull0 = empty0 + 8 * STAGES, qempty0 = qfull0 + 16;
    int2 *info = reinterpret_cast<int2 *>(smem + SM::kInfo);
    int4 *desc = reinterpret_cast<int4 *>(smem + SM::kDesc);    // (tmap row, flags|nv, seq, -)
    int4 *items = reinterpret_cast<int4 *>(smem + SM::kItems);  // (row, part, -, -) by seq % ring
    float *scratch = reinterpret_cast<float *>(smem + SM::kScratch);
    __shared__ int s_dhead;         // descriptors written (scheduler)
    __shared__ int s_dtail;         // descriptors consumed (TMA warp)
    __shared__ int s_arrive[SM::kNSlot];  // consumers done with the item in slot
    __shared__ int s_merged[SM::kNSlot];  // seq + 1 of the last item merged out of the slot
    __shared__ int s_nitems;              // items taken by this CTA (set at the end)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, (sp.dbg & 4) ? 32 : 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(qfull0 + 8 * i, 1);
            mbar_init(qempty0 + 8 * i, NC);
        }
        for (int i = 0; i < SM::kNSlot; ++i) {
            s_arrive[i] = 0;
            s_merged[i] = 0;
        }
        s_nitems = -1;
        s_dhead = 0;
        s_dtail = 0;
        fence_mbar_init();
    }
    __syncthreads();
    const int TPP = p.S / TT;
    volatile int *vdhead = &s_dhead, *vdtail = &s_dtail;
    unsigned long long *dts = sp.dbg_ts ? sp.dbg_ts + blockIdx.x * 8 : nullptr;
    if (dts && threadIdx.x == 0) dts[0] = globaltimer();

    if (warp == NC + 1) {
        // ================================ scheduler ================================
        int head = 0, seq = 0;
        for (;;) {
            int item = 0;
            if (lane == 0) {
                // take a new item only when the TMA warp is within STAGES descriptors of the
                // end of the queued work: ~one item of look-ahead, so early CTAs cannot hoard
                while (head - *vdtail > STAGES) nanosleep_ns(64);
                item = (int)atomicAdd(sp.work, 1u);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (item >= sp.n_items) break;
            if (dts && lane == 0 && seq == 0) dts[1] = globaltimer();
            const int row = item / sp.ipr, part = item % sp.ipr;
            const int b = row / p.Hkv, g = row % p.Hkv;
            if (sp.ready) {
                if (lane == 0)
                    while (ld_acquire_u32(sp.ready + row) == 0) nanosleep_ns(32);
                __syncwarp();
            }
            const int L = p.seq_lens[b];
            const int cnt = __ldcg(p.sel_count + row);
            const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
            const int a = part * sp.is, e = min(sp.tpr, a + sp.is);
            const int len = e - a, lpad = (len + NC - 1) / NC * NC;
            if (lane == 0) items[seq % SM::kItemRing] = make_int4(row, part, 0, 0);
            for (int x0 = 0; x0 < lpad; x0 += 32) {
                const int x = x0 + lane;
                int y = 0, nv = 0;
                if (x < len) {
                    const int sl = a + x;
                    const int u = sl / TPP, sub = sl % TPP;
                    if (u < cnt) {
                        const int gid = __ldcg(ids + u);
                        if (gid >= 0 && gid % p.stride == p.offset) {
                            const int blk = p.page_table[(size_t)b * p.max_pages + gid / p.stride];
                            nv = max(0, min(TT, min(p.S, L - gid * p.S) - sub * TT));
                            y = (blk * p.Hkv + g) * p.S + sub * TT;
                        }
                    }
                }
                const int nb = min(32, lpad - x0);
                if (lane == 0)  // ring space for this batch
                    while (head + nb - *vdtail > DR) nanosleep_ns(32);
                __syncwarp();
                if (lane < nb) {
                    const int flags = (x < NC ? kFirst : 0) | (x >= lpad - NC ? kLast : 0);
                    desc[(head + lane) % DR] = make_int4(y, nv | flags, seq, 0);
                }
                head += nb;
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    *vdhead = head;
                    if (dts && seq == 0 && x0 == 0) dts[2] = globaltimer();
                }
            }
            ++seq;
        }
        // termination: NC end markers (one per consumer); item count for the merge warp
        if (lane == 0) {
            *reinterpret_cast<volatile int *>(&s_nitems) = seq;
            while (head + NC - *vdtail > DR) nanosleep_ns(32);
            for (int c = 0; c < NC; ++c) desc[(head + c) % DR] = make_int4(0, kEnd, seq, 0);
            __threadfence_block();
            *vdhead = head + NC;
            // the last CTA out re-arms the work counter for the next launch
            __threadfence();
            if (atomicAdd(sp.work + 1, 1u) == gridDim.x - 1) {
                sp.work[0] = 0u;
                sp.work[1] = 0u;
            }
        }
        return;
    }

    if (warp == NC + 2) {
        stream_merge_warp<NC, STAGES>(sp, smem, s_arrive, s_merged, &s_nitems);
        return;
    }

    if (warp == NC) {
        // =================================== TMA ===================================
        const bool lsu = sp.dbg & 4;  // development: cp.async copies by all 32 lanes
        if (!lsu && lane != 0) return;
        const uint64_t pol = l2_policy_evict_first();
        const int qbytes = p.G * kAttnD * 2;
        int prev_seq = -1;
        for (int i = 0;; ++i) {
            while (*vdhead <= i) nanosleep_ns(20);
            const int4 d = make_int4(reinterpret_cast<volatile int *>(desc + i % DR)[0],
                                     reinterpret_cast<volatile int *>(desc + i % DR)[1],
                                     reinterpret_cast<volatile int *>(desc + i % DR)[2], 0);
            if (lsu) __syncwarp();
            if (lane == 0) *vdtail = i + 1;
            const uint32_t st = i % STAGES;
            const bool end = d.y & kEnd;
            if (!end && d.z != prev_seq) {  // new item: Q group -> qbuf[seq & 1]
                prev_seq = d.z;
                if (lane == 0) {
                    const int par = d.z & 1, use = d.z >> 1;
                    const int row = reinterpret_cast<volatile int *>(items + d.z % SM::kItemRing)[0];
                    const int b = row / p.Hkv, g = row % p.Hkv;
                    mbar_wait(qempty0 + 8 * par, (use & 1) ^ 1);
                    mbar_arrive_expect_tx(qfull0 + 8 * par, qbytes);
                    bulk_load(sb + SM::kQ + par * 8 * kRowBytes,
                              static_cast<const uint16_t *>(p.q) + ((size_t)b * p.Hq + g * p.G) * kAttnD,
                              qbytes, qfull0 + 8 * par);
                }
            }
            mbar_wait(empty0 + 8 * st, ((i / STAGES) & 1) ^ 1);
            if (lane == 0) {
                info[st] = make_int2(d.y, d.z);
                __threadfence_block();
            }
            if (lsu) __syncwarp();
            const int nv = d.y & 0xff;
            const uint32_t dst = sb + st * SM::kStage;
            if (!end && nv > 0) {
                if (lsu) {  // 2 x TT rows x 8 chunks of 16 B, swizzled like the TMA layout
                    const char *ks = sp.kpool_dbg + (size_t)d.x * kRowBytes;
                    const char *vs = sp.vpool_dbg + (size_t)d.x * kRowBytes;
#pragma unroll
                    for (int j = 0; j < TT / 4; ++j) {
                        const int c = lane + 32 * j, r = c >> 3, ch = c & 7;
                        const uint32_t off = r * kRowBytes + ((ch ^ (r & 7)) << 4);
                        cp_async16(dst + off, ks + r * kRowBytes + ch * 16);
                        cp_async16(dst + SM::kTile + off, vs + r * kRowBytes + ch * 16);
                    }
                    cp_async_mbar_arrive(full0 + 8 * st);
                } else {
                    mbar_arrive_expect_tx(full0 + 8 * st, kStageTx);
                    if (sp.dbg & 2) {  // development: 1-D bulk copies (no swizzle)
                        bulk_load(dst, sp.kpool_dbg + (size_t)d.x * kRowBytes, TT * kRowBytes,
                                  full0 + 8 * st);
                        bulk_load(dst + SM::kTile, sp.vpool_dbg + (size_t)d.x * kRowBytes,
                                  TT * kRowBytes, full0 + 8 * st);
                    } else {
                        tma_load_2d(dst, &tmK, 0, d.x, full0 + 8 * st, pol);
                        tma_load_2d(dst + SM::kTile, &tmV, 0, d.x, full0 + 8 * st, pol);
                    }
                }
                if (dts && i == 0 && lane == 0) dts[3] = globaltimer();
            } else {
                mbar_arrive(full0 + 8 * st);
            }
            if (end) {
                if (dts && lane == 0) dts[6] = globaltimer();
                // the NC end markers are consecutive: pass on the remaining ones and stop
                for (int c = 1; c < NC; ++c) {
                    const int j = i + c;
                    while (*vdhead <= j) nanosleep_ns(20);
                    if (lane == 0) *vdtail = j + 1;
                    const uint32_t sj = j % STAGES;
                    mbar_wait(empty0 + 8 * sj, ((j / STAGES) & 1) ^ 1);
                    if (lane == 0) info[sj] = make_int2(kEnd, d.z);
                    if (lsu) __syncwarp();
                    mbar_arrive(full0 + 8 * sj);
                }
                return;
            }
        }
    }

    // ================================= consumers =================================
    const int gid = lane >> 2, t = lane & 3;
    const float sl2 = p.scale * kLog2e;
    uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    float m = kNegInf, lpart = 0.f;
    float oacc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
    for (int i = warp;; i += NC) {
        const uint32_t st = i % STAGES;
        mbar_wait(full0 + 8 * st, (i / STAGES) & 1);
        const int2 inf = info[st];
        const int flags = inf.x, seq = inf.y, nv = flags & 0xff;
        if (dts && i == 0 && lane == 0) dts[4] = globaltimer();
        if (flags & kEnd) {
            if (dts && warp == 0 && lane == 0) dts[5] = globaltimer();
            break;
        }
        const int par = seq & 1;
        if (flags & kFirst) {  // item start: Q fragments + fresh accumulators
            mbar_wait(qfull0 + 8 * par, (seq >> 1) & 1);
            const uint32_t qrow = sb + SM::kQ + par * 8 * kRowBytes + gid * kRowBytes + 32 * t;
            const bool live = gid < p.G;
            const uint4 x0 = live ? lds_v4(qrow) : make_uint4(0, 0, 0, 0);
            const uint4 x1 = live ? lds_v4(qrow + 16) : make_uint4(0, 0, 0, 0);
            qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
            qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
            __syncwarp();
            if (lane == 0) mbar_arrive(qempty0 + 8 * par);
            m = kNegInf;
            lpart = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
        }
        if (nv > 0 && !(sp.dbg & 1)) {
            const uint32_t kb = sb + st * SM::kStage, vb = kb + SM::kTile;
            if (nv < TT) {  // zero V rows past seq_len (0 * garbage must not make NaN)
                for (int c = lane; c < (TT - nv) * 8; c += 32)
                    sts_v4(vb + nv * kRowBytes + c * 16, make_uint4(0, 0, 0, 0));
                __syncwarp();
            }
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
            float x[NT][2];
            float tmax = kNegInf;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    const int tok = nt * 8 + 2 * t + q2;
                    x[nt][q2] = tok < nv ? sacc[nt][q2] * sl2 : kNegInf;
                    tmax = fmaxf(tmax, x[nt][q2]);
                }
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
            tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
            const float mnew = fmaxf(m, tmax);
            const float corr = exp2f(m - mnew);
            m = mnew;
            float pr[NT][2];
            float psum = 0.f;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int q2 = 0; q2 < 2; ++q2) {
                    pr[nt][q2] = exp2f(x[nt][q2] - mnew);
                    psum += pr[nt][q2];
                }
            lpart = lpart * corr + psum;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                oacc[j][0] *= corr;
                oacc[j][1] *= corr;
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int q0 = nt * 8 + 2 * t, q1 = q0 + 1;
                const uint4 v0 = lds_v4(vb + q0 * kRowBytes + ((gid ^ (q0 & 7)) << 4));
                const uint4 v1 = lds_v4(vb + q1 * kRowBytes + ((gid ^ (q1 & 7)) << 4));
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
        if (lane == 0) mbar_arrive(empty0 + 8 * st);
        if (!(flags & kLast)) continue;

        // ---- item end: drop my partial into item slot seq % kNSlot and move on
        const float lrow = lpart + __shfl_xor_sync(0xffffffffu, lpart, 1);
        const float lsum = lrow + __shfl_xor_sync(0xffffffffu, lrow, 2);
        const int sl = seq % SM::kNSlot;
        if (seq >= SM::kNSlot)  // the slot still holds item seq - kNSlot until it is merged
            while (*reinterpret_cast<volatile int *>(&s_merged[sl]) < seq - SM::kNSlot + 1)
                nanosleep_ns(20);
        float *slot = scratch + sl * NC * 8 * kPS;
        if (gid < p.G) {
            float *wr = slot + (warp * 8 + gid) * kPS;
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
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            atomicAdd(&s_arrive[sl], 1);
        }
    }
}

// Merge warp of attn_stream_kernel (see the header comment).
template <int NC, int STAGES>
TS_DEV void stream_merge_warp(const StreamParams &sp, uint8_t *smem, int *s_arrive, int *s_merged,
                              const int *s_nitems) {
    using SM = StreamSmem<NC, STAGES>;
    const AttnParams &p = sp.a;
    const int lane = threadIdx.x & 31;
    const int4 *items = reinterpret_cast<const int4 *>(smem + SM::kItems);
    const float *scratch = reinterpret_cast<const float *>(smem + SM::kScratch);
    for (int seq = 0;; ++seq) {
        const int sl = seq % SM::kNSlot;
        // wait for the NC partials of item seq (or for the end of this CTA's items)
        for (;;) {
            if (*reinterpret_cast<volatile int *>(&s_arrive[sl]) == NC) break;
            const int n = *reinterpret_cast<volatile const int *>(s_nitems);
            if (n >= 0 && seq >= n) {
                if (sp.dbg_ts && lane == 0) sp.dbg_ts[blockIdx.x * 8 + 7] = globaltimer();
                return;
            }
            nanosleep_ns(32);
        }
        __threadfence_block();
        const int row = reinterpret_cast<const volatile int *>(items + seq % SM::kItemRing)[0];
        const int part = reinterpret_cast<const volatile int *>(items + seq % SM::kItemRing)[1];
        const int b = row / p.Hkv, g = row % p.Hkv;
        const bool whole = sp.ipr == 1;
        const float *slot = scratch + sl * NC * 8 * kPS;
        float *prow = p.part + ((size_t)row * sp.ipr + part) * 8 * kPS;
        for (int xw = lane; xw < p.G * (kAttnD / 4); xw += 32) {
            const int h = xw / (kAttnD / 4), d0 = (xw % (kAttnD / 4)) * 4;
            float M = kNegInf;
#pragma unroll
            for (int w = 0; w < NC; ++w) M = fmaxf(M, slot[(w * 8 + h) * kPS + kAttnD]);
            float acc[4] = {0.f, 0.f, 0.f, 0.f}, l = 0.f;
            if (M != kNegInf) {
#pragma unroll
                for (int w = 0; w < NC; ++w) {
                    const float *wr = slot + (w * 8 + h) * kPS;
                    const float mw = wr[kAttnD];
                    const float f = mw == kNegInf ? 0.f : exp2f(mw - M);
                    l += wr[kAttnD + 1] * f;
                    const float4 v = *reinterpret_cast<const float4 *>(wr + d0);
                    acc[0] += v.x * f; acc[1] += v.y * f; acc[2] += v.z * f; acc[3] += v.w * f;
                }
            }
            if (whole) {
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
        __syncwarp();
        if (lane == 0) {  // slot free again
            s_arrive[sl] = 0;
            __threadfence_block();
            *reinterpret_cast<volatile int *>(&s_merged[sl]) = seq + 1;
        }
        if (whole) {
            if (lane == 0 && sp.ready) sp.ready[row] = 0u;
            continue;
        }
        __threadfence();
        __syncwarp();
        int fin = 0;
        if (lane == 0) fin = atomicAdd(p.tickets + row, 1u) == unsigned(sp.ipr - 1);
        fin = __shfl_sync(0xffffffffu, fin, 0);
        if (!fin) continue;
        __threadfence();
        // final merge of the row's ipr item partials: lane-parallel over (head, 4 channels)
        const float *pbase = p.part + (size_t)row * sp.ipr * 8 * kPS;
        for (int xw = lane; xw < p.G * (kAttnD / 4); xw += 32) {
            const int h = xw / (kAttnD / 4), d0 = (xw % (kAttnD / 4)) * 4;
            float M = kNegInf;
            for (int s2 = 0; s2 < sp.ipr; ++s2)
                M = fmaxf(M, __ldcg(pbase + (s2 * 8 + h) * kPS + kAttnD));
            float acc[4] = {0.f, 0.f, 0.f, 0.f}, l = 0.f;
            if (M != kNegInf)
                for (int s2 = 0; s2 < sp.ipr; ++s2) {
                    const float *pr = pbase + (s2 * 8 + h) * kPS;
                    const float ms = __ldcg(pr + kAttnD);
                    const float ls = __ldcg(pr + kAttnD + 1);
                    const float4 v = __ldcg(reinterpret_cast<const float4 *>(pr + d0));
                    const float f = ms == kNegInf ? 0.f : exp2f(ms - M);
                    l += ls * f;
                    acc[0] += v.x * f; acc[1] += v.y * f; acc[2] += v.z * f; acc[3] += v.w * f;
                }
            const size_t oh = (size_t)b * p.Hq + g * p.G + h;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
            if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
        }
        if (lane == 0) {
            p.tickets[row] = 0u;
            if (sp.ready) sp.ready[row] = 0u;
        }
    }
}

}  // namespace ts
