// step_pipe.cuh — the bf16 decode step (Alg. 1; "integrates page scoring,
// sparse memory access, and masked attention in a single pass") as ONE kernel in
// which a CTA (or a thread-block cluster of C CTAs) carries NR = 1 or 2 rows (b, kv head g)
// at once — one consumer group of 4 warps per row — fed by ONE producer warp through ONE
// shared TMA ring, in the HBM order
//
//      meta(A)  meta(B)  K/V(A)  K/V(B)
//
// Group A scores A, then selects A while meta(B) streams; group B scores B, then selects B
// while K/V(A) streams; then each group attends its row.  The exact top-K (latency-bound:
// shared-memory round trips and barriers, no HBM traffic) of one row therefore always runs
// under the other row's stream: with every CTA of the grid in the same phase at the same time
// (one wave), a one-row-per-CTA kernel leaves HBM idle during the select.
//
//  1. score (Eq. 2; Alg. 1 Step 1): the CTA's contiguous chunk of the row's
//     metadata records (logical layout: one run per row) is bulk-copied (cp.async.bulk,
//     L2 evict-first) in 8 KB stages of 32 pages; the group computes [m | M] x [q^- ; q^+]
//     on mma.m16n8k16 (exact bf16 products, fp32 sums) and the max over the GQA group (R9);
//  2. select (TopK; Alg. 1 Step 2): C > 1 — the chunk keys (one-level) or
//     the chunk's own top-K candidates (two-level, rows >> C K) are pushed into every peer's
//     shared memory (DSMEM stores) and announced by remote mbarrier arrives (release.cluster;
//     no cluster-wide barrier, so neither the producer nor the other group waits for it);
//     every CTA then runs the same exact radix top-K on the group's 128 threads (cta_topk,
//     lowest page id wins ties, R6) and keeps its share of the ascending selection;
//  3. gather: the producer streams the share's [16 x 64] K and V tiles (2 tiles per 8 KB
//     stage) with 2-D TMA (128-byte swizzle, L2 evict-first), 4 lanes issuing in parallel;
//  4. attend (SparseAttn): S = Q K^T (mma.m16n8k16), fp32 online softmax
//     in exp2, O += P V (mma.m16n8k8, tf32 P — R10), tokens >= seq_len masked (R7); warp
//     partials merge in smem; a split row's C CTA partials through an L2 workspace, the last
//     CTA of the row (acq_rel ticket) combining them.
#pragma once
#include "attn.cuh"
#include "common.cuh"
#include "score_select.cuh"
#include "sparse_attn.cuh"

namespace ts {

constexpr int kPipeW = 4;                    // consumer warps per group
constexpr int kPipeCT = kPipeW * 32;         // consumer threads per group
constexpr int kPipeMaxNR = 2;                // rows (groups) per CTA
constexpr int kPipeNT = kPipeMaxNR * kPipeCT + 32;  // + the producer warp (warp 8)
constexpr int kPipeStage = 8192;             // ring stage: 32 metadata records or 2 K/V tiles

struct PipeParams {
    const uint16_t *q;        // [B][Hq][64]
    const uint16_t *meta;     // [B][Hkv][max_pages][2][64]  (APP: patched in place)
    const int *page_table;    // [B][max_pages]
    const int *seq_lens;      // [B]
    int *sel_ids;             // [rows][kmax] ascending, -1 padding
    int *sel_count;           // [rows]
    const uint16_t *k_new;    // APP: [B][Hkv][64] the newest token (slot seq_len - 1)
    const uint16_t *v_new;
    uint16_t *k_pool;         // APP: [NB][Hkv][S][64]
    uint16_t *v_pool;
    float *o;                 // [B][Hq][64]
    float *lse;               // [B][Hq] (nullable)
    float *part;              // [rows][C][8][kPS] split partials (C > 1)
    unsigned *tickets;        // [rows] zero on entry, re-armed by the kernel
    float scale;
    int B, Hq, Hkv, G, S, max_pages, kmax, rows;
    int NR;                   // rows per cluster (1 or 2)
    int C;                    // CTAs per cluster (chunks per row)
    int chunk;                // pages per CTA chunk (multiple of 32)
    int R;                    // ring stages
    int two;                  // two-level select (chunk top-K, then top-K of C * kmax candidates)
    int share;                // sel entries per row kept by a CTA (>= its pages of the selection)
    int pt_smem;              // page-table rows prefetched into shared memory
    int flags;                // bit 4: PDL trigger after the attention loop
    unsigned long long *dbg;  // development: per-CTA globaltimer stamps [grid][16] (nullable)
};

// Byte offsets of the shared-memory regions (from the 1024-aligned base); host and device.
// Everything but the ring and the barriers is per group (row slot) r: base + r * gstride.
struct PipeLayout {
    int ring, bars, seq, grp, gstride, total;
    int q, hist, red, wpart, kmm, sel, sc, pt, cand;  // offsets inside a group's block
    int scap, ptcap, candcap;  // per row: score entries, page-table entries, candidate words
    __host__ __device__ static int up(int x, int a) { return (x + a - 1) / a * a; }
    __host__ __device__ static PipeLayout make(int R, int NR, int C, int max_pages, int kmax, int chunk,
                                               int two, int share, int pt_smem) {
        PipeLayout l;
        const int mp4 = up(max_pages, 4);
        l.scap = two ? up(chunk, 4) : mp4;
        l.ptcap = pt_smem ? mp4 : 0;
        l.candcap = two ? 2 * C * kmax : 0;
        l.ring = 0;
        l.bars = R * kPipeStage;                   // full[R] empty[R] q pt[NR] sel[NR] keys[NR]
        l.seq = l.bars + (2 * R + 1 + 3 * NR) * 8;  // [R] int: the stage each slot holds
        l.grp = up(l.seq + R * 4, 128);
        l.q = 0;                                   // [8][64] bf16
        l.hist = l.q + 8 * kRowBytes;              // [2048] int
        l.red = l.hist + kSsHist * 4;              // [64] int (+ s_last)
        l.wpart = l.red + 64 * 4;                  // [W][8][kSaPart] fp32 (select scratch before)
        l.kmm = l.wpart + kPipeW * 8 * kSaPart * 4;  // key range [2]
        l.sel = up(l.kmm + 8, 16);                 // [share] int2 (block row, first token)
        l.sc = up(l.sel + share * 8, 16);          // [scap] fp32 scores -> keys
        l.pt = l.sc + l.scap * 4;                  // [ptcap] int
        l.cand = up(l.pt + l.ptcap * 4, 16);       // [C][kmax] keys, then [C][kmax] ids
        l.gstride = up(l.cand + l.candcap * 4, 128);
        l.total = l.grp + NR * l.gstride;
        return l;
    }
};

TS_DEV void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
// arrive (release, cluster scope) on the mbarrier at the same offset in CTA `peer`'s smem
TS_DEV void mbar_arrive_remote(uint32_t bar, uint32_t peer) {
    uint32_t rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(bar), "r"(peer));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
}
TS_DEV void mbar_wait_cluster(uint32_t bar, uint32_t parity) {  // acquire at cluster scope
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// What every thread of a CTA knows about row slot r of its cluster (from seq_lens only, so
// every CTA of the cluster and every warp role agree on every stage count).
struct PipeRow {
    int row, b, g, L, P;
    int nloc, nst;     // this CTA's valid pages of the row, metadata stages
    int kk, t0, t1;    // selection size; this CTA's K/V tiles [t0, t1)
    int u0, w0, w1;    // first selected page of its tiles; its sel_ids entries [w0, w1)
    int nkv;           // K/V stages (2 tiles each)
    bool valid;
};

TS_DEV PipeRow pipe_row(const PipeParams &p, int cluster, int r, int rank) {
    PipeRow x;
    x.row = cluster * p.NR + r;
    x.valid = r < p.NR && x.row < p.rows;
    const int row = x.valid ? x.row : 0;
    x.b = row / p.Hkv;
    x.g = row % p.Hkv;
    x.L = x.valid ? clamp_len(p.seq_lens[x.b], p.max_pages, 1, p.S) : 0;
    x.P = (x.L + p.S - 1) / p.S;
    const int j0 = rank * p.chunk;
    x.nloc = max(0, min(x.P - j0, p.chunk));
    x.nst = x.valid ? (x.nloc + kSsStagePages - 1) / kSsStagePages : 0;
    x.kk = min(p.kmax, x.P);
    const int tpp = p.S >> 4, tps = __ffs(tpp) - 1;
    const int ntile = x.kk * tpp;
    x.t0 = (int)((long long)ntile * rank / p.C);
    x.t1 = (int)((long long)ntile * (rank + 1) / p.C);
    x.u0 = x.t0 >> tps;
    x.w0 = x.kk * rank / p.C;
    x.w1 = x.kk * (rank + 1) / p.C;
    x.nkv = x.valid ? (x.t1 - x.t0 + 1) >> 1 : 0;
    return x;
}

template <bool APP>
__global__ void __launch_bounds__(kPipeNT, 2) decode_pipe_kernel(
    const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, PipeParams p) {
    constexpr int W = kPipeW, CT = kPipeCT;
    extern __shared__ uint8_t pp_raw[];
    // 1024-byte aligned (TMA swizzle atoms) by pointer arithmetic on the __shared__ array
    // itself, so the compiler keeps the shared state space (LDS / ATOMS, not generic LD / ATOM)
    uint8_t *smem = pp_raw + ((1024u - (smem_u32(pp_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(smem);
    const PipeLayout LY = PipeLayout::make(p.R, p.NR, p.C, p.max_pages, p.kmax, p.chunk, p.two,
                                           p.share, p.pt_smem);
    const int R = p.R, NR = p.NR, C = p.C;
    const uint32_t full0 = sb + LY.bars, empty0 = full0 + 8 * R, qbar = empty0 + 8 * R;
    const uint32_t ptbar0 = qbar + 8, selbar0 = ptbar0 + 8 * NR, keybar0 = selbar0 + 8 * NR;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cluster = blockIdx.x / C, rank = blockIdx.x % C;
    const int j0 = rank * p.chunk;
    const int S = p.S, tpp = S >> 4, tps = __ffs(tpp) - 1;
    unsigned long long *dts = p.dbg ? p.dbg + (size_t)blockIdx.x * 16 : nullptr;
#define PP_STAMP(e, who) \
    if (dts && tid == (who)) dts[e] = globaltimer();

    // slot_seq[s]: the global stage number the producer last issued into slot s.  Consumers
    // of the two groups skip each other's stages, so a warp may reach stage n of slot s while
    // the slot's previous stage n - R has not even landed; the full barrier's parity alone
    // would then alias (phase k - 1 in progress reads as "phase k complete").  Seeing
    // slot_seq[s] == n first pins the barrier to stage n's phase (the slot cannot be refilled
    // before its owner consumes stage n).
    volatile int *slot_seq = reinterpret_cast<volatile int *>(smem + LY.seq);
    if (warp == 0) {  // full[R] empty[R] q pt[NR] sel[NR]: count 1; keys[NR]: the C - 1 peers
        for (int i = lane; i < R; i += 32) slot_seq[i] = -1;
        for (int i = lane; i < 2 * R + 1 + 2 * NR; i += 32) mbar_init(full0 + 8 * i, 1);
        if (lane < NR) mbar_init(keybar0 + 8 * lane, C > 1 ? C - 1 : 1);
        fence_mbar_init();
    } else if (warp == 1 && lane < 2) {
        prefetch_tmap(lane ? &tmV : &tmK);
    } else if (warp >= 2 && warp < 2 + NR) {  // group block of row slot warp - 2
        uint8_t *gb = smem + LY.grp + (warp - 2) * LY.gstride;
        for (int i = lane; i < kSsHist / 4; i += 32) reinterpret_cast<int4 *>(gb + LY.hist)[i] = make_int4(0, 0, 0, 0);
        if (lane == 0) {
            reinterpret_cast<unsigned *>(gb + LY.kmm)[0] = 0xffffffffu;
            reinterpret_cast<unsigned *>(gb + LY.kmm)[1] = 0u;
        }
    }
    __syncthreads();
    // "this CTA is running and initialised" (before any DSMEM access by a peer); only the
    // consumer groups wait for the peers, right before their first remote store
    if (C > 1) cluster_arrive_release();
    pdl_wait();  // inputs may come from the previous kernel in the stream
    PP_STAMP(0, 0);

    if (warp == 2 * W) {
        // ===================================== producer =====================================
        PipeRow rw[kPipeMaxNR];
#pragma unroll
        for (int r = 0; r < kPipeMaxNR; ++r) rw[r] = pipe_row(p, cluster, r, rank);
        const int nmeta0 = rw[0].nst, nmeta = rw[0].nst + rw[1].nst;
        const uint64_t pol = l2_policy_evict_first();
        if (lane == 31) {  // the rows' q groups (G x 128 B each)
            uint32_t bytes = 0;
#pragma unroll
            for (int r = 0; r < kPipeMaxNR; ++r) bytes += rw[r].valid ? p.G * kRowBytes : 0;
            mbar_arrive_expect_tx(qbar, bytes);
#pragma unroll
            for (int r = 0; r < kPipeMaxNR; ++r)
                if (rw[r].valid)
                    bulk_load(sb + LY.grp + r * LY.gstride + LY.q,
                              p.q + ((size_t)rw[r].b * p.Hq + rw[r].g * p.G) * kAttnD, p.G * kRowBytes, qbar);
        }
#pragma unroll
        for (int r = 0; r < kPipeMaxNR; ++r)  // page-table rows -> smem (page -> block map)
            if (lane == 29 + r && r < NR) {
                const PipeRow &x = rw[r];
                if (p.pt_smem && x.valid && x.P > 0) {
                    const uint32_t ptb = min(((uint32_t)x.P * 4 + 15) & ~15u, (uint32_t)LY.ptcap * 4);
                    mbar_arrive_expect_tx(ptbar0 + 8 * r, ptb);
                    bulk_load(sb + LY.grp + r * LY.gstride + LY.pt, p.page_table + (size_t)x.b * p.max_pages, ptb,
                              ptbar0 + 8 * r);
                } else {
                    mbar_arrive(ptbar0 + 8 * r);
                }
            }
        auto issue_meta = [&](int n) {
            const int r = n >= nmeta0 ? 1 : 0;
            const int i = n - (r ? nmeta0 : 0), st = n % R;
            const int np = min(kSsStagePages, (r ? rw[1].nloc : rw[0].nloc) - i * kSsStagePages);
            const uint32_t bytes = np * 2 * kRowBytes;
            const uint16_t *src =
                p.meta + ((size_t)(r ? rw[1].row : rw[0].row) * p.max_pages + j0 + i * kSsStagePages) * 2 * kAttnD;
            slot_seq[st] = n;
            mbar_arrive_expect_tx(full0 + 8 * st, bytes);  // (release: orders the slot_seq store)
            bulk_load_hint(sb + st * kPipeStage, src, bytes, full0 + 8 * st, pol);
        };
        // the ring starts empty: its first stages are issued lane-parallel (TMA issue ~100
        // cycles each); lane 0 refills in order as the consumers release stages
        if (lane < min(R, nmeta)) issue_meta(lane);
        if (lane == 0)
            for (int n = R; n < nmeta; ++n) {
                mbar_wait(empty0 + 8 * (n % R), ((n / R) & 1) ^ 1);
                issue_meta(n);
            }
        __syncwarp();
        PP_STAMP(8, 2 * W * 32);
        int kbase = nmeta;
#pragma unroll
        for (int r = 0; r < kPipeMaxNR; ++r) {
            const PipeRow &x = rw[r];
            if (x.nkv == 0) continue;
            mbar_wait(selbar0 + 8 * r, 0);  // the row's selection (this CTA's share) is in sel[r]
            PP_STAMP(9 + 2 * r, 2 * W * 32);
            // the ring was last read by the generic proxy; APP: the appended K/V row (generic
            // stores of some CTA of the cluster, published through the key exchange) is read
            // by TMA below
            if constexpr (APP)
                fence_proxy_async_all();
            else
                fence_proxy_async();
            const int2 *sel = reinterpret_cast<const int2 *>(smem + LY.grp + r * LY.gstride + LY.sel);
            for (int i = 0; i < x.nkv; ++i) {
                const int n = kbase + i, st = n % R;
                const int nt = min(2, x.t1 - x.t0 - 2 * i);
                if (lane == 0) {
                    if (n >= R) mbar_wait(empty0 + 8 * st, ((n / R) & 1) ^ 1);
                    slot_seq[st] = n;
                    mbar_arrive_expect_tx(full0 + 8 * st, nt * 2 * 16 * kRowBytes);
                }
                __syncwarp();
                if (lane < 2 * nt) {  // lane = 2 * tile + (0: K, 1: V)
                    const int e = lane >> 1, kv = lane & 1;
                    const int tl = x.t0 + 2 * i + e;
                    const int2 pg = sel[(tl >> tps) - x.u0];
                    tma_load_2d(sb + st * kPipeStage + e * 2 * 16 * kRowBytes + kv * 16 * kRowBytes,
                                kv ? &tmV : &tmK, 0, pg.x + 16 * (tl & (tpp - 1)), full0 + 8 * st, pol);
                }
            }
            kbase += x.nkv;
            PP_STAMP(10 + 2 * r, 2 * W * 32);
        }
        return;
    }

    // ================================ consumer group r (row slot r) ==========================
    const int r = warp / W, gw = warp % W, ct = tid - r * CT;
    const int bar = 1 + r;  // the group's named barrier
    const PipeRow x = pipe_row(p, cluster, r, rank);
    if (!x.valid) return;  // uniform across the cluster (row index only)
    const PipeRow xo = pipe_row(p, cluster, r ^ 1, rank);  // the other slot: stage bases only
    const int mbase = r ? xo.nst : 0;
    const int kbase = (r ? xo.nst + xo.nkv : 0) + x.nst + (r ? 0 : xo.nst);
    uint8_t *gb = smem + LY.grp + r * LY.gstride;
    const uint32_t gsb = sb + LY.grp + r * LY.gstride;
    int *hist = reinterpret_cast<int *>(gb + LY.hist);
    int *red = reinterpret_cast<int *>(gb + LY.red);
    float *wpart = reinterpret_cast<float *>(gb + LY.wpart);
    unsigned *kmm = reinterpret_cast<unsigned *>(gb + LY.kmm);
    int2 *sel = reinterpret_cast<int2 *>(gb + LY.sel);
    float *sc = reinterpret_cast<float *>(gb + LY.sc);
    const int gid = lane >> 2, t = lane & 3;
    auto wait_stage = [&](int n) {  // stage n is in its slot (see slot_seq above) and has landed
        const int st = n % R;
        while (slot_seq[st] != n) nanosleep_ns(20);
        mbar_wait(full0 + 8 * st, (n / R) & 1);
    };
    mbar_wait(qbar, 0);

    int ja = 0, aslot = 0, apl = -1;  // APP: the appended page (chunk-local apl when owned)
    if constexpr (APP) {
        // fused append (ts_decode_step_append; Eq. 1): the CTA whose chunk holds
        // the newest token's page writes its K / V row (16 B per lane of the group's warp 0);
        // the group barrier + release of the key exchange publish it to every CTA's TMA
        if (x.L > 0) {
            ja = (x.L - 1) / S;
            aslot = (x.L - 1) - ja * S;
            if (ja >= j0 && ja < j0 + x.nloc) apl = ja - j0;
        }
        if (apl >= 0 && gw == 0 && lane < 16) {
            const int c = lane & 7;
            const int blk = p.page_table[(size_t)x.b * p.max_pages + ja];
            const size_t src = ((size_t)x.b * p.Hkv + x.g) * kAttnD + c * 8;
            const size_t dst = (((size_t)blk * p.Hkv + x.g) * S + aslot) * kAttnD + c * 8;
            uint16_t *pool = lane < 8 ? p.k_pool : p.v_pool;
            const uint16_t *nw = lane < 8 ? p.k_new : p.v_new;
            *reinterpret_cast<uint4 *>(pool + dst) = *reinterpret_cast<const uint4 *>(nw + src);
            fence_proxy_async_all();  // before any TMA read of that page
        }
    }

    // ------------------------------------------------------------------ 1. score
    const int sb0 = p.two ? 0 : j0;  // index of this CTA's first page in sc[]
    {
        uint32_t qa[8], qp[8];
        {
            const bool live = gid < p.G;
            const uint32_t qrow = gsb + LY.q + gid * kRowBytes;
            const uint4 x0 = live ? lds_v4(qrow + 16 * t) : make_uint4(0, 0, 0, 0);
            const uint4 x1 = live ? lds_v4(qrow + 16 * (t + 4)) : make_uint4(0, 0, 0, 0);
            const uint32_t u0w[4] = {x0.x, x0.y, x0.z, x0.w}, u1w[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                qa[e] = bf16x2_min0(u0w[e]);
                qa[4 + e] = bf16x2_min0(u1w[e]);
                qp[e] = bf16x2_max0(u0w[e]);
                qp[4 + e] = bf16x2_max0(u1w[e]);
            }
        }
        const bool c0 = 2 * t < p.G, c1 = 2 * t + 1 < p.G;
        uint32_t kmn = 0xffffffffu, kmx = 0u;
        uint4 kn = make_uint4(0, 0, 0, 0);
        if (APP && apl >= 0 && lane < 16 && (apl / kSsStagePages) % W == gw)
            kn = *reinterpret_cast<const uint4 *>(p.k_new + ((size_t)x.b * p.Hkv + x.g) * kAttnD + (lane & 7) * 8);
        for (int i = gw; i < x.nst; i += W) {
            const int n = mbase + i, st = n % R;
            wait_stage(n);
            const uint32_t kb = sb + st * kPipeStage;
            if (APP && apl >= i * kSsStagePages && apl < (i + 1) * kSsStagePages) {  // warp-uniform
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
                    uint16_t *mrec = const_cast<uint16_t *>(p.meta) + ((size_t)x.row * p.max_pages + ja) * 2 * kAttnD +
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
                        const bool valid = pg < x.nloc;
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
            if (lane == 0) mbar_arrive(empty0 + 8 * st);
        }
        kmn = __reduce_min_sync(0xffffffffu, kmn);
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        if (lane == 0 && kmn <= kmx) {
            atomicMin(&kmm[0], kmn);
            atomicMax(&kmm[1], kmx);
        }
    }
    for (int pg = x.nst * kSsStagePages + ct; pg < p.chunk; pg += CT)  // chunk pages past P_b
        if (j0 + pg < p.max_pages) sc[sb0 + pg] = kNegInf;
    named_bar_sync(bar, CT);
    PP_STAMP(1 + 2 * r, r * CT);

    // ------------------------------------------------------------------ 2. select
    {
        cg::cluster_group cl = cg::this_cluster();
        const int *ptrow = p.pt_smem ? reinterpret_cast<const int *>(gb + LY.pt)
                                     : p.page_table + (size_t)x.b * p.max_pages;
        int *out_id = p.sel_ids + (size_t)x.row * p.kmax;
        uint32_t *cand = reinterpret_cast<uint32_t *>(wpart);  // select scratch (attention later)
        auto emit_pg = [&](int pos, int pg) {
            const int u = pos - x.u0;
            if (u >= 0 && u < p.share) sel[u] = make_int2((ptrow[pg] * p.Hkv + x.g) * S, pg * S);
            if (pos >= x.w0 && pos < x.w1) out_id[pos] = pg;
        };
        // push n4 x 16 B at each of the `nsrc` local arrays into every peer's copy (same
        // offsets), then announce it with one remote arrive per peer and wait for the peers'
        auto exchange = [&](uint32_t *const *src, int nsrc, int n4, bool key_range) {
            cluster_wait();  // every CTA of the cluster has initialised its barriers
            for (int e = ct; e < nsrc * (C - 1) * n4; e += CT) {
                const int which = e / ((C - 1) * n4), f = e % ((C - 1) * n4);
                const int rr = rank + 1 + f / n4, u = f % n4;
                const int peer = rr < C ? rr : rr - C;
                reinterpret_cast<uint4 *>(cl.map_shared_rank(src[which], peer))[u] =
                    reinterpret_cast<const uint4 *>(src[which])[u];
            }
            if (key_range && ct >= 1 && ct < C && kmm[0] <= kmm[1]) {
                const int rr = rank + ct, peer = rr < C ? rr : rr - C;
                atomicMin(cl.map_shared_rank(&kmm[0], peer), kmm[0]);
                atomicMax(cl.map_shared_rank(&kmm[1], peer), kmm[1]);
            }
            named_bar_sync(bar, CT);
            if (ct == 0) {
                fence_acq_rel_cluster();
                for (int q = 1; q < C; ++q) mbar_arrive_remote(keybar0 + 8 * r, (rank + q) % C);
            }
            mbar_wait_cluster(keybar0 + 8 * r, 0);
        };
        if (p.two && C > 1) {
            // two-level: this chunk's top-K (exact: a page of the row's top-K is beaten by
            // fewer than K pages of its own chunk, same order), pushed to every peer
            uint32_t *lkeys = reinterpret_cast<uint32_t *>(sc);
            for (int i = ct; i < ((x.nloc + 3) & ~3); i += CT) lkeys[i] = i < x.nloc ? score_key(sc[i]) : 0u;
            uint32_t *ckey = reinterpret_cast<uint32_t *>(gb + LY.cand);
            int *cid = reinterpret_cast<int *>(ckey) + C * p.kmax;
            uint32_t *myk = ckey + rank * p.kmax;
            int *myi = cid + rank * p.kmax;
            named_bar_sync(bar, CT);
            const int kl = cta_topk<CT, 1, 0>(lkeys, x.nloc, p.kmax, kmm[0], kmm[1], hist, red, cand,
                                              [&](int pos, int i) {
                                                  myk[pos] = lkeys[i];
                                                  myi[pos] = j0 + i;
                                              }, nullptr, false, -1, bar, r * CT);
            for (int i = kl + ct; i < p.kmax; i += CT) myk[i] = 0u;  // absent
            for (int i = ct; i < kSsHist / 4; i += CT) reinterpret_cast<int4 *>(hist)[i] = make_int4(0, 0, 0, 0);
            named_bar_sync(bar, CT);
            uint32_t *const srcs[2] = {myk, reinterpret_cast<uint32_t *>(myi)};
            exchange(srcs, 2, p.kmax >> 2, false);  // host: kmax % 4 == 0
            const int nc = C * p.kmax;
            int nlive = 0;  // live candidates: sum over chunks of min(K, chunk pages)
            for (int c = 0; c < C; ++c) nlive += min(p.kmax, max(0, min(x.P - c * p.chunk, p.chunk)));
            uint32_t mn = 0xffffffffu, mx = 0u;
            for (int i = ct; i < nc; i += CT)
                if (ckey[i]) {
                    mn = min(mn, ckey[i]);
                    mx = max(mx, ckey[i]);
                }
            mbar_wait(ptbar0 + 8 * r, 0);
            block_minmax<CT, 1>(mn, mx, red, bar, r * CT);
            // candidates are chunk-major, ids ascending inside a chunk: entry order == id order
            cta_topk<CT, 1, 11>(ckey, nc, p.kmax, mn, mx, hist, red, cand,
                                [&](int pos, int i) { emit_pg(pos, cid[i]); }, nullptr, false, nlive, bar, r * CT);
        } else {
            uint32_t *keys = reinterpret_cast<uint32_t *>(sc);
            const int e1 = min(j0 + p.chunk, (x.P + 3) & ~3);
            for (int i = j0 + ct; i < e1; i += CT) keys[i] = i < x.P ? score_key(sc[i]) : 0u;
            if (C > 1) {
                named_bar_sync(bar, CT);
                uint32_t *const srcs[1] = {keys + j0};
                exchange(srcs, 1, max(0, e1 - j0) >> 2, true);
            }
            mbar_wait(ptbar0 + 8 * r, 0);
            named_bar_sync(bar, CT);
            cta_topk<CT, 1, 0>(keys, x.P, p.kmax, kmm[0], kmm[1], hist, red, cand,
                               [&](int pos, int i) { emit_pg(pos, i); }, nullptr, false, -1, bar, r * CT);
        }
        if (rank == 0) {
            for (int i = x.kk + ct; i < p.kmax; i += CT) out_id[i] = -1;
            if (ct == 0) p.sel_count[x.row] = x.kk;
        }
        named_bar_sync(bar, CT);
        if (ct == 0) mbar_arrive(selbar0 + 8 * r);  // release: sel complete -> producer
        PP_STAMP(2 + 2 * r, r * CT);
    }

    // ------------------------------------------------------------------ 3-4. attend + merge
    {
        const float sl2 = p.scale * kLog2e;
        uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (gid < p.G) {
            const uint32_t qrow = gsb + LY.q + gid * kRowBytes + 32 * t;
            const uint4 x0 = lds_v4(qrow), x1 = lds_v4(qrow + 16);
            qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
            qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
        }
        float m = kNegInf, lp = 0.f;
        float oacc[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
        for (int i = gw; i < x.nkv; i += W) {
            const int n = kbase + i, st = n % R;
            const int nt = min(2, x.t1 - x.t0 - 2 * i);
            int tok0[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {  // first tokens, from sel[] (complete), ahead of the wait
                const int tl = x.t0 + 2 * i + min(e, nt - 1);
                tok0[e] = sel[(tl >> tps) - x.u0].y + 16 * (tl & (tpp - 1));
            }
            wait_stage(n);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (e >= nt) break;
                const uint32_t kb = sb + st * kPipeStage + e * 2 * 16 * kRowBytes, vb = kb + 16 * kRowBytes;
                float sacc[2][4];
#pragma unroll
                for (int ntl = 0; ntl < 2; ++ntl) {
                    sacc[ntl][0] = sacc[ntl][1] = sacc[ntl][2] = sacc[ntl][3] = 0.f;
                    const int rr = ntl * 8 + gid;
                    const uint32_t ra = kb + rr * kRowBytes;
                    const uint4 k0 = lds_v4(ra + (((2 * t) ^ (rr & 7)) << 4));
                    const uint4 k1 = lds_v4(ra + (((2 * t + 1) ^ (rr & 7)) << 4));
                    mma_bf16_16816(sacc[ntl], qa[0], 0u, qa[1], 0u, k0.x, k0.y);
                    mma_bf16_16816(sacc[ntl], qa[2], 0u, qa[3], 0u, k0.z, k0.w);
                    mma_bf16_16816(sacc[ntl], qa[4], 0u, qa[5], 0u, k1.x, k1.y);
                    mma_bf16_16816(sacc[ntl], qa[6], 0u, qa[7], 0u, k1.z, k1.w);
                }
                float xs[2][2];
                float tmax = kNegInf;
#pragma unroll
                for (int ntl = 0; ntl < 2; ++ntl)
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2) {
                        const bool ok = tok0[e] + ntl * 8 + 2 * t + q2 < x.L;
                        xs[ntl][q2] = ok ? sacc[ntl][q2] * sl2 : kNegInf;
                        tmax = fmaxf(tmax, xs[ntl][q2]);
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
                for (int ntl = 0; ntl < 2; ++ntl)
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2) {
                        pr[ntl][q2] = exp2f(xs[ntl][q2] - mref);
                        psum += pr[ntl][q2];
                    }
                lp = lp * corr + psum;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    oacc[j][0] *= corr;
                    oacc[j][1] *= corr;
                }
#pragma unroll
                for (int ntl = 0; ntl < 2; ++ntl) {
                    const int q0 = ntl * 8 + 2 * t, q1 = q0 + 1;
                    uint4 v0 = lds_v4(vb + q0 * kRowBytes + ((gid ^ (q0 & 7)) << 4));
                    uint4 v1 = lds_v4(vb + q1 * kRowBytes + ((gid ^ (q1 & 7)) << 4));
                    if (tok0[e] + q0 >= x.L) v0 = make_uint4(0, 0, 0, 0);  // past seq_len: may be anything
                    if (tok0[e] + q1 >= x.L) v1 = make_uint4(0, 0, 0, 0);
                    const uint32_t a0 = f32_to_tf32(pr[ntl][0]), a2 = f32_to_tf32(pr[ntl][1]);
                    const uint32_t w0v[4] = {v0.x, v0.y, v0.z, v0.w};
                    const uint32_t w1v[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t b0 = (j & 1) ? (w0v[j >> 1] & 0xffff0000u) : (w0v[j >> 1] << 16);
                        const uint32_t b1 = (j & 1) ? (w1v[j >> 1] & 0xffff0000u) : (w1v[j >> 1] << 16);
                        mma_tf32_1688(oacc[j], a0, 0u, a2, 0u, b0, b1);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * st);
        }
        lp += __shfl_xor_sync(0xffffffffu, lp, 1);
        lp += __shfl_xor_sync(0xffffffffu, lp, 2);
        if (gid < p.G) {
            float *wr = wpart + (gw * 8 + gid) * kSaPart;
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
    }
    named_bar_sync(bar, CT);
    PP_STAMP(5 + r, r * CT);
    // the next kernel in the stream may launch once the last row slot's loop is done; its
    // prologue overlaps our merge / tail
    if ((p.flags & 16) && r == NR - 1) pdl_launch_dependents();
    // ---- CTA merge of the W warp partials (C == 1: straight to o / lse)
    for (int xi = ct; xi < p.G * 16; xi += CT) {
        const int h = xi >> 4, d0 = (xi & 15) * 4;
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
            const size_t oh = (size_t)x.b * p.Hq + x.g * p.G + h;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
            if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
        } else {
            float *pr = p.part + (((size_t)x.row * C + rank) * 8 + h) * kPS;
            *reinterpret_cast<float4 *>(pr + d0) = acc;
            if (d0 == 0) {
                pr[kAttnD] = M;
                pr[kAttnD + 1] = l;
            }
        }
    }
    if (C > 1) {  // the last CTA of the row (acq_rel ticket) merges the C partials
        int *s_last = red + 63;
        named_bar_sync(bar, CT);
        if (ct == 0) *s_last = atom_add_acq_rel_gpu(p.tickets + x.row, 1u) == unsigned(C - 1);
        named_bar_sync(bar, CT);
        if (*s_last) {
            constexpr int kMaxC = 16;
            const float *pb = p.part + (size_t)x.row * C * 8 * kPS;
            for (int xi = ct; xi < p.G * 16; xi += CT) {
                const int h = xi >> 4, d0 = (xi & 15) * 4;
                float mr[kMaxC];
#pragma unroll
                for (int c = 0; c < kMaxC; ++c) mr[c] = c < C ? __ldcg(pb + (c * 8 + h) * kPS + kAttnD) : kNegInf;
                float M = kNegInf;
#pragma unroll
                for (int c = 0; c < kMaxC; ++c) M = fmaxf(M, mr[c]);
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                float l = 0.f;
                if (M != kNegInf) {
#pragma unroll
                    for (int c0i = 0; c0i < kMaxC; c0i += 4) {
                        if (c0i >= C) break;
                        float lq[4];
                        float4 vq[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float *pr = pb + ((c0i + e) * 8 + h) * kPS;
                            lq[e] = c0i + e < C ? __ldcg(pr + kAttnD + 1) : 0.f;
                            vq[e] = c0i + e < C ? __ldcg(reinterpret_cast<const float4 *>(pr + d0))
                                                : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float f = mr[c0i + e] == kNegInf ? 0.f : exp2f(mr[c0i + e] - M);
                            l += lq[e] * f;
                            acc.x += vq[e].x * f; acc.y += vq[e].y * f; acc.z += vq[e].z * f; acc.w += vq[e].w * f;
                        }
                    }
                }
                const size_t oh = (size_t)x.b * p.Hq + x.g * p.G + h;
                const float inv = l > 0.f ? 1.f / l : 0.f;
                *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                    make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
                if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
            }
            if (ct == 0) p.tickets[x.row] = 0u;  // re-armed for the next launch
        }
    }
    PP_STAMP(13 + r, r * CT);
}

}  // namespace ts
