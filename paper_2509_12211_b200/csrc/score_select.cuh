// score_select.cuh — fused page scoring + top-K selection (Alg. 1 Steps 1-2,
// PAPER.md:217-228; Eq. 2; TopK PAPER.md:162-167), the first kernel of
// the bf16 decode step (head_dim 64, GQA group G <= 8).
//
//  * grid = rows x C CTAs; the C CTAs of one row (b, kv head g) form a thread-block
//    cluster and split the row's pages into contiguous chunks of `chunk` pages;
//  * per CTA one producer lane streams the chunk's metadata records (logical layout: one
//    contiguous run per row) with 1-D bulk copies (cp.async.bulk, L2 evict-first) into a
//    ring of 8 KB stages (32 pages) tracked by mbarriers; W consumer warps take the stages
//    round-robin and compute Eq. 2 for 16 pages x G heads per mma.m16n8k16:
//    [m | M] rows (K = 2d) times [q^- ; q^+] columns, exact bf16 products, fp32 sums,
//    then the max over the group (reading R9) by quad shuffles.  Pages >= P_b: -inf;
//  * the chunk scores are pushed into the cluster leader's shared memory (DSMEM); the
//    leader runs an exact CTA-wide top-K (cta_topk below) and writes the selection
//    (ascending page ids), its count and the physical block of every selected page
//    (page-table row prefetched into smem at kernel start) for the attention kernel;
//  * every CTA triggers its programmatic dependents at once, so the attention kernel's
//    prologue runs while pages are still being scored (PDL).
// A page's score depends only on (q, its record): fixed fragment assignment and reduction
// order, independent of the chunk / cluster split.
#pragma once


#include "attn.cuh"
#include "common.cuh"

namespace ts {


struct ScoreSelParams {
    const uint16_t *q;        // [B][Hq][64]
    const uint16_t *meta;     // [B][Hkv][max_pages][2][64]
    const int *page_table;    // [B][max_pages]
    const int *seq_lens;      // [B]
    int *sel_ids;             // [rows][kmax] ascending, -1 padding
    int *sel_blk;             // [rows][kmax] physical block of each selected page
    int *sel_count;           // [rows]
    int B, Hq, Hkv, G, S, max_pages, kmax;
    int flags;                // step_cluster: bit 0 page-table prefetch, 1 two-level select, 2 DSMEM merge, 3 / 4 early / late PDL trigger
    int C;                    // CTAs per row (cluster size)
    int chunk;                // pages per CTA (multiple of 32)
    unsigned long long *dbg;  // development: per-CTA stamps (nullable)
    // step_cluster, ts_decode_step_append: the newest token of every row (t = seq_len - 1)
    // to append before scoring (nullable: plain decode step)
    const uint16_t *k_new;    // [B][Hkv][64]
    const uint16_t *v_new;    // [B][Hkv][64]
    // step_cluster, ts_decode_step_prefetch (cross-step reuse, "prefetching
    // selected pages"): the previous step's selection [rows][kmax] / counts [rows], read at
    // kernel start (before this step overwrites them) and prefetched into L2 (nullable)
    const int *prev_ids;
    const int *prev_count;
    const uint16_t *k_pool;   // pools for the prefetch addresses ([NB][Hkv][S][64])
    const uint16_t *v_pool;
    // score_select_kernel, ts_select_candidates (the local half of the sequence-sharded step,
    // DESIGN.md §6): block-cyclic ownership (stride > 1: local page jl = global jl * stride +
    // offset); the selection is emitted with GLOBAL ids and, if sel_scores is set, its scores
    int stride, offset;
    float *sel_scores;        // [rows][kmax] (nullable), -inf padding
};

constexpr int kSsStagePages = 32;                         // pages per ring stage
constexpr int kSsStageBytes = kSsStagePages * 2 * kRowBytes;  // 8 KB
constexpr int kSsHist = 2048;                             // radix bins per pass (11 bits)

template <int W, int R>
struct SsSmem {
    static constexpr int NT = (W + 1) * 32;
    static constexpr int kRing = 0;                                 // R x 8 KB
    static constexpr int kQ = kRing + R * kSsStageBytes;           // [8][64] bf16
    static constexpr int kHist = kQ + 8 * kRowBytes;                // [2048] int
    static constexpr int kRed = kHist + kSsHist * 4;                // [64] int scratch
    static constexpr int kBars = kRed + 64 * 4;                     // full[R], empty[R], q, pt
    static constexpr int kScores = (kBars + (2 * R + 2) * 8 + 127) / 128 * 128;  // [max_pages] fp32 / keys
    static size_t bytes(int max_pages) {
        return kScores + (size_t)((max_pages + 3) & ~3) * 4 /* scores */ + (size_t)max_pages * 4 /* page table */ + 16;
    }
};

// ---------------------------------------------------------------------------------------
// Barrier over the NT participating threads: the whole CTA (BAR = 0) or a named barrier
// (BAR > 0) over warps 0 .. NT/32 - 1, so that other warps (a producer) need not join.
// bar: runtime barrier id (0 = the whole CTA); a thread group of NT threads starting at
// thread `tb` (a multiple of 32) may run its own select with its own named barrier.
template <int NT>
TS_DEV void sel_sync(int bar) {
    if (bar == 0)
        __syncthreads();
    else
        named_bar_sync(bar, NT);
}

// Block reductions (NT threads, scratch red[>= NT/32 + 2]).
template <int NT, int BAR = 0>
TS_DEV int block_sum(int v, int *red, int bar = BAR, int tb = 0) {
    v = __reduce_add_sync(0xffffffffu, v);
    const int lane = threadIdx.x & 31, warp = (threadIdx.x - tb) >> 5;
    if (lane == 0) red[warp] = v;
    sel_sync<NT>(bar);
    int s = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w];
    sel_sync<NT>(bar);
    return s;
}
template <int NT, int BAR = 0>
TS_DEV void block_minmax(uint32_t &mn, uint32_t &mx, int *red, int bar = BAR, int tb = 0) {
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    const int lane = threadIdx.x & 31, warp = (threadIdx.x - tb) >> 5;
    if (lane == 0) {
        red[warp] = (int)mn;
        red[32 + warp] = (int)mx;
    }
    sel_sync<NT>(bar);
    uint32_t a = 0xffffffffu, b = 0u;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        a = min(a, (uint32_t)red[w]);
        b = max(b, (uint32_t)red[32 + w]);
    }
    mn = a;
    mx = b;
    sel_sync<NT>(bar);
}
// exclusive scan of one int per thread in thread order; *total = sum
template <int NT, int BAR = 0>
TS_DEV int block_scan(int v, int *red, int *total, int bar = BAR, int tb = 0) {
    const int lane = threadIdx.x & 31, warp = (threadIdx.x - tb) >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) red[warp] = x;
    sel_sync<NT>(bar);
    int before = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
        const int s = red[w];
        before += w < warp ? s : 0;
        tot += s;
    }
    sel_sync<NT>(bar);
    *total = tot;
    return before + x - v;
}

// ---------------------------------------------------------------------------------------
// Exact top-k of the orderable keys[0..n) in shared memory by a whole CTA (NT threads).
// Every key is valid (> key(-inf)); kmin / kmax are their smallest / largest values and
// hist[0..2048) is zero on entry.  Selects kk = min(k, n) entries with the largest keys;
// equal keys go to the lower index (reading R6).  Emits the selected indices in ascending
// order through emit(pos, index) and returns kk.
//
// Adaptive radix select: the candidates are the keys in [kmin, kmax]; a pass buckets them
// by (key - kmin) >> shift into <= 2048 bins (shift makes the range fit), one warp finds
// the bin holding the rem-th largest candidate, and every key above that bin is taken.
// Then either the whole bin is taken, or it is a single key value (ties by index), or its
// <= 64 keys are ranked exactly by one warp, or the search recurses into the bin (each
// pass removes >= 11 bits of the key range, so <= 3 passes).  Scores are spread, so one
// pass plus the ranking is the common case.  The final compaction is one block scan of
// packed (greater, equal) counts over contiguous per-thread segments (ascending output).
#ifndef TS_TOPK_PROF
#ifdef TS_SEL_PROF  // development build (TS_NVCC_EXTRA=-DTS_SEL_PROF): phase stamps in dts[0..4]
#define TS_TOPK_PROF(i) \
    if (dts && threadIdx.x == 0) dts[i] = globaltimer();
#else
#define TS_TOPK_PROF(i)
#endif
#endif
#ifndef TS_TOPK_PROF2
#define TS_TOPK_PROF2(i)
#endif
// Histogram bin b lives at int index hsw(b): the 16-bin runs read as 4 x int4 by one thread
// of the bin search are XOR-rotated by (run >> 1) & 3, so 8 consecutive lanes hit 8
// different 16-byte bank groups (no bank conflicts); a bijection on every 64-bin block.
TS_DEV int hsw(int b) { return b ^ ((b >> 3) & 12); }

// pre(x, nc): called by every thread once the first pass has found its boundary bin, with x
// such that every key > x is selected and nc = their count (a caller may start using them)
struct NoPre {
    TS_DEV void operator()(uint32_t, int) const {}
};
template <int NT, int BAR, int HB = 11, typename Emit, typename Pre = NoPre>
TS_DEV int cta_topk(const uint32_t *keys, int n, int k, uint32_t kmin, uint32_t kmax, int *hist,
                    int *red, uint32_t *cand, Emit emit, unsigned long long *dts = nullptr,
                    bool hist0_built = false, int nvalid = -1, int bar = BAR, int tb = 0, Pre pre = Pre()) {
    // nvalid: number of live (non-zero) keys when keys[] holds zero padding (default n)
    // hist0_built: the first pass histogram over [kmin, kmax] (shift as below) is already
    // in hist (built in parallel by the CTAs of a cluster, score_select / step_cluster)
    // keys[] is 16-byte aligned and zero-padded to a multiple of 4 (0 < every valid key):
    // the scans below read it as uint4 for memory-level parallelism (smem latency ~30 cycles)
    const int tid = threadIdx.x - tb, lane = tid & 31, warp = tid >> 5;
    // HB = 0: radix width by length at run time (~1 key per bin on the first pass), one
    // instantiation instead of two (instruction-cache footprint of the fused kernel)
    const int hb = HB ? HB : (n <= 512 ? 9 : 11);
    const int nlive = nvalid < 0 ? n : nvalid;
    const int kk = min(k, nlive);
    TS_TOPK_PROF(0);
    if (kk <= 0) return 0;
    const uint4 *k4 = reinterpret_cast<const uint4 *>(keys);
    const int n4 = (n + 3) >> 2;
    // selected = {key > tgt} + the first need_eq (lowest index) keys == teq
    uint32_t tgt = 0u, teq = 0xffffffffu;
    int need_eq = 0;
    if (kk < nlive) {
        int rem = kk;
#pragma unroll 1
        for (int pass = 0;; ++pass) {
            if (kmin == kmax) {  // every candidate has the same key: ties by index
                tgt = kmin;
                teq = kmin;
                need_eq = rem;
                break;
            }
            const uint32_t span = kmax - kmin;
            const int bits = 32 - __clz(span);
            const int shift = bits > hb ? bits - hb : 0;
            if (pass > 0) {
                for (int i = tid; i < (1 << hb); i += NT) hist[i] = 0;
                sel_sync<NT>(bar);
            }
            if (pass > 0 || !hist0_built) {
#pragma unroll 2
                for (int i = tid; i < n4; i += NT) {
                    const uint4 v = k4[i];
                    const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {  // branch-free: a key out of range adds 0
                        const bool in = e[j] >= kmin && e[j] <= kmax;
                        const int bn = in ? (int)((e[j] - kmin) >> shift) : lane;
                        atomicAdd(&hist[hsw(bn)], in ? 1 : 0);
                    }
                }
                sel_sync<NT>(bar);
            }
            TS_TOPK_PROF(1);
            {  // boundary bin: thread t < TT owns bins [16 t, 16 t + 16); block suffix scan
                constexpr int PB = 16;
                static_assert((1 << 11) / PB <= NT, "bin search needs (1 << hb) / 16 threads");
                const int TT = (1 << hb) / PB, TW = (TT + 31) / 32;
                int c[PB], sm = 0, suf = 0;
                TS_TOPK_PROF2(8);
                if (warp < TW) {
                    if (tid < TT) {
                        const int4 *h4 = reinterpret_cast<const int4 *>(hist) + tid * (PB / 4);
#pragma unroll
                        for (int j = 0; j < PB / 4; ++j) {
                            const int4 v = h4[j ^ ((tid >> 1) & 3)];  // hsw layout
                            c[4 * j] = v.x; c[4 * j + 1] = v.y; c[4 * j + 2] = v.z; c[4 * j + 3] = v.w;
                        }
                        sm = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7])) +
                             ((c[8] + c[9]) + (c[10] + c[11])) + ((c[12] + c[13]) + (c[14] + c[15]));
                    }
                    suf = sm;  // inclusive suffix over the lanes >= lane of this warp
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_down_sync(0xffffffffu, suf, o);
                        if (lane + o < 32) suf += y;
                    }
                    if (lane == 0) red[40 + warp] = suf;  // warp total
                }
                TS_TOPK_PROF2(9);
                sel_sync<NT>(bar);
                TS_TOPK_PROF2(10);
                if (tid < TT) {
#pragma unroll
                    for (int w = 0; w < TW; ++w)
                        if (w > warp) suf += red[40 + w];
                    const int above_run = suf - sm;
                    if (above_run < rem && suf >= rem) {  // exactly one thread
                        int acc = above_run, bsel = 0, cb = 0, ab = 0;
                        bool done = false;
#pragma unroll
                        for (int j = PB - 1; j >= 0; --j) {
                            if (!done && acc + c[j] >= rem) {
                                bsel = j;
                                cb = c[j];
                                ab = acc;
                                done = true;
                            }
                            acc += c[j];
                        }
                        red[48] = tid * PB + bsel;
                        red[49] = ab;
                        red[50] = cb;
                    }
                }
                if (tid == 0) red[51] = 0;  // candidate counter
                TS_TOPK_PROF2(11);
            }
            sel_sync<NT>(bar);
            if (dts && tid == 0 && pass == 0) dts[5] = globaltimer();
            TS_TOPK_PROF(2);
            const int bsel = red[48], above = red[49], cnt = red[50];
            const uint32_t blo = kmin + ((uint32_t)bsel << shift);
            const uint32_t bhi = shift ? min(kmax, blo + ((1u << shift) - 1u)) : blo;
            rem -= above;
            if (pass == 0) pre(cnt == rem ? blo - 1u : bhi, cnt == rem ? kk : kk - rem);
            if (cnt == rem) {  // the whole bin is taken: keys >= blo
                tgt = blo - 1u;
                break;
            }
            if (shift == 0) {  // the bin is one key value
                tgt = blo;
                teq = blo;
                need_eq = rem;
                break;
            }
            if (cnt <= 64) {  // rank the bin's keys exactly in one warp
#pragma unroll 2
                for (int i = tid; i < n4; i += NT) {
                    const uint4 v = k4[i];
                    const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (e[j] >= blo && e[j] <= bhi) {
                            const int at = atomicAdd(&red[51], 1);
                            cand[2 * at] = e[j];
                            cand[2 * at + 1] = (uint32_t)(4 * i + j);
                        }
                }
                sel_sync<NT>(bar);
                TS_TOPK_PROF(3);
                if (warp == 0) {
                    // rank(c) = #{x : key_x > key_c or (key_x == key_c and idx_x < idx_c)}
                    // (rolled loops: the select is latency-bound and its code shares the
                    // instruction cache with the rest of the fused step)
#pragma unroll 1
                    for (int h = 0; h < 2; ++h) {
                        const int c = lane + 32 * h;
                        if (c < cnt) {
                            const uint32_t kc = cand[2 * c], ic = cand[2 * c + 1];
                            int rk = 0, gt = 0;
#pragma unroll 4
                            for (int x = 0; x < cnt; ++x) {
                                const uint2 cx = reinterpret_cast<const uint2 *>(cand)[x];
                                rk += cx.x > kc || (cx.x == kc && cx.y < ic);
                                gt += cx.x > kc;
                            }
                            if (rk == rem - 1) {  // the last selected candidate
                                red[52] = (int)kc;
                                red[53] = rem - gt;  // ties at kc still to take (by index)
                            }
                        }
                    }
                }
                sel_sync<NT>(bar);
                tgt = (uint32_t)red[52];
                teq = tgt;
                need_eq = red[53];
                break;
            }
            // recurse into the bin
            kmin = 0xffffffffu;
            kmax = 0u;
            for (int i = tid; i < n4; i += NT) {
                const uint4 v = k4[i];
                const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (e[j] >= blo && e[j] <= bhi) {
                        kmin = min(kmin, e[j]);
                        kmax = max(kmax, e[j]);
                    }
            }
            block_minmax<NT, BAR>(kmin, kmax, red, bar, tb);
        }
    }
    if (dts && tid == 0) dts[6] = globaltimer();
    TS_TOPK_PROF(4);
    // compaction in index order: thread owns the contiguous run of uint4 [tid*per4, +per4);
    // one scan of packed (greater, equal) counts: before me, min(need_eq, eq_before) ties.
    // Runs of <= 64 keys keep (greater, equal) bit masks, so the emit visits only the
    // selected keys (about k / NT per thread) without re-reading shared memory.
    const int per4 = (n4 + NT - 1) / NT;
    const int i0 = tid * per4, i1 = min(n4, i0 + per4);
    if (per4 <= 16) {
        uint64_t gm = 0, em = 0;
#pragma unroll 2
        for (int i = i0; i < i1; ++i) {
            const uint4 v = k4[i];
            const uint32_t e[4] = {v.x, v.y, v.z, v.w};
            uint32_t g4 = 0, e4 = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                g4 |= (uint32_t)(e[j] > tgt && e[j] != teq) << j;
                e4 |= (uint32_t)(e[j] == teq) << j;
            }
            gm |= (uint64_t)g4 << (4 * (i - i0));
            em |= (uint64_t)e4 << (4 * (i - i0));
        }
        const int n_gt = __popcll(gm), n_eq = __popcll(em);
        int tot;
        const int before = block_scan<NT, BAR>((n_gt << 16) | n_eq, red, &tot, bar, tb);
        const int eq_before = before & 0xffff, gt_before = before >> 16;
        TS_TOPK_PROF(5);
        int pos = gt_before + min(need_eq, eq_before);
        uint64_t sm = gm;
        for (int t = max(0, min(need_eq - eq_before, n_eq)); t > 0; --t) {  // lowest-index ties
            sm |= em & (~em + 1);
            em &= em - 1;
        }
        while (sm) {
            emit(pos++, 4 * i0 + __ffsll((long long)sm) - 1);
            sm &= sm - 1;
        }
    } else {
        int n_gt = 0, n_eq = 0;
#pragma unroll 2
        for (int i = i0; i < i1; ++i) {
            const uint4 v = k4[i];
            n_gt += (v.x > tgt) + (v.y > tgt) + (v.z > tgt) + (v.w > tgt);
            n_eq += (v.x == teq) + (v.y == teq) + (v.z == teq) + (v.w == teq);
        }
        int tot;
        const int before = block_scan<NT, BAR>((n_gt << 16) | n_eq, red, &tot, bar, tb);
        const int eq_before = before & 0xffff, gt_before = before >> 16;
        TS_TOPK_PROF(5);
        int pos = gt_before + min(need_eq, eq_before);
        int taken = eq_before;
        if (n_gt + n_eq > 0)
            for (int i = i0; i < i1; ++i) {
                const uint4 v = k4[i];
                const uint32_t e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    bool sel = e[j] > tgt;
                    if (e[j] == teq) sel = taken++ < need_eq;
                    if (sel) emit(pos++, 4 * i + j);
                }
            }
    }
    TS_TOPK_PROF(6);
    return kk;
}

TS_DEV void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
TS_DEV void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
TS_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <int W, int R>
__global__ void __launch_bounds__((W + 1) * 32) score_select_kernel(ScoreSelParams p) {
    using SM = SsSmem<W, R>;
    constexpr int NT = SM::NT;
    extern __shared__ __align__(128) uint8_t ss_smem[];
    uint8_t *smem = ss_smem;
    const uint32_t sb = smem_u32(smem);
    const uint32_t full0 = sb + SM::kBars, empty0 = full0 + 8 * R;
    const uint32_t qbar = empty0 + 8 * R, ptbar = qbar + 8;
    float *sc = reinterpret_cast<float *>(smem + SM::kScores);
    int *pt_s = reinterpret_cast<int *>(smem + SM::kScores) + ((p.max_pages + 3) & ~3);  // (score_select_kernel)
    int *hist = reinterpret_cast<int *>(smem + SM::kHist);
    int *red = reinterpret_cast<int *>(smem + SM::kRed);
    unsigned *s_kmin = reinterpret_cast<unsigned *>(red + 60), *s_kmax = s_kmin + 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row = blockIdx.x / p.C, rank = blockIdx.x % p.C;
    const int b = row / p.Hkv, g = row % p.Hkv;
    unsigned long long *dts = p.dbg && blockIdx.x < 4096 ? p.dbg + blockIdx.x * 8 : nullptr;
#define SS_STAMP(e) \
    if (dts && tid == 0) dts[e] = globaltimer();
    SS_STAMP(0);
    pdl_launch_dependents();  // the attention kernel may be scheduled from now on
    if (tid == 0) {
        for (int i = 0; i < R; ++i) {
            mbar_init(full0 + 8 * i, 1);
            mbar_init(empty0 + 8 * i, 1);
        }
        mbar_init(qbar, 1);
        mbar_init(ptbar, 1);
        fence_mbar_init();
        *s_kmin = 0xffffffffu;
        *s_kmax = 0u;
    }
    if (rank == 0)  // the leader's first radix pass histogram
        for (int i = tid; i < kSsHist; i += NT) hist[i] = 0;
    __syncthreads();
    if (p.C > 1) cluster_arrive_relaxed();  // "this CTA is running" (before any DSMEM access)
    pdl_wait();  // inputs may come from the previous kernel in the stream (PDL launch)

    // q and the first R metadata stages of the chunk's storage leave before the row length is
    // known (its load is a global round trip; as in decode_cluster_kernel: full stages, pages
    // past P_b scored -inf, every issued stage consumed)
    const int j0 = rank * p.chunk;
    const int cstore = max(0, min(p.chunk, p.max_pages - j0));
    const int nspec = min(R, (cstore + kSsStagePages - 1) / kSsStagePages);
    if (warp == W && lane == 0) {
        mbar_arrive_expect_tx(qbar, p.G * kRowBytes);
        bulk_load(sb + SM::kQ, p.q + ((size_t)b * p.Hq + g * p.G) * kAttnD, p.G * kRowBytes, qbar);
        for (int i = 0; i < nspec; ++i) {  // slots 0 .. R-1 are free
            const uint32_t bytes = min(kSsStagePages, cstore - i * kSsStagePages) * 2 * kRowBytes;
            mbar_arrive_expect_tx(full0 + 8 * i, bytes);
            bulk_load_hint(sb + i * kSsStageBytes,
                           p.meta + ((size_t)row * p.max_pages + j0 + (size_t)i * kSsStagePages) * 2 * kAttnD,
                           bytes, full0 + 8 * i, l2_policy_evict_first());
        }
    }
    const int sst = p.stride > 1 ? p.stride : 1;  // block-cyclic sharding (ts_select_candidates)
    const int L = clamp_len(p.seq_lens[b], p.max_pages, sst, p.S);
    const int P = sst > 1 ? local_pages(L, p.S, sst, p.offset) : (L + p.S - 1) / p.S;  // local pages
    // page-table row -> smem only when the blocks of the selection are wanted (sel_blk)
    const bool pt_bulk = (p.max_pages & 3) == 0 && p.sel_blk != nullptr;  // row start 16-byte aligned
    const int nloc = max(0, min(P - j0, p.chunk));  // valid pages of this CTA
    const int nst = (nloc + kSsStagePages - 1) / kSsStagePages;

    if (warp == W) {
        // ================================ producer ================================
        if (lane == 0) {
            const uint64_t pol = l2_policy_evict_first();
            if (rank == 0 && P > 0 && pt_bulk) {  // page-table row -> smem (page -> block)
                const uint32_t ptb = min(((uint32_t)P * 4 + 15) & ~15u, (uint32_t)p.max_pages * 4);
                mbar_arrive_expect_tx(ptbar, ptb);
                bulk_load(sb + SM::kScores + (uint32_t)((p.max_pages + 3) & ~3) * 4,
                          p.page_table + (size_t)b * p.max_pages, ptb, ptbar);
            }
            const uint16_t *mrow = p.meta + ((size_t)row * p.max_pages + j0) * 2 * kAttnD;
            for (int i = nspec; i < nst; ++i) {
                const int st = i % R;
                mbar_wait(empty0 + 8 * st, ((i / R) & 1) ^ 1);
                const int np = min(kSsStagePages, nloc - i * kSsStagePages);
                const uint32_t bytes = np * 2 * kRowBytes;
                mbar_arrive_expect_tx(full0 + 8 * st, bytes);
                bulk_load_hint(sb + st * kSsStageBytes, mrow + (size_t)i * kSsStagePages * 2 * kAttnD,
                               bytes, full0 + 8 * st, pol);
            }
        }
    } else {
        // ================================ consumers ===============================
        const int gid = lane >> 2, t = lane & 3;
        mbar_wait(qbar, 0);
        uint32_t qa[8], qp[8];  // [q^- ; q^+] coefficients of head gid, channels 8t.., 8(t+4)..
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
        uint32_t kmn = 0xffffffffu, kmx = 0u;  // key range of the valid pages (lanes t < 2)
        for (int i = warp; i < max(nst, nspec); i += W) {
            const int st = i % R;
            mbar_wait(full0 + 8 * st, (i / R) & 1);
            const uint32_t kb = sb + st * kSsStageBytes;
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
                    const int pg = i * kSsStagePages + tile * 16 + gid + 8 * t;  // local page
                    if (j0 + pg < p.max_pages) {
                        const bool valid = pg < nloc;
                        const float v = valid ? (t ? m1 : m0) + 0.0f : kNegInf;
                        sc[j0 + pg] = v;
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
            atomicMin(s_kmin, kmn);
            atomicMax(s_kmax, kmx);
        }
    }
    // pages of the chunk past P_b (no stage covered them)
    for (int pg = max(nst, nspec) * kSsStagePages + tid; pg < p.chunk; pg += NT)
        if (j0 + pg < p.max_pages) sc[j0 + pg] = kNegInf;
    __syncthreads();
    SS_STAMP(1);

    // ---- chunk scores (and key range) -> the leader's shared memory, then the leader selects
    if (p.C > 1) {
        cg::cluster_group cl = cg::this_cluster();
        cluster_wait();  // every CTA of the cluster is running
        if (rank != 0) {
            float *dst = cl.map_shared_rank(sc, 0);
            const int n = min(p.chunk, p.max_pages - j0);
            for (int i = tid; i < n; i += NT) dst[j0 + i] = sc[j0 + i];
            if (tid == 0 && *s_kmin <= *s_kmax) {
                atomicMin(cl.map_shared_rank(s_kmin, 0), *s_kmin);
                atomicMax(cl.map_shared_rank(s_kmax, 0), *s_kmax);
            }
        }
        cluster_arrive_release();
        cluster_wait();
        if (rank != 0) return;
    }
    SS_STAMP(2);
    // ---- leader: exact top-K over the row's P pages (keys in place of the scores)
    uint32_t *keys = reinterpret_cast<uint32_t *>(sc);
    for (int i = tid; i < ((P + 3) & ~3); i += NT) keys[i] = i < P ? score_key(sc[i]) : 0u;
    if (P > 0 && pt_bulk) mbar_wait(ptbar, 0);
    const int *ptrow = pt_bulk ? pt_s : p.page_table + (size_t)b * p.max_pages;
    __syncthreads();
    SS_STAMP(4);
    int *out_id = p.sel_ids + (size_t)row * p.kmax;
    int *out_blk = p.sel_blk ? p.sel_blk + (size_t)row * p.kmax : nullptr;
    float *out_sc = p.sel_scores ? p.sel_scores + (size_t)row * p.kmax : nullptr;
    uint32_t *cand = reinterpret_cast<uint32_t *>(smem + SM::kQ);  // q is in registers by now
    const int kk = cta_topk<NT, 0>(keys, P, p.kmax, *s_kmin, *s_kmax, hist, red, cand,
                                [&](int pos, int i) {
                                    out_id[pos] = i * sst + (sst > 1 ? p.offset : 0);  // global id
                                    if (out_blk) out_blk[pos] = ptrow[i];
                                    if (out_sc) out_sc[pos] = key_score(keys[i]);
                                }, dts);
    SS_STAMP(7);
    for (int i = kk + tid; i < p.kmax; i += NT) {
        out_id[i] = -1;
        if (out_blk) out_blk[i] = 0;
        if (out_sc) out_sc[i] = kNegInf;
    }
    if (tid == 0) p.sel_count[row] = kk;
    SS_STAMP(3);
}

}  // namespace ts
