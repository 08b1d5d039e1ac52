// decode_pipe.cuh — the fused decode step (Alg. 1, "integrates page
// scoring, sparse memory access, and masked attention in a single pass") as ONE
// persistent, warp-specialised kernel, plus its attention-only mode (ts_sparse_decode_attn).
//
// Work items, numbered in the order they are handed out through a global counter:
//   [0, n_score)            score items: (row, chunk) — SCH metadata tiles of 16 pages
//   [n_score, n_score+n_attn) attention items: (row, part) — IS KV tiles of TT tokens
// Rows are (b, kv head g) in row-major order, so rows are scored, selected and attended in
// the same order and a row's attention starts while later rows are still being scored; the
// HBM request stream never drains between the phases.
//
// CTA = NC consumer warps + 1 TMA warp + 1 scheduler warp + 1 merge/select warp, sharing a
// STAGES-deep ring of 4 KB smem stages:
//  * scheduler: takes an item (with ~one item of look-ahead so early CTAs cannot hoard),
//    waits for the row's selection before an attention item (per-row ready flag), resolves
//    page ids -> physical blocks, and appends per-slot descriptors to a smem ring; every
//    item is padded with empty slots to a multiple of NC so each consumer sees each item.
//  * TMA warp: per item loads the row's Q group (bulk copy); per slot issues either one
//    1-D bulk copy of a metadata tile (16 pages x [m | M], the logical metadata layout
//    makes it contiguous) or the two 2-D TMA tile loads of K and V ([TT x 64] bf16,
//    128-byte swizzle, L2 evict-first).
//  * consumers (stage i -> consumer i % NC):
//      metadata tile: Eq. 2 for 16 pages x G heads on mma.m16n8k16 ([m | M] rows times
//        [q^- ; q^+] columns, exact bf16 products, fp32 sums), max over the group,
//        written into the item's smem score buffer (pages past P_b are -inf);
//      KV tile: S^T = Q K^T (mma.m16n8k16 bf16), fp32 online softmax (exp2),
//        O += P V (mma.m16n8k8, tf32 P, bf16 V widened exactly) — maps in attn.cuh.
//  * merge/select warp, per finished item in order:
//      score item: exact top-K of the chunk (warp radix select, lowest page id wins ties,
//        ids ascending); a one-chunk row is final, otherwise the chunk's candidates go to
//        the workspace and the last chunk (atomic ticket) selects the global top-K from
//        the candidate union (exact: every global top-K page is in its chunk's top-K).
//        The selection is written and the row's ready flag released.
//      attention item: merges the NC consumer partials (o, m, l); a one-item row is
//        finished in place, otherwise the item partial goes to the workspace and the last
//        item of the row (ticket) merges them, re-arming ticket and ready flag.
//    The last CTA to exit re-arms the work counter.
#pragma once
#include "attn.cuh"
#include "common.cuh"

namespace ts {

struct PipeParams {
    AttnParams a;              // shapes / pointers (a.part: [rows][ipr][8][kPS], a.tickets)
    const uint16_t *meta;      // decode mode: logical metadata [B][Hkv][max_pages][2][64]
    unsigned *ready;           // [rows] selection released; nullptr in attention-only mode
    unsigned *sc_tickets;      // [rows] score-chunk tickets (spr > 1)
    float *cand_sc;            // [rows][spr][kmax] chunk candidates (spr > 1)
    int *cand_id;
    int *sel_out;              // decode mode: [rows][kmax] selection (ascending page ids)
    int *cnt_out;              // decode mode: [rows]
    unsigned *work;            // [2] global work counter + exit counter (self re-arming)
    int kmax;                  // K = min(max_pages, max(1, budget / S))
    int sch;                   // metadata tiles per score item
    int spr;                   // score items per row (0: attention-only mode)
    int mtiles;                // metadata tiles per row = ceil(max_pages / 16)
    int n_score;               // rows * spr
    int tpr;                   // KV tile slots per row
    int is;                    // KV slots per attention item
    int ipr;                   // attention items per row
    int n_attn;                // rows * ipr
    int dbg;                   // development: bit 0 = consumers skip the math
    unsigned long long *dbg_ts;
    volatile int *dbg_state;   // development: live per-CTA state [grid][16] (host-mapped)
};

template <int NC, int STAGES>
struct PipeSmem {
    static constexpr int kTile = 16 * kRowBytes;                   // 2 KB
    static constexpr int kStage = 2 * kTile;                       // 4 KB: K + V, or 16 metadata rows
    static constexpr int kRing = STAGES * kStage;
    static constexpr int kQ = kRing;                               // 2 x [8][64] bf16
    static constexpr int kNSlot = 2;                               // item slots
    static constexpr int kSlotFloats = NC * 8 * kPS;               // partials or chunk scores
    static constexpr int kScratch = kQ + 2 * 8 * kRowBytes;
    static constexpr int kSelKeys = 1024;                          // candidate-merge entries
    static constexpr int kMaxParts = 64;                           // = kMaxItemsPerRow (api.cu)
    static constexpr int kHist = kScratch + kNSlot * kSlotFloats * 4;  // merge weights [parts][8]
    static constexpr int kDR = 256;                                // descriptor ring entries
    static constexpr int kDesc = kHist + kMaxParts * 8 * 4;
    static constexpr int kBars = kDesc + kDR * 16;
    static constexpr int kInfo = kBars + (2 * STAGES + 4) * 8;     // per-stage int4 info
    static constexpr int kItemRing = 64;                           // > items in flight
    static constexpr int kItems = kInfo + STAGES * 16;
    static constexpr int kTotal = kItems + kItemRing * 16;
    static constexpr size_t bytes() { return 1024 + kTotal; }
    static constexpr int max_chunk_pages() { return kSlotFloats; }
};

// development: record an error code + value in the host-mapped state, then trap
#define PIPE_CHECK(cond, code, val)                                                       \
    do {                                                                                  \
        if (sp.dbg_state && !(cond)) {                                                    \
            sp.dbg_state[blockIdx.x * 16 + 14] = (code);                                  \
            sp.dbg_state[blockIdx.x * 16 + 15] = (int)(val);                              \
            __threadfence();                                                              \
            for (;;) nanosleep_ns(1000);                                                  \
        }                                                                                 \
    } while (0)

// descriptor / stage flags (bits above the 8-bit valid count)
constexpr int kFirst = 1 << 8, kLast = 1 << 9, kEnd = 1 << 10, kScoreTile = 1 << 11;

// ---------------------------------------------------------------------------------------
// Warp-level exact top-k over n scores in smem (ids ascending with the index: id(i) =
// ids ? ids[i] : id0 + i).  -inf entries are "no page" and never selected.  Ties at the
// threshold go to the lower index (= lower page id, reading R6).  Writes the kk selected
// ids (ascending) and scores to out_id / out_sc (global or shared), pads up to k with
// (-1, -inf), returns kk.
//
// Threshold search, no histogram: T = the kk-th largest orderable key is the largest t
// with #{key >= t} >= kk, found bit by bit from the highest bit in which the smallest and
// the largest valid key differ (the bits above are common to every candidate threshold).
// Each step is one compare per key + one warp reduction (REDUX); keys live in registers
// (KR per lane) when n <= 32 * KR, else they are re-read from smem.  It stops early when a
// prefix bin is taken whole (#{key >= t} == kk).
template <int KR>
TS_DEV int warp_topk(const float *sc, const int *ids, int id0, int n, int k, int *out_id,
                     float *out_sc) {
    const int lane = threadIdx.x & 31;
    const bool inreg = n <= 32 * KR;
    uint32_t kr[KR];
    int nvalid = 0;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int j = 0; j < KR; ++j) {
        const int i = lane + 32 * j;
        kr[j] = (inreg && i < n) ? score_key(sc[i]) : 0u;
    }
    if (inreg) {
#pragma unroll
        for (int j = 0; j < KR; ++j)
            if (kr[j] > kKeyNegInf) {
                ++nvalid;
                kmin = min(kmin, kr[j]);
                kmax = max(kmax, kr[j]);
            }
    } else {
        for (int i = lane; i < n; i += 32) {
            const uint32_t key = score_key(sc[i]);
            if (key > kKeyNegInf) {
                ++nvalid;
                kmin = min(kmin, key);
                kmax = max(kmax, key);
            }
        }
    }
    nvalid = __reduce_add_sync(0xffffffffu, nvalid);
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    const int kk = min(k, nvalid);
    // count of keys >= t over the warp
    auto count_ge = [&](uint32_t t) -> int {
        int c = 0;
        if (inreg) {
#pragma unroll
            for (int j = 0; j < KR; ++j) c += kr[j] >= t;
        } else {
            for (int i = lane; i < n; i += 32) c += score_key(sc[i]) >= t;
        }
        return __reduce_add_sync(0xffffffffu, c);
    };
    // take every key > tgt, plus the first need_eq keys == teq in index order
    uint32_t tgt = kKeyNegInf, teq = 0xffffffffu;
    int need_eq = 0;
    if (kk > 0 && kk < nvalid) {
        uint32_t T = kmin;
        if (kmin != kmax) {
            const int h = 31 - __clz(kmin ^ kmax);
            T = kmax & ~((2u << h) - 1u);  // 2u << 31 == 0: T = 0 when h == 31
            bool whole = false;
#pragma unroll 1
            for (int bit = h; bit >= 0; --bit) {
                const uint32_t cand = T | (1u << bit);
                const int c = count_ge(cand);
                if (c >= kk) {
                    T = cand;
                    if (c == kk) { whole = true; break; }  // keys >= T are exactly kk
                }
            }
            if (whole) {
                tgt = T - 1u;  // key > T - 1  <=>  key >= T
            } else {
                tgt = T;
                teq = T;
                need_eq = kk - count_ge(T + 1u);
            }
        } else {  // every valid key is equal: take the first kk in index order
            teq = T;
            need_eq = kk;
            tgt = T;
        }
    }
    // compaction in index order: lane owns the contiguous segment [lane*per, +per)
    const int per = (n + 31) / 32;
    const int lo = lane * per, hi = min(n, lo + per);
    int n_gt = 0, n_eq = 0;
    if (kk > 0) {
        for (int i = lo; i < hi; ++i) {
            const uint32_t key = score_key(sc[i]);
            n_gt += key > tgt;
            n_eq += key == teq;
        }
    }
    int eq_inc = n_eq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, eq_inc, o);
        if (lane >= o) eq_inc += y;
    }
    const int take = max(0, min(n_eq, need_eq - (eq_inc - n_eq)));
    const int mine = n_gt + take;
    int pos_inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pos_inc, o);
        if (lane >= o) pos_inc += y;
    }
    int pos = pos_inc - mine, seen = 0;
    if (mine > 0) {
        for (int i = lo; i < hi; ++i) {
            const float s = sc[i];
            const uint32_t key = score_key(s);
            bool take_i = key > tgt;
            if (key == teq) { take_i = seen < take; ++seen; }
            if (take_i) {
                out_id[pos] = ids ? ids[i] : id0 + i;
                if (out_sc) out_sc[pos] = s + 0.0f;
                ++pos;
            }
        }
    }
    for (int i = kk + lane; i < k; i += 32) {
        out_id[i] = -1;
        if (out_sc) out_sc[i] = kNegInf;
    }
    __syncwarp();
    return kk;
}

template <int NC, int STAGES>
TS_DEV void pipe_merge_warp(const PipeParams &sp, uint8_t *smem, int *s_arrive, int *s_merged,
                            const int *s_nitems);

template <int TT, int NC, int STAGES>
__global__ void __launch_bounds__((NC + 3) * 32, 2)
    decode_pipe_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                       PipeParams sp) {
    using SM = PipeSmem<NC, STAGES>;
    constexpr int NT = TT / 8;
    constexpr int kStageTx = 2 * TT * kRowBytes;
    constexpr int DR = SM::kDR;
    // Stage i is consumed by warp i % NC.  The same warp must own every use of a stage
    // (slots i, i + STAGES, ...): otherwise a second consumer can start waiting on the
    // stage's full barrier for phase k+1 while phase k is still pending, and
    // try_wait.parity((k+1) & 1) == parity of the completed phase k-1 passes at once.
    static_assert(STAGES % NC == 0, "mbarrier parity: STAGES must be a multiple of NC");
    const AttnParams &p = sp.a;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t full0 = sb + SM::kBars, empty0 = full0 + 8 * STAGES;
    const uint32_t qfull0 = empty0 + 8 * STAGES, qempty0 = qfull0 + 16;
    int4 *info = reinterpret_cast<int4 *>(smem + SM::kInfo);
    int4 *desc = reinterpret_cast<int4 *>(smem + SM::kDesc);    // (src, flags|nv, seq, tile)
    int4 *items = reinterpret_cast<int4 *>(smem + SM::kItems);  // (row, part, kind, -)
    float *scratch = reinterpret_cast<float *>(smem + SM::kScratch);
    __shared__ int s_dhead;                // descriptors written (scheduler)
    __shared__ int s_dtail;                // descriptors consumed (TMA warp)
    __shared__ int s_arrive[SM::kNSlot];   // consumers done with the item in slot
    __shared__ int s_merged[SM::kNSlot];   // seq + 1 of the last item merged out of the slot
    __shared__ int s_nitems;               // items taken by this CTA (set at the end)
    __shared__ int s_total;                // descriptors incl. end markers (set at the end)

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (sp.dbg_state && threadIdx.x == 0) sp.dbg_state[blockIdx.x * 16 + 7] += 1;  // entered
    if (threadIdx.x == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full0 + 8 * i, 1);
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
        s_total = -1;
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
        const int n_items = sp.n_score + sp.n_attn;
        for (;;) {
            // the first item of CTA x is item x (grid <= items); later ones come from the
            // global counter, which therefore counts from gridDim.x
            int item = blockIdx.x;
            if (seq > 0 && lane == 0) {
                while (head - *vdtail > STAGES) nanosleep_ns(64);  // ~one item of look-ahead
                item = (int)gridDim.x + (int)atomicAdd(sp.work, 1u);
            }
            item = __shfl_sync(0xffffffffu, item, 0);
            if (sp.dbg_state && lane == 0) { sp.dbg_state[blockIdx.x * 16 + 0] = item; sp.dbg_state[blockIdx.x * 16 + 1] = seq; }
            if (item >= n_items) break;
            if (dts && lane == 0 && seq == 0) dts[1] = globaltimer();
            const bool score = item < sp.n_score;
            int row, part, a, len;
            if (score) {
                row = item / sp.spr;
                part = item % sp.spr;
                a = part * sp.sch;
                len = min(sp.mtiles, a + sp.sch) - a;
            } else {
                row = (item - sp.n_score) / sp.ipr;
                part = (item - sp.n_score) % sp.ipr;
                a = part * sp.is;
                len = min(sp.tpr, a + sp.is) - a;
            }
            const int b = row / p.Hkv, g = row % p.Hkv;
            const int L = p.seq_lens[b];
            int cnt = 0;
            const int *ids = p.sel_ids + (size_t)row * p.sel_stride;
            if (!score) {
                if (sp.ready) {
                    if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 2] = row;
                    if (lane == 0)
                        while (ld_acquire_u32(sp.ready + row) == 0) nanosleep_ns(32);
                    __syncwarp();
                    if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 2] = -1;
                }
                cnt = __ldcg(p.sel_count + row);
                PIPE_CHECK(cnt >= 0 && cnt <= p.sel_stride, 3, cnt);
            }
            const int P = (L + p.S - 1) / p.S;  // decode mode is unsharded
            const int lpad = (len + NC - 1) / NC * NC;
            if (lane == 0) items[seq % SM::kItemRing] = make_int4(row, part, score ? 1 : 0, 0);
            for (int x0 = 0; x0 < lpad; x0 += 32) {
                const int x = x0 + lane;
                int src = 0, nv = 0;
                if (x < len) {
                    if (score) {  // metadata tile: 16 pages from page (a + x) * 16
                        const int page0 = (a + x) * 16;
                        nv = max(0, min(16, P - page0));
                        src = row * p.max_pages + page0;  // in 256-byte page records
                    } else {
                        const int sl = a + x;
                        const int u = sl / TPP, sub = sl % TPP;
                        if (u < cnt) {
                            const int gid = __ldcg(ids + u);
                            PIPE_CHECK(gid >= 0 && gid < P, 1, gid);
                            if (gid >= 0 && gid % p.stride == p.offset) {
                                const int blk = p.page_table[(size_t)b * p.max_pages + gid / p.stride];
                                PIPE_CHECK(blk >= 0 && blk < p.num_blocks, 2, blk);
                                nv = max(0, min(TT, min(p.S, L - gid * p.S) - sub * TT));
                                src = (blk * p.Hkv + g) * p.S + sub * TT;  // tensor-map row
                            }
                        }
                    }
                }
                const int nb = min(32, lpad - x0);
                if (lane == 0)
                    while (head + nb - *vdtail > DR) nanosleep_ns(32);
                __syncwarp();
                if (lane < nb) {
                    const int flags = (x < NC ? kFirst : 0) | (x >= lpad - NC ? kLast : 0) |
                                      (score ? kScoreTile : 0);
                    desc[(head + lane) % DR] = make_int4(src, nv | flags, seq, x);
                }
                head += nb;
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    *vdhead = head;
                    if (sp.dbg_state) sp.dbg_state[blockIdx.x * 16 + 3] = head;
                    if (dts && seq == 0 && x0 == 0) dts[2] = globaltimer();
                }
            }
            ++seq;
        }
        if (lane == 0) {  // NC end markers (one per consumer); item count for the merge warp
            *reinterpret_cast<volatile int *>(&s_nitems) = seq;
            while (head + NC - *vdtail > DR) nanosleep_ns(32);
            for (int c = 0; c < NC; ++c) desc[(head + c) % DR] = make_int4(0, kEnd, seq, 1);
            __threadfence_block();
            *vdhead = head + NC;
            *reinterpret_cast<volatile int *>(&s_total) = head + NC;
            __threadfence();  // the last CTA out re-arms the work counter for the next launch
            if (atomicAdd(sp.work + 1, 1u) == gridDim.x - 1) {
                sp.work[0] = 0u;
                sp.work[1] = 0u;
            }
            if (sp.dbg_state) sp.dbg_state[blockIdx.x * 16 + 3] = -99;
        }
        return;
    }

    if (warp == NC + 2) {
        pipe_merge_warp<NC, STAGES>(sp, smem, s_arrive, s_merged, &s_nitems);
        if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 6] = -99;
        if (dts && lane == 0) dts[7] = globaltimer();
        return;
    }

    if (warp == NC) {
        // =================================== TMA ===================================
        // Lane-parallel issue: lane l owns slot i + l of each batch of kBatch slots (its
        // own stage, empty-wait, info, expect_tx and copies), so the per-stage wait/issue
        // latency is paid once per batch instead of once per stage.
        constexpr int kBatch = STAGES / 2;
        const uint64_t pol = l2_policy_evict_first();
        const int qbytes = p.G * kAttnD * 2;
        volatile int *vtotal = &s_total;
        for (int i0 = 0;;) {
            // a batch = the descriptors already published, up to kBatch: never wait for a
            // full batch (the scheduler may be blocked on a row these very slots complete)
            int n = 0;
            if (lane == 0) {
                for (;;) {
                    const int h = *vdhead;
                    if (h > i0) { n = min(kBatch, h - i0); break; }
                    const int tot = *vtotal;
                    if (tot >= 0 && i0 >= tot) break;
                    nanosleep_ns(20);
                }
            }
            n = __shfl_sync(0xffffffffu, n, 0);
            if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 4] = i0 + n;
            if (n == 0) break;  // every descriptor (end markers included) has been issued
            const int i = i0 + lane;
            const bool mine = lane < n;
            int4 d = make_int4(0, 0, 0, 0);
            if (mine) {
                volatile int *dv = reinterpret_cast<volatile int *>(desc + i % DR);
                d = make_int4(dv[0], dv[1], dv[2], dv[3]);
            }
            __syncwarp();
            if (lane == 0) *vdtail = i0 + n;
            // first slot of an item: Q group -> qbuf[seq & 1]
            if (mine && !(d.y & kEnd) && d.w == 0) {
                const int par = d.z & 1, use = d.z >> 1;
                if (sp.dbg_state) sp.dbg_state[blockIdx.x * 16 + 5] = 1000000 + d.z;
                const int row = reinterpret_cast<volatile int *>(items + d.z % SM::kItemRing)[0];
                const int b = row / p.Hkv, g = row % p.Hkv;
                mbar_wait(qempty0 + 8 * par, (use & 1) ^ 1);
                mbar_arrive_expect_tx(qfull0 + 8 * par, qbytes);
                bulk_load(sb + SM::kQ + par * 8 * kRowBytes,
                          static_cast<const uint16_t *>(p.q) + ((size_t)b * p.Hq + g * p.G) * kAttnD,
                          qbytes, qfull0 + 8 * par);
            }
            if (mine) {
                const uint32_t st = i % STAGES;
                if (sp.dbg_state) sp.dbg_state[blockIdx.x * 16 + 5] = i;
                mbar_wait(empty0 + 8 * st, ((i / STAGES) & 1) ^ 1);
                info[st] = make_int4(d.y, d.z, d.w, 0);
                const int nv = d.y & 0xff;
                const uint32_t dst = sb + st * SM::kStage;
                if (!(d.y & kEnd) && nv > 0) {
                    PIPE_CHECK(d.x >= 0, 6, d.x);
                    if (d.y & kScoreTile) {
                        PIPE_CHECK(d.x + nv <= p.B * p.Hkv * p.max_pages, 7, d.x);
                        const uint32_t bytes = nv * 2 * kRowBytes;
                        mbar_arrive_expect_tx(full0 + 8 * st, bytes);
                        bulk_load_hint(dst, sp.meta + (size_t)d.x * 2 * kAttnD, bytes, full0 + 8 * st, pol);
                    } else {
                        mbar_arrive_expect_tx(full0 + 8 * st, kStageTx);
                        tma_load_2d(dst, &tmK, 0, d.x, full0 + 8 * st, pol);
                        tma_load_2d(dst + SM::kTile, &tmV, 0, d.x, full0 + 8 * st, pol);
                    }
                    if (dts && i == 0) dts[3] = globaltimer();
                } else {
                    mbar_arrive(full0 + 8 * st);  // empty slot or end marker
                }
            }
            __syncwarp();
            i0 += n;
        }
        if (dts && lane == 0) dts[6] = globaltimer();
        if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 4] = -99;
        return;
    }

    // ================================= consumers =================================
    const int gid = lane >> 2, t = lane & 3;
    const float sl2 = p.scale * kLog2e;
    uint32_t qa[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // attention: Q fragments; score: q^-
    uint32_t qp[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // score: q^+
    float m = kNegInf, lpart = 0.f;
    float oacc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
    for (int i = warp;; i += NC) {
        const uint32_t st = i % STAGES;
        if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 8 + warp] = i;
        mbar_wait(full0 + 8 * st, (i / STAGES) & 1);
        const int4 inf = info[st];
        const int flags = inf.x, seq = inf.y, tile = inf.z, nv = flags & 0xff;
        PIPE_CHECK((flags & kEnd) || (tile >= 0 && tile < 64 && nv <= 16), 4, tile * 1000 + nv);
        if (sp.dbg_ts && blockIdx.x < 4 && i < 256 && lane == 0)
            sp.dbg_ts[16384 + 4096 + blockIdx.x * 256 + i] = globaltimer();
        if (dts && i == 0 && lane == 0) dts[4] = globaltimer();
        if (flags & kEnd) {
            if (dts && warp == 0 && lane == 0) dts[5] = globaltimer();
            if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 8 + warp] = -99;
            break;
        }
        const int par = seq & 1, sl = seq % SM::kNSlot;
        const bool score = flags & kScoreTile;
        float *slot = scratch + sl * SM::kSlotFloats;
        if (flags & kFirst) {  // item start: slot free?  Q fragments, fresh accumulators
            if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 8 + warp] = -(1000000 + seq);
            if (seq >= SM::kNSlot)
                while (*reinterpret_cast<volatile int *>(&s_merged[sl]) < seq - SM::kNSlot + 1)
                    nanosleep_ns(20);
            if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 8 + warp] = -(2000000 + seq);
            mbar_wait(qfull0 + 8 * par, (seq >> 1) & 1);
            const uint32_t qrow = sb + SM::kQ + par * 8 * kRowBytes + gid * kRowBytes;
            const bool live = gid < p.G;
            if (score) {  // q channels 8t.., 8(t+4).. -> q^- (min part), q^+ (max part)
                const uint4 x0 = live ? lds_v4(qrow + 16 * t) : make_uint4(0, 0, 0, 0);
                const uint4 x1 = live ? lds_v4(qrow + 16 * (t + 4)) : make_uint4(0, 0, 0, 0);
                const uint32_t w0[4] = {x0.x, x0.y, x0.z, x0.w}, w1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    qa[e] = bf16x2_min0(w0[e]);      // record chunk t      (min part): q^-
                    qa[4 + e] = bf16x2_min0(w1[e]);  // record chunk t + 4  (min part): q^-
                    qp[e] = bf16x2_max0(w0[e]);      // record chunk t + 8  (max part): q^+
                    qp[4 + e] = bf16x2_max0(w1[e]);  // record chunk t + 12 (max part): q^+
                }
            } else {
                const uint4 x0 = live ? lds_v4(qrow + 32 * t) : make_uint4(0, 0, 0, 0);
                const uint4 x1 = live ? lds_v4(qrow + 32 * t + 16) : make_uint4(0, 0, 0, 0);
                qa[0] = x0.x; qa[1] = x0.y; qa[2] = x0.z; qa[3] = x0.w;
                qa[4] = x1.x; qa[5] = x1.y; qa[6] = x1.z; qa[7] = x1.w;
                m = kNegInf;
                lpart = 0.f;
#pragma unroll
                for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(qempty0 + 8 * par);
        }
        const uint32_t kb = sb + st * SM::kStage;
        if (score) {
            // ---- Eq. 2 for 16 pages: A rows = [m | M] records (256 B, unswizzled), B =
            // [q^- ; q^+]; thread chunks t + 4i of the record, k-step s uses chunk s/2.
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if (nv > 0 && !(sp.dbg & 1)) {
#pragma unroll
                for (int ci = 0; ci < 4; ++ci) {
                    const uint4 lo = lds_v4(kb + gid * 2 * kRowBytes + 16 * (t + 4 * ci));
                    const uint4 hi = lds_v4(kb + (gid + 8) * 2 * kRowBytes + 16 * (t + 4 * ci));
                    // coefficients of record chunk t + 4ci (pairs 0..3)
                    const uint32_t *cf = ci < 2 ? qa + 4 * ci : qp + 4 * (ci - 2);
                    const uint32_t b0 = cf[0], b1 = cf[1], b2 = cf[2], b3 = cf[3];
                    mma_bf16_16816(acc, lo.x, hi.x, lo.y, hi.y, b0, b1);
                    mma_bf16_16816(acc, lo.z, hi.z, lo.w, hi.w, b2, b3);
                }
            }
            const bool c0 = 2 * t < p.G, c1 = 2 * t + 1 < p.G;
            float m0 = fmaxf(c0 ? acc[0] : kNegInf, c1 ? acc[1] : kNegInf);
            float m1 = fmaxf(c0 ? acc[2] : kNegInf, c1 ? acc[3] : kNegInf);
            m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 1));
            m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, 2));
            m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
            m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
            if (t < 2) {
                const int pg = gid + 8 * t;
                slot[tile * 16 + pg] = pg < nv ? (t ? m1 : m0) + 0.0f : kNegInf;
            }
        } else if (nv > 0 && !(sp.dbg & 1)) {
            const uint32_t vb = kb + SM::kTile;
            if (nv < TT) {  // zero V rows past seq_len (0 * garbage must not make NaN)
                for (int c = lane; c < (TT - nv) * 8; c += 32)
                    sts_v4(vb + nv * kRowBytes + c * 16, make_uint4(0, 0, 0, 0));
                fence_proxy_async();  // generic writes before the next TMA write of the stage
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
        if (sp.dbg_ts && blockIdx.x < 4 && i < 256 && lane == 0)
            sp.dbg_ts[16384 + blockIdx.x * 1024 + i * 2 + 1] = globaltimer();
        if (!(flags & kLast)) continue;

        // ---- item end: attention partial into the slot (scores are already there)
        if (!score) {
            const float lrow = lpart + __shfl_xor_sync(0xffffffffu, lpart, 1);
            const float lsum = lrow + __shfl_xor_sync(0xffffffffu, lrow, 2);
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
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            atomicAdd(&s_arrive[sl], 1);
        }
    }
}

// Merge / select warp (see the header comment).
template <int NC, int STAGES>
TS_DEV void pipe_merge_warp(const PipeParams &sp, uint8_t *smem, int *s_arrive, int *s_merged,
                            const int *s_nitems) {
    using SM = PipeSmem<NC, STAGES>;
    const AttnParams &p = sp.a;
    const int lane = threadIdx.x & 31;
    const int4 *items = reinterpret_cast<const int4 *>(smem + SM::kItems);
    float *scratch = reinterpret_cast<float *>(smem + SM::kScratch);
    static_assert(SM::kSlotFloats >= 2 * SM::kSelKeys, "candidate merge reuses the item slot");
    for (int seq = 0;; ++seq) {
        const int sl = seq % SM::kNSlot;
        if (sp.dbg_state && lane == 0) sp.dbg_state[blockIdx.x * 16 + 6] = seq;
        for (;;) {  // wait for the NC consumers of item seq (or the end of this CTA's items)
            if (*reinterpret_cast<volatile int *>(&s_arrive[sl]) == NC) break;
            const int n = *reinterpret_cast<volatile const int *>(s_nitems);
            if (n >= 0 && seq >= n) return;
            nanosleep_ns(32);
        }
        __threadfence_block();
        const volatile int *itv = reinterpret_cast<const volatile int *>(items + seq % SM::kItemRing);
        const int row = itv[0], part = itv[1], kind = itv[2];
        PIPE_CHECK(row >= 0 && row < p.B * p.Hkv, 5, row);
        const int b = row / p.Hkv, g = row % p.Hkv;
        float *slot = scratch + sl * SM::kSlotFloats;

        if (kind == 1) {
            // ================= score item: top-K of this chunk of pages =================
            const int L = p.seq_lens[b];
            const int P = (L + p.S - 1) / p.S;
            const int page0 = part * sp.sch * 16;
            const int n = max(0, min(P - page0, sp.sch * 16));
            bool publish = sp.spr == 1;
            // development: merge-warp stamps per score item (dbg_ts[12288 + item * 4 + e])
#define STAMP(e)                                                                              \
    if (sp.dbg_ts && lane == 0 && (row * sp.spr + part) < 1024)                               \
        sp.dbg_ts[12288 + (row * sp.spr + part) * 4 + (e)] = globaltimer();
            STAMP(0);
            if (publish) {
                const int kk = warp_topk<16>(slot, nullptr, page0, n, sp.kmax,
                                             sp.sel_out + (size_t)row * sp.kmax, nullptr);
                if (lane == 0) sp.cnt_out[row] = kk;
                STAMP(1);
            } else {
                const size_t cb = ((size_t)row * sp.spr + part) * sp.kmax;
                warp_topk<16>(slot, nullptr, page0, n, sp.kmax, sp.cand_id + cb, sp.cand_sc + cb);
                STAMP(1);
                __threadfence();
                __syncwarp();
                int fin = 0;
                if (lane == 0) fin = atomicAdd(sp.sc_tickets + row, 1u) == unsigned(sp.spr - 1);
                fin = __shfl_sync(0xffffffffu, fin, 0);
                if (fin) {  // global top-K over the union of the chunk candidates
                    __threadfence();
                    const int nc = sp.spr * sp.kmax;  // <= kSelKeys (host-checked)
                    const size_t c0 = (size_t)row * sp.spr * sp.kmax;
                    float *csc = slot;  // the chunk scores are consumed: reuse the slot
                    int *cid = reinterpret_cast<int *>(slot + SM::kSelKeys);
                    // batches of 8 independent loads per lane (one L2 round trip each)
                    for (int i0 = 0; i0 < nc; i0 += 256) {
                        float vs[8];
                        int vi[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int i = i0 + 32 * e + lane;
                            vs[e] = i < nc ? __ldcg(sp.cand_sc + c0 + i) : 0.f;
                            vi[e] = i < nc ? __ldcg(sp.cand_id + c0 + i) : 0;
                        }
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int i = i0 + 32 * e + lane;
                            if (i < nc) {
                                csc[i] = vs[e];
                                cid[i] = vi[e];
                            }
                        }
                    }
                    __syncwarp();
                    STAMP(2);
                    // candidates are ordered by chunk, ids ascending inside a chunk, and the
                    // chunks cover ascending page ranges: index order == page-id order
                    const int kk = warp_topk<16>(csc, cid, 0, nc, sp.kmax,
                                             sp.sel_out + (size_t)row * sp.kmax, nullptr);
                    if (lane == 0) {
                        sp.cnt_out[row] = kk;
                        sp.sc_tickets[row] = 0u;
                    }
                    STAMP(3);
                    publish = true;
                }
            }
            __syncwarp();
            if (lane == 0) {  // slot free again
                s_arrive[sl] = 0;
                __threadfence_block();
                *reinterpret_cast<volatile int *>(&s_merged[sl]) = seq + 1;
            }
            if (publish) {
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    st_release_u32(sp.ready + row, 1u);
                    if (sp.dbg_ts) sp.dbg_ts[4096 + row] = globaltimer();
                    if (sp.dbg_state) {
                        sp.dbg_state[8192 + row * 4 + 0] += 1;
                        sp.dbg_state[8192 + row * 4 + 1] = blockIdx.x * 1000 + seq;
                    }
                }
            }
            continue;
        }

        // ================= attention item: merge the NC partials =================
        const bool whole = sp.ipr == 1;
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
            if (lane == 0 && sp.dbg_state) {
                sp.dbg_state[8192 + row * 4 + 2] += 1;
                sp.dbg_state[8192 + row * 4 + 3] = blockIdx.x * 1000 + seq;
            }
            continue;
        }
        __threadfence();
        __syncwarp();
        int fin = 0;
        if (lane == 0) fin = atomicAdd(p.tickets + row, 1u) == unsigned(sp.ipr - 1);
        fin = __shfl_sync(0xffffffffu, fin, 0);
        if (!fin) continue;
        __threadfence();
        // Row merge of the ipr item partials, written for memory-level parallelism (every
        // load of a phase is independent): (1) lanes (sub, h) = (lane / 8, lane % 8) reduce
        // m and l of parts s = sub (mod 4) -> per-head max M_h and l-sum, weights
        // f[s][h] = exp2(m - M_h) into merge-private smem; (2) each lane accumulates its
        // float4 outputs over all parts.
        const float *pbase = p.part + (size_t)row * sp.ipr * 8 * kPS;
        float *wf = reinterpret_cast<float *>(smem + SM::kHist);
        const int sub = lane >> 3, h8 = lane & 7;
        float Mh = kNegInf;
        if (h8 < p.G)
            for (int s2 = sub; s2 < sp.ipr; s2 += 4)
                Mh = fmaxf(Mh, __ldcg(pbase + (s2 * 8 + h8) * kPS + kAttnD));
        Mh = fmaxf(Mh, __shfl_xor_sync(0xffffffffu, Mh, 8));
        Mh = fmaxf(Mh, __shfl_xor_sync(0xffffffffu, Mh, 16));
        float lh = 0.f;
        if (h8 < p.G)
            for (int s2 = sub; s2 < sp.ipr; s2 += 4) {
                const float *pr = pbase + (s2 * 8 + h8) * kPS;
                const float ms = __ldcg(pr + kAttnD), ls = __ldcg(pr + kAttnD + 1);
                const float f = ms == kNegInf ? 0.f : exp2f(ms - Mh);
                wf[s2 * 8 + h8] = f;
                lh += ls * f;
            }
        lh += __shfl_xor_sync(0xffffffffu, lh, 8);
        lh += __shfl_xor_sync(0xffffffffu, lh, 16);
        __syncwarp();
        for (int xw = lane; xw < p.G * (kAttnD / 4); xw += 32) {
            const int h = xw / (kAttnD / 4), d0 = (xw % (kAttnD / 4)) * 4;
            const float M = __shfl_sync(0xffffffffu, Mh, h);
            const float l = __shfl_sync(0xffffffffu, lh, h);
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
            if (M != kNegInf) {
#pragma unroll 4
                for (int s2 = 0; s2 < sp.ipr; ++s2) {
                    const float f = wf[s2 * 8 + h];
                    const float4 v =
                        __ldcg(reinterpret_cast<const float4 *>(pbase + (s2 * 8 + h) * kPS + d0));
                    acc[0] += v.x * f; acc[1] += v.y * f; acc[2] += v.z * f; acc[3] += v.w * f;
                }
            }
            const size_t oh = (size_t)b * p.Hq + g * p.G + h;
            const float inv = l > 0.f ? 1.f / l : 0.f;
            *reinterpret_cast<float4 *>(p.o + oh * kAttnD + d0) =
                make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
            if (p.lse && d0 == 0) p.lse[oh] = l > 0.f ? (M + log2f(l)) * kLn2 : kNegInf;
        }
        __syncwarp();
        if (lane == 0) {
            p.tickets[row] = 0u;
            if (sp.ready) sp.ready[row] = 0u;
        }
    }
}

}  // namespace ts
