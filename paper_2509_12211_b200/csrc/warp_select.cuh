// warp_select.cuh — exact top-K of a row of page scores by ONE warp, keys in registers
// (Alg. 1 Step 2 "radix select"; TopK PAPER.md:162-167).
//
// Lane l holds the orderable keys of entries i = 32 j + l (j < KPL) — entry order is page
// order, so "lower index" is "lower page id" (tie rule, reading R6).  Key 0 marks an
// absent entry (every real key of a finite score is > key(-inf) > 0).
//  * range: kmin / kmax of the live candidates by warp reductions (REDUX);
//  * pass: bucket the candidates by (key - lo) >> shift into <= 256 bins of a warp-private
//    shared-memory histogram, find the bin holding the rem-th largest candidate with one
//    warp suffix scan, take every key above it; stop if the bin is taken whole or is one
//    key value; rank its <= 32 keys exactly by shuffles; else recurse into it (each pass
//    removes >= 8 bits of the range: <= 4 passes);
//  * compaction: per register slot j one ballot of "selected", so the output positions
//    follow entry order (ascending page ids) with no sort.
// No block barrier anywhere: the warp runs beside the streaming warps of its CTA.
#pragma once
#include "common.cuh"

namespace ts {

constexpr int kWsBins = 256;

// scratch: hist [256] int (warp-private shared memory).  emit(pos, entry) writes output
// position pos (0 .. kk-1, ascending entry order).  Returns kk = min(k, #live keys).
template <int KPL, typename Emit>
TS_DEV int warp_select(const uint32_t (&key)[KPL], int k, int *hist, Emit emit) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    int nlive = 0;
    uint32_t kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int j = 0; j < KPL; ++j)
        if (key[j]) {
            ++nlive;
            kmin = min(kmin, key[j]);
            kmax = max(kmax, key[j]);
        }
    nlive = __reduce_add_sync(0xffffffffu, nlive);
    const int kk = min(k, nlive);
    if (kk <= 0) return 0;
    // selected = {key > tgt} + the first need_eq (lowest entry) keys == teq
    uint32_t tgt = 0u, teq = 0xffffffffu;
    int need_eq = 0;
    if (kk < nlive) {
        uint32_t lo = __reduce_min_sync(0xffffffffu, kmin);
        uint32_t hi = __reduce_max_sync(0xffffffffu, kmax);
        int rem = kk;
#pragma unroll 1
        for (;;) {
            if (lo == hi) {  // one key value left: ties by entry order
                tgt = lo;
                teq = lo;
                need_eq = rem;
                break;
            }
            const uint32_t span = hi - lo;
            const int bits = 32 - __clz(span);
            const int shift = bits > 8 ? bits - 8 : 0;
            reinterpret_cast<int4 *>(hist)[2 * lane] = make_int4(0, 0, 0, 0);
            reinterpret_cast<int4 *>(hist)[2 * lane + 1] = make_int4(0, 0, 0, 0);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < KPL; ++j)
                if (key[j] >= lo && key[j] <= hi) atomicAdd(&hist[(key[j] - lo) >> shift], 1);
            __syncwarp();
            // lane owns bins [8 lane, 8 lane + 8): suffix scan from the top bin
            const int4 h0 = reinterpret_cast<const int4 *>(hist)[2 * lane];
            const int4 h1 = reinterpret_cast<const int4 *>(hist)[2 * lane + 1];
            const int c[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
            const int s = c[0] + c[1] + c[2] + c[3] + c[4] + c[5] + c[6] + c[7];
            int suf = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_down_sync(0xffffffffu, suf, o);
                if (lane + o < 32) suf += y;
            }
            const int above_run = suf - s;
            const unsigned hit = __ballot_sync(0xffffffffu, above_run < rem && suf >= rem);
            const int L = __ffs(hit) - 1;
            int bsel = 0, ab = 0, cb = 0;
            {
                int acc = above_run;
                bool done = false;
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    if (!done && acc + c[e] >= rem) {
                        bsel = 8 * lane + e;
                        ab = acc;
                        cb = c[e];
                        done = true;
                    }
                    acc += c[e];
                }
            }
            bsel = __shfl_sync(0xffffffffu, bsel, L);
            ab = __shfl_sync(0xffffffffu, ab, L);
            cb = __shfl_sync(0xffffffffu, cb, L);
            __syncwarp();  // the histogram is reused by the next pass
            const uint32_t blo = lo + ((uint32_t)bsel << shift);
            const uint32_t bhi = shift ? min(hi, blo + ((1u << shift) - 1u)) : blo;
            rem -= ab;
            if (cb == rem) {  // the whole bin is taken: keys >= blo
                tgt = blo - 1u;
                break;
            }
            if (shift == 0) {  // the bin is one key value
                tgt = blo;
                teq = blo;
                need_eq = rem;
                break;
            }
            if (cb <= 32) {  // rank the bin's keys exactly: candidate c -> lane c
                uint32_t ck = 0u;
                int ci = 0x7fffffff, base = 0;
#pragma unroll
                for (int j = 0; j < KPL; ++j) {
                    const bool in = key[j] >= blo && key[j] <= bhi;
                    const unsigned m = __ballot_sync(0xffffffffu, in);
                    // candidate (slot j, lane sl) goes to lane base + #candidates before it
#pragma unroll 1
                    for (unsigned mm = m; mm; mm &= mm - 1) {
                        const int sl = __ffs(mm) - 1;
                        const int dst = base + __popc(m & ((1u << sl) - 1u));
                        const uint32_t kv = __shfl_sync(0xffffffffu, key[j], sl);
                        if (lane == dst) {
                            ck = kv;
                            ci = 32 * j + sl;
                        }
                    }
                    base += __popc(m);
                }
                // rank(c) = #{x : key_x > key_c or (key_x == key_c and entry_x < entry_c)}
                int rk = 0, gtc = 0;
                for (int x = 0; x < cb; ++x) {
                    const uint32_t kx = __shfl_sync(0xffffffffu, ck, x);
                    const int ix = __shfl_sync(0xffffffffu, ci, x);
                    rk += kx > ck || (kx == ck && ix < ci);
                    gtc += kx > ck;
                }
                const unsigned last = __ballot_sync(0xffffffffu, lane < cb && rk == rem - 1);
                const int Ll = __ffs(last) - 1;
                tgt = __shfl_sync(0xffffffffu, ck, Ll);
                teq = tgt;
                need_eq = rem - __shfl_sync(0xffffffffu, gtc, Ll);
                break;
            }
            // recurse into the bin, narrowed to its actual key range
            uint32_t a = 0xffffffffu, z = 0u;
#pragma unroll
            for (int j = 0; j < KPL; ++j)
                if (key[j] >= blo && key[j] <= bhi) {
                    a = min(a, key[j]);
                    z = max(z, key[j]);
                }
            lo = __reduce_min_sync(0xffffffffu, a);
            hi = __reduce_max_sync(0xffffffffu, z);
        }
    }
    // compaction in entry order (slot-major, then lane)
    int pos0 = 0, eq0 = 0;
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
        const bool eq = key[j] == teq;
        const unsigned meq = __ballot_sync(0xffffffffu, eq);
        const bool take = key[j] > tgt || (eq && eq0 + __popc(meq & lt) < need_eq);
        const unsigned mt = __ballot_sync(0xffffffffu, take);
        if (take) emit(pos0 + __popc(mt & lt), 32 * j + lane);
        pos0 += __popc(mt);
        eq0 += __popc(meq);
    }
    return kk;
}

}  // namespace ts
