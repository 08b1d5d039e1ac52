// attn.cuh — shared attention definitions + the fp32 CUDA-core path and the LSE merge
// (SparseAttn PAPER.md:169-172; Alg. 1 Steps 3-4).
//
// bf16 tensor-core attention (step_cluster.cuh, sparse_attn.cuh) fragment maps, lane =
// (gid = lane / 4, t = lane % 4):
//   S = Q K^T   : mma.m16n8k16 bf16; A rows = the G q heads of the kv group (rows >= G are
//                 zero), k-slot permutation d = 16t + 4s + {0..3} so that a thread's two
//                 128-bit smem reads of a K row feed all four k16 steps; B = K^T (n = 8
//                 tokens).  The lane ends with head gid's scores of tokens 2t, 2t+1 (+8).
//   O^T += V^T P^T : mma.m16n8k16 (or m16n8k8 for 8-token octets) bf16; B = P^T exactly as
//                 the lane holds it (k = its tokens, n = head gid) as a hi + lo bf16 pair
//                 (16 significant bits; reading R10), A = V^T with rows = channels
//                 8 gid + 2 db (rows gid) and 8 gid + 2 db + 1 (rows gid + 8), built by PRMT
//                 from the lane's 128-bit reads of its V rows (channels 8 gid .. 8 gid + 7).
//                 The lane accumulates channels (8 gid + 2 db, + 1) x heads (2t, 2t + 1).
// fp32 path (attn_simt_kernel): CUDA-core FFMA, one warp per q head, lane-parallel dot
// products with a fixed shuffle tree (no tf32 anywhere; reading R10).
#pragma once
#include "common.cuh"

namespace ts {

struct AttnParams {
    const void *q;
    const void *k_pool;  // [NB][Hkv][S][D] (sparse_attn.cuh; the SIMT / pipeline kernels take them as arguments)
    const void *v_pool;
    const int *page_table;
    const int *seq_lens;
    const int *sel_ids;
    const int *sel_count;
    const int *sel_blk;  // nullable: physical block of each selected page (fused step)
    int sel_stride;
    int B, Hq, Hkv, G, D, S, max_pages, stride, offset, num_blocks;
    float scale;       // softmax scale (reading R1)
    float *o;
    float *lse;        // nullable
    float *part;       // [rows][splits][8][kPS]
    unsigned *tickets; // [rows]
    int splits, items;
    unsigned long long *dbg;  // development: per-CTA globaltimer stamps (nullable)
    int dense;                // 1: attend every page (FullCache baseline), sel_* unused
    // ts_shard_attend (sequence sharding): the selection is the global top-k
    // over `cand_parts` candidate lists (part q of row r: cand_k entries at
    // q * cand_part_stride + r * cand_k; -inf = none), merged in the kernel's prologue;
    // rank-0 CTAs write it to sel_out / sel_cnt_out (nullable)
    const float *cand_scores;
    const int *cand_ids;
    int cand_parts, cand_k;
    long long cand_part_stride;
    int *sel_out, *sel_cnt_out;
};

constexpr int kAttnD = 64;        // head_dim of the tensor-core path
constexpr int kRowBytes = kAttnD * 2;
constexpr int kPS = kAttnD + 4;   // floats per (split, head) partial: o[D], m, l, pad (16 B aligned)

// ------------------------------------------------------------------ O^T = V^T P^T helpers
// rescale the lane's O^T entries (heads 2t, 2t+1) by their heads' factors (held by lanes 4h)
TS_DEV void ot_rescale(float (&oacc)[4][4], float corr, int t) {
    const float c0 = __shfl_sync(0xffffffffu, corr, 8 * t), c1 = __shfl_sync(0xffffffffu, corr, 8 * t + 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        oacc[j][0] *= c0; oacc[j][1] *= c1; oacc[j][2] *= c0; oacc[j][3] *= c1;
    }
}
// 16-token tile: vr[nt][q2] = the lane's 16-byte read (channels 8 gid .. + 7) of the V row of
// its k-slot nt * 8 + 2t + q2 (zeroed past seq_len), pr[nt][q2] = that token's weight
TS_DEV void ot_pv_tile_bf16(float (&oacc)[4][4], const uint4 (&vr)[2][2], const float (&pr)[2][2]) {
    const uint32_t ph0 = bf16x2_pack(pr[0][0], pr[0][1]), ph1 = bf16x2_pack(pr[1][0], pr[1][1]);
    const uint32_t pl0 = bf16x2_pack(pr[0][0] - bf16lo_to_f32(ph0), pr[0][1] - bf16hi_to_f32(ph0));
    const uint32_t pl1 = bf16x2_pack(pr[1][0] - bf16lo_to_f32(ph1), pr[1][1] - bf16hi_to_f32(ph1));
#pragma unroll
    for (int db = 0; db < 4; ++db) {
        const uint32_t wa0 = u4_word(vr[0][0], db), wb0 = u4_word(vr[0][1], db);
        const uint32_t wa1 = u4_word(vr[1][0], db), wb1 = u4_word(vr[1][1], db);
        const uint32_t a0 = __byte_perm(wa0, wb0, 0x5410), a1 = __byte_perm(wa0, wb0, 0x7632);
        const uint32_t a2 = __byte_perm(wa1, wb1, 0x5410), a3 = __byte_perm(wa1, wb1, 0x7632);
        mma_bf16_16816(oacc[db], a0, a1, a2, a3, ph0, ph1);
        mma_bf16_16816(oacc[db], a0, a1, a2, a3, pl0, pl1);
    }
}
// 8-token octet (k = tokens 2t, 2t+1 only): mma.m16n8k8
TS_DEV void ot_pv_octet_bf16(float (&oacc)[4][4], uint4 v0, uint4 v1, float p0, float p1) {
    const uint32_t ph = bf16x2_pack(p0, p1);
    const uint32_t pl = bf16x2_pack(p0 - bf16lo_to_f32(ph), p1 - bf16hi_to_f32(ph));
#pragma unroll
    for (int db = 0; db < 4; ++db) {
        const uint32_t wa = u4_word(v0, db), wb = u4_word(v1, db);
        const uint32_t a0 = __byte_perm(wa, wb, 0x5410), a1 = __byte_perm(wa, wb, 0x7632);
        mma_bf16_1688(oacc[db], a0, a1, ph);
        mma_bf16_1688(oacc[db], a0, a1, pl);
    }
}
// the warp's partial for heads 2t, 2t+1 (< G) into wpart[(warp * 8 + h) * ld + channel]
TS_DEV void ot_store(float *wpart_warp, int ld, const float (&oacc)[4][4], int gid, int t, int G, float s = 1.f) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
        if (2 * t + hh < G) {
            float *wr = wpart_warp + (2 * t + hh) * ld + 8 * gid;
#pragma unroll
            for (int db = 0; db < 4; ++db)
                *reinterpret_cast<float2 *>(wr + 2 * db) = make_float2(oacc[db][hh] * s, oacc[db][2 + hh] * s);
        }
    }
}

// ------------------------------------------------------------------ fp32 CUDA-core path
// grid = rows (b, g); block = 32 * min(G, 8) threads; warp w handles q heads w, w+8, ...
template <int D>
__global__ void __launch_bounds__(256) attn_simt_kernel(AttnParams p, const float *__restrict__ k_pool,
                                                        const float *__restrict__ v_pool) {
    pdl_launch_dependents();
    pdl_wait();
    constexpr int E = D / 32;  // elements per lane: d = lane + 32 e
    const int row = blockIdx.x;
    const int b = row / p.Hkv, g = row % p.Hkv;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int L = clamp_len(p.seq_lens[b], p.max_pages, p.stride, p.S);
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
            const int blk = checked_block(p.page_table[(size_t)b * p.max_pages + j / p.stride], p.num_blocks);
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
    pdl_launch_dependents();
    pdl_wait();
    const int r = blockIdx.x;
    if (parts <= 64) {
        // warp 0 reads the <= 64 partial lse values in one round (two per lane), reduces max and
        // sum by shuffles and publishes the normalised weights w_q = exp(lse_q - lse); every
        // thread then sums its channel over the parts with the loads in flight together
        __shared__ float w[64];
        __shared__ float s_tot;
        if (threadIdx.x < 32) {
            const int q0 = threadIdx.x, q1 = threadIdx.x + 32;
            const float a = q0 < parts ? lse_parts[q0 * sl + r] : kNegInf;
            const float b = q1 < parts ? lse_parts[q1 * sl + r] : kNegInf;
            float M = fmaxf(a, b);
#pragma unroll
            for (int o2 = 16; o2; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
            float l = M != kNegInf ? (a != kNegInf ? expf(a - M) : 0.f) + (b != kNegInf ? expf(b - M) : 0.f) : 0.f;
#pragma unroll
            for (int o2 = 16; o2; o2 >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o2);
            const float tot = M != kNegInf ? M + logf(l) : kNegInf;
            w[q0] = a != kNegInf ? expf(a - tot) : 0.f;
            w[q1] = b != kNegInf ? expf(b - tot) : 0.f;
            if (threadIdx.x == 0) s_tot = tot;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < d; i += blockDim.x) {
            float acc = 0.f;
#pragma unroll 8
            for (int q = 0; q < parts; ++q) {
                const float wq = w[q];
                if (wq != 0.f) acc += wq * o_parts[q * so + (size_t)r * d + i];
            }
            o[(size_t)r * d + i] = acc;
        }
        if (threadIdx.x == 0 && lse) lse[r] = s_tot;
        return;
    }
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
