// attn.cuh — shared attention definitions + the fp32 CUDA-core path and the LSE merge
// (SparseAttn PAPER.md:169-172; Alg. 1 Steps 3-4).
//
// The bf16 tensor-core path (the hot one) is decode_pipe.cuh.  Its fragment maps, used
// there, are:
//   S^T = Q K^T : mma.m16n8k16 bf16; A rows = the G q heads of the kv group (rows >= G are
//                 zero), k-slot permutation d = 16t + 4s + {0..3} so that a thread's two
//                 128-bit smem reads of a K row (logical chunks 2t, 2t+1 of the 128-byte
//                 swizzled row) feed all four k16 steps; B = K^T (n = 8 tokens).
//   O  += P V   : mma.m16n8k8 tf32; A = P straight from the S accumulators with the token
//                 order permuted (k slot t <-> token 2t, t+4 <-> 2t+1); B = V, n-tile j <->
//                 channels {8n + j}, so thread (n, t) reads V rows 2t, 2t+1 chunk n once.
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
    const int8_t *k_exp;      // FP8 KV (reading R21): row exponents [NB][Hkv][S] (else null)
    const int8_t *v_exp;
};

constexpr int kAttnD = 64;        // head_dim of the tensor-core path
constexpr int kRowBytes = kAttnD * 2;
constexpr int kPS = kAttnD + 4;   // floats per (split, head) partial: o[D], m, l, pad (16 B aligned)

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
    pdl_launch_dependents();
    pdl_wait();
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
