// tcgen05 vs mma.sync for the decode-attention contraction S = Q K^T (development tool,
// VERDICT r1 item 9).  One CTA per SM, 4 consumer warps, a 128-token K block [128][64] bf16
// (128-byte swizzled rows, as the TMA ring holds it) and the G = 8 query heads [8][64] bf16
// in shared memory; each iteration computes the 128 x 8 score block:
//   A (legacy): every warp runs the fused kernel's QK^T on its 2 x 16-token tiles
//               (mma.sync.m16n8k16, 8 HMMA per tile), scores in registers;
//   B (tcgen05): one thread issues 4 x tcgen05.mma.cta_group::1.kind::f16 (M = 128 tokens,
//               N = 8 heads, K = 16) from smem descriptors into TMEM, commits to an mbarrier;
//               the 4 warps wait and tcgen05.ld their 32 tokens x 8 heads (32x32b.x8).
// Reports cycles per 128-token block for each and the max |S_A - S_B| (both fp32 accumulate).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tcgen05bench scripts/tcgen05bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define DEV __device__ __forceinline__

DEV uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
DEV uint4 lds_v4(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}
DEV void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
DEV void mbar_init(uint32_t bar, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(n)); }
DEV void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

// smem matrix descriptor (sm100 UMMA): K-major, 128-byte swizzle, 8-row groups 1024 B apart
DEV uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);          // start address >> 4, bits [0,14)
    d |= (uint64_t)1 << 16;                           // leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                 // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                           // version (sm100)
    d |= (uint64_t)2 << 61;                           // layout: SWIZZLE_128B
    return d;
}
// instruction descriptor kind::f16: D f32, A / B bf16, K-major both, N = 8, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((8u >> 3) << 17) | ((128u >> 4) << 24);

DEV void umma_f16(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}

template <int MODE>  // 0 = mma.sync, 1 = tcgen05 (serial), 2 = tcgen05 double-buffered (issue block i+1 before reading i)
__global__ void __launch_bounds__(128) bench(const uint16_t *kg, const uint16_t *qg, int iters,
                                             float *out, unsigned long long *cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t *base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
    const uint32_t kb = smem_u32(base), qb = kb + 128 * 128, bar = qb + 1024, bar2 = bar + 8;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // stage K [128][64] and q [8][64] with the 128-byte swizzle (16 B chunk c of row r at c ^ (r & 7))
    for (int i = tid; i < 128 * 8; i += 128) {
        const int r = i >> 3, c = i & 7;
        *reinterpret_cast<uint4 *>(base + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4 *>(kg)[i];
    }
    for (int i = tid; i < 8 * 8; i += 128) {
        const int r = i >> 3, c = i & 7;
        *reinterpret_cast<uint4 *>(base + 128 * 128 + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4 *>(qg)[i];
    }
    if (tid == 0) { mbar_init(bar, 1); mbar_init(bar2, 1); }
    if (MODE >= 1 && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = MODE >= 1 ? tmem_base : 0u;
    if (MODE == 2 && tid == 0) {  // prologue: block 0 into columns [0, 8)
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_f16(tm, sw128_desc(kb + 32 * k), sw128_desc(qb + 32 * k), kIdesc, k > 0);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    }
    const int gid = lane >> 2, t = lane & 3;
    float acc = 0.f;
    float s[8];
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
            // q fragments: head gid, channels 16t .. 16t + 15 (k-slot permutation of the kernel)
            const uint32_t qrow = qb + gid * 128;
            const uint4 x0 = lds_v4(qrow + (((2 * t) ^ (gid & 7)) << 4)), x1 = lds_v4(qrow + (((2 * t + 1) ^ (gid & 7)) << 4));
#pragma unroll
            for (int tile = 0; tile < 2; ++tile) {
                const int tb = (warp * 2 + tile) * 16;
                float sacc[2][4];
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    sacc[nt][0] = sacc[nt][1] = sacc[nt][2] = sacc[nt][3] = 0.f;
                    const int r = tb + nt * 8 + gid;
                    const uint4 k0 = lds_v4(kb + r * 128 + (((2 * t) ^ (r & 7)) << 4));
                    const uint4 k1 = lds_v4(kb + r * 128 + (((2 * t + 1) ^ (r & 7)) << 4));
                    mma16816(sacc[nt], x0.x, 0u, x0.y, 0u, k0.x, k0.y);
                    mma16816(sacc[nt], x0.z, 0u, x0.w, 0u, k0.z, k0.w);
                    mma16816(sacc[nt], x1.x, 0u, x1.y, 0u, k1.x, k1.y);
                    mma16816(sacc[nt], x1.z, 0u, x1.w, 0u, k1.z, k1.w);
                }
                // keep: token tb + nt*8 + 2t + q2, head gid
                if (it == iters - 1) {
#pragma unroll
                    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                        for (int q2 = 0; q2 < 2; ++q2)
                            out[((size_t)blockIdx.x * 128 + tb + nt * 8 + 2 * t + q2) * 8 + gid] = sacc[nt][q2];
                }
                acc += sacc[0][0] + sacc[1][1];
            }
        } else if (MODE == 2) {
            const uint32_t cur = (it & 1) * 8, nxt = ((it + 1) & 1) * 8;
            if (tid == 0 && it + 1 < iters) {  // block it+1 into the other column set
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_f16(tm + nxt, sw128_desc(kb + 32 * k), sw128_desc(qb + 32 * k), kIdesc, k > 0);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"((it + 1) & 1 ? bar2 : bar) : "memory");
            }
            mbar_wait((it & 1) ? bar2 : bar, (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(tm + cur + ((uint32_t)(warp * 32) << 16)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j) s[j] = __uint_as_float(r[j]);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            if (it == iters - 1)
#pragma unroll
                for (int j = 0; j < 8; ++j) out[((size_t)blockIdx.x * 128 + warp * 32 + lane) * 8 + j] = s[j];
            acc += s[0] + s[7];
            __syncthreads();  // columns `cur` are free for block it+2
        } else {
            if (warp == 0 && lane == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int k = 0; k < 4; ++k)  // K = 16 channels = 32 bytes per step along the row
                    umma_f16(tm, sw128_desc(kb + 32 * k), sw128_desc(qb + 32 * k), kIdesc, k > 0);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
            }
            mbar_wait(bar, it & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(tm + ((uint32_t)(warp * 32) << 16)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 8; ++j) s[j] = __uint_as_float(r[j]);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (it == iters - 1)
#pragma unroll
                for (int j = 0; j < 8; ++j) out[((size_t)blockIdx.x * 128 + warp * 32 + lane) * 8 + j] = s[j];
            acc += s[0] + s[7];
            __syncthreads();  // TMEM columns reused by the next iteration's MMA
        }
    }
    unsigned long long t1 = clock64();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 1.2345f) out[0] = acc;
    if (MODE >= 1) {
        __syncthreads();
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
    }
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7fff + ((u >> 16) & 1)) >> 16); }

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<uint16_t> hk(128 * 64), hq(8 * 64);
    srand(1);
    for (auto &x : hk) x = f2bf((rand() / (float)RAND_MAX - 0.5f) * 4);
    for (auto &x : hq) x = f2bf((rand() / (float)RAND_MAX - 0.5f) * 4);
    uint16_t *dk, *dq;
    float *o0, *o1;
    unsigned long long *cyc;
    cudaMalloc(&dk, hk.size() * 2); cudaMalloc(&dq, hq.size() * 2);
    cudaMemcpy(dk, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice);
    cudaMalloc(&o0, sms * 128 * 8 * 4); cudaMalloc(&o1, sms * 128 * 8 * 4);
    cudaMalloc(&cyc, sms * 8);
    const size_t smb = 1024 + 128 * 128 + 1024 + 64;
    cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    const int iters = 2000;
    const char *names[3] = {"mma.sync m16n8k16 (64 HMMA, 4 warps)", "tcgen05.mma M128 N8 x4, serial issue->commit->wait->ld",
                            "tcgen05.mma M128 N8 x4, double-buffered TMEM (issue i+1 before ld of i)"};
    for (int bps : {1, 4}) {
        const int grid = sms * bps;
        std::vector<unsigned long long> c(grid);
        cudaFree(cyc); cudaMalloc(&cyc, grid * 8);
        cudaFree(o0); cudaFree(o1); cudaMalloc(&o0, grid * 128 * 8 * 4); cudaMalloc(&o1, grid * 128 * 8 * 4);
        for (int mode = 0; mode < 3; ++mode) {
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) bench<0><<<grid, 128, smb>>>(dk, dq, iters, o0, cyc);
                else if (mode == 1) bench<1><<<grid, 128, smb>>>(dk, dq, iters, o1, cyc);
                else bench<2><<<grid, 128, smb>>>(dk, dq, iters, o1, cyc);
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
            cudaMemcpy(c.data(), cyc, grid * 8, cudaMemcpyDeviceToHost);
            double mean = 0;
            for (auto x : c) mean += x;
            mean /= grid;
            printf("%d CTA/SM  %-75s %7.1f cycles per block per CTA, %6.1f per block per SM\n", bps, names[mode],
                   mean / iters, mean / iters / bps);
        }
    }
    std::vector<float> a(sms * 128 * 8), b(sms * 128 * 8);
    cudaMemcpy(a.data(), o0, a.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), o1, b.size() * 4, cudaMemcpyDeviceToHost);
    double md = 0, mref = 0;
    for (size_t i = 0; i < 128 * 8; ++i) {  // CTA 0 vs a double reference
        const int tok = i / 8, h = i % 8;
        double ref = 0;
        for (int d = 0; d < 64; ++d) {
            uint32_t uk = (uint32_t)hk[tok * 64 + d] << 16, uq = (uint32_t)hq[h * 64 + d] << 16;
            float fk, fq; memcpy(&fk, &uk, 4); memcpy(&fq, &uq, 4);
            ref += (double)fk * fq;
        }
        md = fmax(md, fabs(a[i] - b[i]));
        mref = fmax(mref, fabs(b[i] - ref));
    }
    printf("max |S_mma.sync - S_tcgen05| = %.3g, max |S_tcgen05 - S_double| = %.3g\n", md, mref);
    return 0;
}
