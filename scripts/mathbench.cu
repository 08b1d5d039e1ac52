// Per-tile cost of the attention consumer math (development tool): every warp runs the
// S = Q K^T / online softmax / O += P V sequence of the TMA consumer on a [16 x 64] K and V
// tile resident in shared memory, `iters` times; reports cycles per tile per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_12211_b200/csrc -o /tmp/mathb scripts/mathbench.cu
#include <cstdio>
#include "common.cuh"
#include "attn.cuh"
using namespace ts;
__global__ void tiles(int iters, float *out, long long *cyc, int L) {
    __shared__ __align__(1024) uint8_t sm[4096];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u ^ (i * 2654435761u & 0x00ff00ffu);
    __syncthreads();
    const uint32_t kb = smem_u32(sm), vb = kb + 2048;
    const int lane = threadIdx.x & 31, gid = lane >> 2, t = lane & 3;
    uint32_t qa[8];
    for (int i = 0; i < 8; ++i) qa[i] = 0x3f803f80u + i + lane;
    float m = kNegInf, lp = 0.f, oacc[8][4];
    for (int j = 0; j < 8; ++j) oacc[j][0] = oacc[j][1] = oacc[j][2] = oacc[j][3] = 0.f;
    const float sl2 = 0.125f * kLog2e;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int tok0 = it * 16;
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
        float x[2][2], tmax = kNegInf;
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
        float pr[2][2], psum = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int q2 = 0; q2 < 2; ++q2) { pr[nt][q2] = exp2f(x[nt][q2] - mref); psum += pr[nt][q2]; }
        lp = lp * corr + psum;
#pragma unroll
        for (int j = 0; j < 8; ++j) { oacc[j][0] *= corr; oacc[j][1] *= corr; }
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            const int q0 = nt * 8 + 2 * t, q1 = q0 + 1;
            uint4 v0 = lds_v4(vb + q0 * kRowBytes + ((gid ^ (q0 & 7)) << 4));
            uint4 v1 = lds_v4(vb + q1 * kRowBytes + ((gid ^ (q1 & 7)) << 4));
            if (tok0 + q0 >= L) v0 = make_uint4(0, 0, 0, 0);
            if (tok0 + q1 >= L) v1 = make_uint4(0, 0, 0, 0);
            const uint32_t a0 = f32_to_tf32(pr[nt][0]), a2 = f32_to_tf32(pr[nt][1]);
            const uint32_t w0[4] = {v0.x, v0.y, v0.z, v0.w}, w1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t b0 = (j & 1) ? (w0[j >> 1] & 0xffff0000u) : (w0[j >> 1] << 16);
                const uint32_t b1 = (j & 1) ? (w1[j >> 1] & 0xffff0000u) : (w1[j >> 1] << 16);
                mma_tf32_1688(oacc[j], a0, 0u, a2, 0u, b0, b1);
            }
        }
    }
    long long t1 = clock64();
    float s = lp + m;
    for (int j = 0; j < 8; ++j) s += oacc[j][0] + oacc[j][1] + oacc[j][2] + oacc[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    float *out; long long *cyc; cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
    for (int warps : {1, 4, 8, 16, 32}) {
        const int iters = 2000;
        tiles<<<148, warps * 32>>>(iters, out, cyc, 1 << 30);
        tiles<<<148, warps * 32>>>(iters, out, cyc, 1 << 30);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%2d warps/SM: %6.1f cycles per tile per warp -> %6.1f tiles per 1000 cycles per SM (%.0f GB/s of K+V at 1.9 GHz, 148 SMs) %s\n",
               warps, (double)c / iters, 1000.0 * warps * iters / c, 4096.0 * warps * iters / c * 1.9e9 * 148 / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
