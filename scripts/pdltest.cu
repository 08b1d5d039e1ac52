// Does a PDL secondary start while the primary still runs? (development tool)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pdl scripts/pdltest.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void primary(unsigned long long *ts, int spin_ns, int trigger) {
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    unsigned long long t0 = gt();
    if (threadIdx.x == 0) ts[blockIdx.x] = t0;
    while (gt() - t0 < (unsigned long long)spin_ns) {}
}
__global__ void secondary(unsigned long long *ts) {
    if (threadIdx.x == 0) ts[4096 + blockIdx.x] = gt();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) ts[8192 + blockIdx.x] = gt();
}
int main() {
    unsigned long long *ts; cudaMalloc(&ts, 16384 * 8);
    cudaStream_t s; cudaStreamCreate(&s);
    for (int trig = 0; trig < 2; ++trig) for (int smem : {0, 40000}) {
        cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(ts, 0, 16384 * 8);
            primary<<<296, 192, smem, s>>>(ts, 20000, trig);
            cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(296); cfg.blockDim = dim3(160); cfg.stream = s;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, secondary, ts);
            cudaStreamSynchronize(s);
        }
        unsigned long long h[16384]; cudaMemcpy(h, ts, sizeof(h), cudaMemcpyDeviceToHost);
        unsigned long long p0 = ~0ull, s0 = ~0ull, s1 = 0, w0 = ~0ull;
        for (int i = 0; i < 296; ++i) { p0 = h[i] < p0 ? h[i] : p0; s0 = h[4096 + i] < s0 ? h[4096 + i] : s0; s1 = h[4096 + i] > s1 ? h[4096 + i] : s1; w0 = h[8192+i] < w0 ? h[8192+i] : w0; }
        printf("trigger %d smem %5d: secondary start first %+.2f us last %+.2f us, after-wait first %+.2f us (primary spins 20 us) %s\n", trig, smem,
               (double)(s0 - p0) / 1e3, (double)(s1 - p0) / 1e3, (double)(w0 - p0) / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
