// topkbench.cu — cycle breakdown of cta_topk (development tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//      -I paper_2509_12211_b200/csrc scripts/topkbench.cu -o /tmp/topkbench && /tmp/topkbench
// One CTA per SM (or `ctas` CTAs), 160 threads, n keys (scores ~ N(40, 3)) in shared memory,
// k selected; clock64 stamps at the cta_topk phase boundaries, averaged over CTAs.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
__device__ long long g_prof[4096 * 16];
#ifdef STOPAT  // return from cta_topk at stage STOPAT: cumulative cost without stamps
#define TS_TOPK_PROF(i) \
    if ((i) == STOPAT) return 0;
#define TS_TOPK_PROF2(i) \
    if ((i) == STOPAT) return 0;
#elif !defined(NOPROF)
#define TS_TOPK_PROF(i) \
    if (threadIdx.x == 0) g_prof[blockIdx.x * 16 + (i)] = clock64();
#define TS_TOPK_PROF2(i) \
    if (threadIdx.x == 0) g_prof[blockIdx.x * 16 + (i)] = clock64();
#endif
#include "score_select.cuh"

using namespace ts;
constexpr int NT = 160;

template <int HB>
__global__ void __launch_bounds__(NT) kern(const float *scores, int n, int k, int *out, int *cnt_out) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint32_t *keys = reinterpret_cast<uint32_t *>(sm);
    int *hist = reinterpret_cast<int *>(sm + ((n + 3) & ~3) * 4);
    int *red = hist + 2048;
    uint32_t *cand = reinterpret_cast<uint32_t *>(red + 64);
    const float *s = scores + (size_t)blockIdx.x * n;
    uint32_t mn = 0xffffffffu, mx = 0u;
    for (int i = threadIdx.x; i < ((n + 3) & ~3); i += NT) {
        const uint32_t key = i < n ? score_key(s[i]) : 0u;
        keys[i] = key;
        if (i < n) { mn = min(mn, key); mx = max(mx, key); }
    }
    for (int i = threadIdx.x; i < 2048; i += NT) hist[i] = 0;
    block_minmax<NT, 0>(mn, mx, red);
    __syncthreads();
    int *o = out + (size_t)blockIdx.x * k;
    const long long t0 = clock64();
    int kk = cta_topk<NT, 0, HB>(keys, n, k, mn, mx, hist, red, cand, [&](int pos, int i) { o[pos] = i; });
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        g_prof[blockIdx.x * 16 + 7] = t1 - t0;
        cnt_out[blockIdx.x] = kk;
    }
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 2048, k = argc > 2 ? atoi(argv[2]) : 128;
    const int ctas = argc > 3 ? atoi(argv[3]) : 148;
    std::mt19937 rng(1);
    std::normal_distribution<float> nd(40.f, 3.f);
    std::vector<float> h((size_t)ctas * n);
    for (auto &x : h) x = nd(rng);
    const int ties = argc > 4 ? atoi(argv[4]) : 0;  // quantise scores: many equal keys
    if (ties)
        for (auto &x : h) x = (float)(int)(x * ties / 10.f);
    float *d;
    int *out, *cnt;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&out, (size_t)ctas * k * 4);
    cudaMalloc(&cnt, ctas * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const size_t smb = ((n + 3) & ~3) * 4 + 2048 * 4 + 64 * 4 + 128 * 4;
    auto run = [&](auto kfn) {
        cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
        for (int it = 0; it < 5; ++it) kfn<<<ctas, NT, smb>>>(d, n, k, out, cnt);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
        std::vector<long long> p((size_t)ctas * 16);
        cudaMemcpyFromSymbol(p.data(), g_prof, p.size() * 8);
        const char *nm[12] = {"start", "hist", "binsearch", "cands", "threshold", "scan", "emit", "total", "bs.enter", "bs.scanned", "bs.bar1", "bs.found"};
        double acc[12] = {0};
        int cn[12] = {0};
        for (int c = 0; c < ctas; ++c)
            for (int i = 1; i < 12; ++i)
                if (i != 7 && p[c * 16 + i] > 0 && p[c * 16 + i] >= p[c * 16]) { acc[i] += p[c * 16 + i] - p[c * 16]; cn[i]++; }
        for (int c = 0; c < ctas; ++c) { acc[7] += p[c * 16 + 7]; cn[7]++; }
        std::vector<int> o((size_t)ctas * k), cn2(ctas);
        cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(cn2.data(), cnt, ctas * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int c = 0; c < ctas; ++c) {  // host reference: score desc, index asc; ids ascending
            std::vector<int> idx(n);
            for (int i = 0; i < n; ++i) idx[i] = i;
            const float *sc = h.data() + (size_t)c * n;
            std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return sc[a] > sc[b]; });
            const int kk = std::min(k, n);
            std::vector<int> ref(idx.begin(), idx.begin() + kk);
            std::sort(ref.begin(), ref.end());
            if (cn2[c] != kk) { bad++; continue; }
            for (int i = 0; i < kk; ++i) if (o[(size_t)c * k + i] != ref[i]) { bad++; break; }
        }
        printf("  verify: %d / %d CTAs wrong\n", bad, ctas);
        for (int i = 1; i < 12; ++i) printf("  %-10s n %4d mean %8.0f cycles\n", nm[i], cn[i], cn[i] ? acc[i] / cn[i] : 0.);
    };
    printf("n %d k %d ctas %d\n", n, k, ctas);
    if (n <= 512) run(kern<9>); else run(kern<11>);
    return 0;
}
