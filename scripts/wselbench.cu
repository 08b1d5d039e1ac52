// warp_select microbenchmark + exactness check (development tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_12211_b200/csrc -o /tmp/wsel scripts/wselbench.cu
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include "warp_select.cuh"
using namespace ts;
template <int KPL>
__global__ void bench(const float *scores, int n, int k, int *out, int *cnt, long long *cyc) {
    __shared__ __align__(16) int hist[kWsBins];
    const float *row = scores + (size_t)blockIdx.x * n;
    const int lane = threadIdx.x;
    uint32_t key[KPL];
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
        const int i = 32 * j + lane;
        key[j] = i < n ? score_key(row[i]) : 0u;
    }
    __syncwarp();
    long long t0 = clock64();
    int *o = out + (size_t)blockIdx.x * k;
    const int kk = warp_select<KPL>(key, k, hist, [&](int pos, int i) { o[pos] = i; });
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0) { cnt[blockIdx.x] = kk; if (blockIdx.x == 0) cyc[0] = t1 - t0; }
}
template <int KPL>
void run(int n, int k, int mode, const char *name) {
    const int rows = 64;
    std::vector<float> h(rows * n);
    std::mt19937 rng(7 + n + k + mode); std::normal_distribution<float> nd(10.f, 3.f); std::uniform_int_distribution<int> ui(-4, 4);
    for (auto &x : h) x = mode == 0 ? nd(rng) : (mode == 1 ? (float)ui(rng) : 5.0f);
    float *d; int *out, *cnt; long long *cyc;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&out, rows * k * 4); cudaMalloc(&cnt, rows * 4); cudaMalloc(&cyc, 8);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    for (int it = 0; it < 3; ++it) bench<KPL><<<rows, 32>>>(d, n, k, out, cnt, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    std::vector<int> o(rows * k), cn(rows);
    cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cn.data(), cnt, rows * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < rows; ++r) {
        std::vector<int> idx(n); for (int i = 0; i < n; ++i) idx[i] = i;
        const float *s = h.data() + (size_t)r * n;
        std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return s[a] > s[b]; });
        const int kk = std::min(k, n);
        std::vector<int> ref(idx.begin(), idx.begin() + kk); std::sort(ref.begin(), ref.end());
        std::vector<int> got(o.begin() + (size_t)r * k, o.begin() + (size_t)r * k + kk);
        if (cn[r] != kk || got != ref) ++bad;
    }
    printf("%-8s n %5d k %4d KPL %3d: %6lld cycles (row 0), %s (%d bad rows) %s\n", name, n, k, KPL, c,
           bad ? "MISMATCH" : "exact", bad, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d); cudaFree(out); cudaFree(cnt); cudaFree(cyc);
}
int main() {
    for (int mode = 0; mode < 3; ++mode) {
        const char *nm = mode == 0 ? "normal" : (mode == 1 ? "int-ties" : "all-eq");
        run<8>(256, 32, mode, nm);
        run<8>(200, 32, mode, nm);
        run<8>(256, 300, mode, nm);
        run<16>(512, 64, mode, nm);
        run<32>(1024, 64, mode, nm);
        run<64>(2048, 128, mode, nm);
        run<64>(2000, 1, mode, nm);
    }
    return 0;
}
