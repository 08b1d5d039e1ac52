// api.cu — the C ABI of libtinyserve.so (include/tinyserve.h): host-side validation,
// launch configuration and TMA descriptor encoding.  Every entry point only enqueues work
// on the caller's stream; nothing here allocates device memory or synchronises.
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "../../include/tinyserve.h"
#include "attn.cuh"
#include "common.cuh"
#include "fp8.cuh"
#include "step_cluster.cuh"
#include "meta.cuh"
#include "score.cuh"
#include "score_select.cuh"
#include "select.cuh"
#include "sparse_attn.cuh"

using namespace ts;

namespace {

thread_local int g_launches = 0;
unsigned long long *g_dbg_ts = nullptr;  // development: attention CTA timestamps
unsigned long long *g_dbg_ss = nullptr;  // development: score/select CTA timestamps
thread_local cudaEvent_t g_phase_ev[4] = {nullptr, nullptr, nullptr, nullptr};

// records phase event i on the stream (external record node when captured in a graph)
inline void phase_mark(int i, cudaStream_t st) {
    if (g_phase_ev[i]) cudaEventRecordWithFlags(g_phase_ev[i], st, cudaEventRecordExternal);
}

constexpr int kMaxSel = 4096;      // max selected pages per row (decode step)
constexpr int kMaxSelAttn = 8192;  // max pages per row handed to the attention kernels (8 B of smem each)

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }
inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

ts_status check_layout(const ts_layout *L) {
    if (!L) return TS_ERR_CONFIG;
    if (L->batch < 0 || L->num_q_heads < 1 || L->num_kv_heads < 1 || L->head_dim < 1 ||
        L->page_size < 1 || L->max_pages < 1 || L->num_blocks < 1)
        return TS_ERR_CONFIG;
    if (L->kv_dtype != TS_F32 && L->kv_dtype != TS_BF16 && L->kv_dtype != TS_FP8E4M3) return TS_ERR_CONFIG;
    if (L->num_q_heads % L->num_kv_heads) return TS_ERR_SHAPE;
    if (L->shard_stride < 1 || L->shard_offset < 0 || L->shard_offset >= L->shard_stride)
        return TS_ERR_SHAPE;
    if (L->head_dim != 64 && L->head_dim != 128) return TS_ERR_UNSUPPORTED;
    // 64M tokens per row: the kernels' 32-bit tile / page arithmetic (tiles x cluster width < 2^31)
    if ((long long)L->max_pages * L->page_size > (1LL << 26)) return TS_ERR_UNSUPPORTED;
    if (L->kv_dtype == TS_FP8E4M3 && (L->head_dim != 64 || L->page_size % 16 != 0)) return TS_ERR_UNSUPPORTED;
    return TS_OK;
}

// q and metadata of an FP8 cache are bf16: the scoring view of the layout
ts_layout score_view(const ts_layout *L) {
    ts_layout v = *L;
    if (v.kv_dtype == TS_FP8E4M3) v.kv_dtype = TS_BF16;
    return v;
}

int group_of(const ts_layout *L) { return L->num_q_heads / L->num_kv_heads; }

// Development A/B knobs: read from the environment (once per call site) only in the dev
// build (libtinyserve_dev.so, -DTS_DEV_KNOBS); the release library always takes the
// measured defaults (DESIGN.md §5 "Development knobs").
int env_int(const char *name, int dflt) {
#ifdef TS_DEV_KNOBS
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
#else
    (void)name;
    return dflt;
#endif
}

bool bf16_attn_supported(const ts_layout *L) {
    const int S = L->page_size;
    return L->kv_dtype == TS_BF16 && L->head_dim == 64 && group_of(L) <= 8 &&
           (S == 4 || S == 8 || S == 16 || S == 32 || S == 64);
}

ts_status launch_status() {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? TS_OK : TS_ERR_CUDA;
}

int device_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex mu;
    static std::unordered_map<int, int> cache;
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = sms;
    return sms;
}

// Co-resident clusters of `cluster` CTAs for a kernel configuration (cached; host only).
template <typename K>
int max_active_clusters(K kern, int threads, size_t smem, int cluster) {
    static std::mutex mu;
    static std::unordered_map<unsigned long long, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long key = (reinterpret_cast<uintptr_t>((const void *)kern) * 1315423911ull) ^
                                   ((unsigned long long)smem << 20) ^ ((unsigned long long)cluster << 8) ^
                                   (unsigned long long)threads ^ ((unsigned long long)dev << 56);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cluster * 64);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (const void *)kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[key] = n;
    return n;
}

// Opt-in shared memory / non-portable cluster size for a kernel, per DEVICE (a process may
// drive several GPUs: cudaFuncSetAttribute applies to the current device only).  Grows the
// opt-in size on demand; cached per (device, kernel).
bool ensure_func_attrs(const void *kern, size_t smem, bool nonportable) {
    static std::mutex mu;
    static std::unordered_map<unsigned long long, size_t> set_smem;
    static std::unordered_map<unsigned long long, bool> set_np;
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned long long key = (unsigned long long)reinterpret_cast<uintptr_t>(kern) ^ ((unsigned long long)dev << 56);
    std::lock_guard<std::mutex> g(mu);
    if (nonportable && !set_np[key]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            return false;
        set_np[key] = true;
    }
    if (smem > set_smem[key]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return false;
        set_smem[key] = smem;
    }
    return true;
}

// Launch with programmatic stream serialization (PDL): the kernel's griddepcontrol.wait
// orders it after the previous kernel in the stream, and its launch overlaps that kernel's
// tail (every standalone kernel starts with launch_dependents + wait).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// Pool [NB][Hkv][S][64] bf16 viewed as a 2-D tensor of NB*Hkv*S rows x 64 columns; box =
// TT rows x 64 columns (128 B rows), 128-byte swizzle.
bool make_pool_map(CUtensorMap *map, const void *pool, const ts_layout *L, int TT) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {64, (cuuint64_t)L->num_blocks * L->num_kv_heads * L->page_size};
    const cuuint64_t strides[1] = {64 * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)TT};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(pool), dims, strides,
              box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- workspace layout
// attention workspace: [tickets: rows u32][work counters: 2 u32][partials: rows x ipr x 8 x kPS]
// with ipr <= kMaxItemsPerRow split parts per row (split-K merge of the attention kernels).
constexpr int kMaxItemsPerRow = 64;
constexpr int kMaxClusterC = 16;  // widest cluster the step planner may choose (partials per row)
struct AttnWs {
    size_t tickets, work, part, total;
};
AttnWs attn_ws_layout(const ts_layout *L, int sel_stride, int min_parts = 1) {
    const size_t rows = (size_t)L->batch * L->num_kv_heads;
    const int tpr = sel_stride * std::max(1, L->page_size / 16);
    // split parts per row: the attention kernels split a row at most into its tiles; the
    // fused step's cluster may be wider than the selection (min_parts = its largest C)
    const int ipr = std::max(min_parts, std::min(kMaxItemsPerRow, std::max(1, tpr)));
    AttnWs w;
    w.tickets = 0;
    w.work = round_up(rows * 4, 256);
    w.part = w.work + 256;
    w.total = w.part + round_up(rows * (size_t)ipr * 8 * kPS * 4, 256);
    return w;
}

struct StepWs {
    AttnWs attn;
    size_t scores, sel_ids, sel_count, sel_blk, total;
};
StepWs step_ws_layout(const ts_layout *L, int kmax) {
    StepWs w;
    w.attn = attn_ws_layout(L, kmax, kMaxClusterC);
    const size_t rows = (size_t)L->batch * L->num_kv_heads;
    w.scores = w.attn.total;
    w.sel_ids = w.scores + round_up(rows * L->max_pages * 4, 256);
    w.sel_count = w.sel_ids + round_up(rows * kmax * 4, 256);
    w.sel_blk = w.sel_count + round_up(rows * 4, 256);
    w.total = w.sel_blk + round_up(rows * kmax * 4, 256);
    return w;
}

// K = floor(budget / S) clipped to [1, max_pages] (reading R4/R5; P_b <= max_pages)
int kmax_of(const ts_layout *L, int budget) {
    const int k = budget / L->page_size > 1 ? budget / L->page_size : 1;
    return k < L->max_pages ? k : L->max_pages;
}

// ---------------------------------------------------------------- launchers
ts_status launch_score(const ts_layout *L, const void *q, const void *meta, const int *pt,
                       const int *sl, float *scores, cudaStream_t st) {
    ScoreParams p{L->batch, L->num_q_heads, L->num_kv_heads, group_of(L), L->head_dim,
                  L->page_size, L->max_pages, L->shard_stride, L->shard_offset};
    const int rows = L->batch * L->num_kv_heads;
    if (rows == 0) return TS_OK;
    if (L->kv_dtype == TS_BF16 && p.G <= 8) {
        dim3 grid((L->max_pages + kScorePagesPerCta - 1) / kScorePagesPerCta, rows);
        if (L->head_dim == 64)
            launch_pdl(score_mma_kernel<64>, dim3(grid), dim3(kScoreWarps * 32), 0, st, 
                p, (const uint16_t *)q, (const uint16_t *)meta, pt, sl, scores);
        else
            launch_pdl(score_mma_kernel<128>, dim3(grid), dim3(kScoreWarps * 32), 0, st, 
                p, (const uint16_t *)q, (const uint16_t *)meta, pt, sl, scores);
    } else {
        dim3 grid((L->max_pages + kSimtPagesPerCta - 1) / kSimtPagesPerCta, rows);
        const size_t sm = (size_t)p.G * 2 * L->head_dim * 4;
        if (sm > 200 * 1024) return TS_ERR_UNSUPPORTED;
        if (L->kv_dtype == TS_BF16) {
            if (L->head_dim == 64) {
                if (!ensure_func_attrs((const void *)score_simt_kernel<uint16_t, 64>, sm, false)) return TS_ERR_CUDA;
                launch_pdl(score_simt_kernel<uint16_t, 64>, dim3(grid), dim3(kSimtWarps * 32), sm, st, p, (const uint16_t *)q, (const uint16_t *)meta, pt, sl, scores);
            } else {
                if (!ensure_func_attrs((const void *)score_simt_kernel<uint16_t, 128>, sm, false)) return TS_ERR_CUDA;
                launch_pdl(score_simt_kernel<uint16_t, 128>, dim3(grid), dim3(kSimtWarps * 32), sm, st, p, (const uint16_t *)q, (const uint16_t *)meta, pt, sl, scores);
            }
        } else {
            if (L->head_dim == 64) {
                if (!ensure_func_attrs((const void *)score_simt_kernel<float, 64>, sm, false)) return TS_ERR_CUDA;
                launch_pdl(score_simt_kernel<float, 64>, dim3(grid), dim3(kSimtWarps * 32), sm, st, p, (const float *)q, (const float *)meta, pt, sl, scores);
            } else {
                if (!ensure_func_attrs((const void *)score_simt_kernel<float, 128>, sm, false)) return TS_ERR_CUDA;
                launch_pdl(score_simt_kernel<float, 128>, dim3(grid), dim3(kSimtWarps * 32), sm, st, p, (const float *)q, (const float *)meta, pt, sl, scores);
            }
        }
    }
    ++g_launches;
    return launch_status();
}

ts_status launch_select(const float *scores, int rows, int stride, const int *row_len,
                        const int *ids_in, int id_stride, int id_offset, int k, int *sel_ids,
                        float *sel_scores, int *sel_count, cudaStream_t st, int parts = 1,
                        long long part_stride = 0) {
    if (rows == 0) return TS_OK;
    const size_t n = (size_t)stride * parts;
    const size_t sm = ids_in ? n * 4 * 3 : ((n + 3) & ~(size_t)3) * 4;  // affine keys padded to 4
    if (sm > 200 * 1024) return TS_ERR_UNSUPPORTED;
    if (ids_in && n > 16 * kSelThreads) return TS_ERR_UNSUPPORTED;
    if (!ensure_func_attrs((const void *)select_topk_kernel, 200 * 1024, false)) return TS_ERR_CUDA;
    SelectParams p{scores, rows, stride * parts, row_len, ids_in, id_stride, id_offset, k,
                   stride, part_stride, sel_ids, sel_scores, sel_count};
    launch_pdl(select_topk_kernel, dim3(rows), dim3(kSelThreads), sm, st, p);
    ++g_launches;
    return launch_status();
}

// bf16 sparse attention (sparse_attn.cuh): grid = rows x C CTAs, one cluster per row.
// W warps per CTA: 4 when the rows alone fill the GPU (4 CTAs / SM), 8 otherwise, 16 for
// very few rows; C = CTAs per row so that rows x C ~ one wave, each warp keeping >= 2
// octets.  pdl: launched as a programmatic dependent of the previous kernel.
template <int W, int DP>
ts_status prepare_sa(size_t sm) {
    auto kern = sparse_attn_kernel<W, DP>;
    return ensure_func_attrs((const void *)kern, sm, true) ? TS_OK : TS_ERR_CUDA;
}

// C = CTAs per row: the largest C <= cdesired whose clusters all fit on the GPU at once
template <int W, int DP>
ts_status launch_sa(const AttnParams &p, int rows, int cdesired, bool pdl, cudaStream_t st,
                    int nclusters = 0) {
    auto kern = sparse_attn_kernel<W, DP>;
    const size_t sm = SaSmem<W>::bytes(p.sel_stride);
    ts_status s = prepare_sa<W, DP>(sm);
    if (s != TS_OK) return s;
    int C = std::max(1, cdesired);
    while (C > 1 && max_active_clusters(kern, W * 32, sm, C) < rows) --C;
    if (nclusters <= 0) nclusters = rows;  // one row per cluster
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nclusters * C);
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = C;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (cudaLaunchKernelEx(&cfg, kern, p, C) != cudaSuccess) return TS_ERR_CUDA;
    ++g_launches;
    return launch_status();
}

// TMA-ring attention (sparse_attn_tma_kernel), S % 16 == 0: one (row, split) per CTA.
template <int W, int R, bool F8 = false>
ts_status launch_sat(const ts_layout *L, const AttnParams &p, bool pdl, cudaStream_t st) {
    auto kern = sparse_attn_tma_kernel<W, R, F8>;
    const int rows = L->batch * L->num_kv_heads;
    const size_t sm = SatSmemT<W, R, F8>::bytes(p.sel_stride);
    if (sm > 227 * 1024) return TS_ERR_UNSUPPORTED;
    if (!ensure_func_attrs((const void *)kern, sm, true)) return TS_ERR_CUDA;
    CUtensorMap tmK, tmV;
    if (!make_pool_map(&tmK, p.k_pool, L, 16) || !make_pool_map(&tmV, p.v_pool, L, 16))
        return TS_ERR_CUDA;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (W + 1) * 32, sm);
    static const int cmax_env = std::min(kMaxClusterC, std::max(1, env_int("TS_SA_CMAX", 16)));
    const int ntile = p.sel_stride * (L->page_size / 16);  // upper bound per row
    // splits per row: fill one wave (rows x C <= CTAs resident), each warp >= 2 tiles
    int C = std::max(1, std::min(cmax_env, device_sms() * std::max(1, per_sm) / std::max(1, rows)));
    C = std::max(1, std::min(C, ntile / (2 * W)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows * C);
    cfg.blockDim = dim3((W + 1) * 32);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    int na = 0;
    if (pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (cudaLaunchKernelEx(&cfg, kern, tmK, tmV, p, C) != cudaSuccess) return TS_ERR_CUDA;
    ++g_launches;
    return launch_status();
}

ts_status launch_sparse_attn(const ts_layout *L, const AttnParams &p, bool pdl, cudaStream_t st) {
    const int rows = L->batch * L->num_kv_heads;
    const int sms = device_sms();
    static const int tma = env_int("TS_SA_TMA", 1);
    if (tma && L->page_size % 16 == 0) {
        static const int rr = env_int("TS_SA_R", 8);
        if (rr == 12) return launch_sat<4, 12>(L, p, pdl, st);
        if (rr == 16) return launch_sat<4, 16>(L, p, pdl, st);
        return launch_sat<4, 8>(L, p, pdl, st);
    }
    const int n_oct = p.sel_stride * std::max(1, L->page_size / 8);  // upper bound per row
    static const int cmax_env = std::min(kMaxClusterC, std::max(1, env_int("TS_SA_CMAX", 16)));
    int W = rows >= 2 * sms ? 4 : (rows * 16 < sms ? 16 : 8);
    static const int w_env = env_int("TS_SA_W", 0);
    if (w_env == 4 || w_env == 8 || w_env == 16) W = w_env;
    const int per_sm = W == 4 ? 4 : (W == 8 ? 2 : 1);
    int C = std::max(1, std::min(cmax_env, sms * per_sm / std::max(1, rows)));
    C = std::max(1, std::min(C, n_oct / (2 * W)));
    if (W == 4) return launch_sa<4, 3>(p, rows, C, pdl, st);
    if (W == 8) return launch_sa<8, 3>(p, rows, C, pdl, st);
    return launch_sa<16, 3>(p, rows, C, pdl, st);
}

// Fused score + select (score_select.cuh): grid = rows x C CTAs (cluster per row), each
// CTA a contiguous chunk of the row's pages; C so that rows x C ~ 3 CTAs per SM.
template <int W, int R>
ts_status launch_ss_t(ScoreSelParams &p, int rows, int cdesired, cudaStream_t st) {
    auto kern = score_select_kernel<W, R>;
    const size_t sm = SsSmem<W, R>::bytes(p.max_pages);
    if (sm > 227 * 1024) return TS_ERR_UNSUPPORTED;
    if (!ensure_func_attrs((const void *)kern, sm, true)) return TS_ERR_CUDA;
    // chunk per CTA (a multiple of the stage), C = CTAs per row; the largest C <= cdesired
    // whose clusters all fit at once (one wave: no row waits for another row's CTAs)
    int C = std::max(1, cdesired), chunk = 0;
    for (;; --C) {
        chunk = (p.max_pages + C - 1) / C;
        chunk = (chunk + kSsStagePages - 1) / kSsStagePages * kSsStagePages;
        const int c = (p.max_pages + chunk - 1) / chunk;
        if (C == 1 || max_active_clusters(kern, (W + 1) * 32, sm, c) >= rows) {
            C = c;
            break;
        }
    }
    p.C = C;
    p.chunk = chunk;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows * p.C);
    cfg.blockDim = dim3((W + 1) * 32);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = p.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    // PDL: the prologue (barriers, histogram, cluster arrival) overlaps the previous kernel's
    // tail; griddepcontrol.wait precedes every read of q / metadata / page table
    static const bool pdl = env_int("TS_NO_PDL", 0) == 0;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, kern, p) != cudaSuccess) return TS_ERR_CUDA;
    ++g_launches;
    return launch_status();
}

// The whole bf16 step as one cluster-per-row kernel (step_cluster.cuh): plan (cluster width
// C, chunk, shared memory, flags) and launch.  DSM: the CTA partials merge in the cluster
// leader's shared memory (a separate instantiation, so the other configurations keep the
// leaner kernel).
struct StepPlan {
    bool ok = false;
    int C = 0, chunk = 0, flags = 0;
    size_t sm = 0;
};

template <int W, int R, bool DSM, bool APP, bool F8>
StepPlan plan_step(const ts_layout *L, int kmax) {
    auto kern = decode_cluster_kernel<W, R, DSM, APP, F8>;
    StepPlan pl;
    const int rows = L->batch * L->num_kv_heads;
    // flags: bit 0 page-table row prefetched to smem (rows up to 2048 pages); bit 1
    // two-level select when rows are much longer than the candidates; bit 2 DSMEM merge
    // area (DSM); bits 3 / 4 early / late PDL trigger (set at launch)
    int fl = (((L->max_pages & 3) == 0 && L->max_pages <= 2048) ? 1 : 0) | (DSM ? 4 : 0);
    static const int two_env = env_int("TS_SC_TWO", -1);
    const bool two_ok = two_env == 1 || (two_env != 0 && L->max_pages > 2048);  // long rows only
    auto allow = [&](size_t smb) -> bool {  // grow the opt-in shared memory on demand
        return ensure_func_attrs((const void *)kern, smb, true);
    };
    static const int cmax = std::min(kMaxClusterC, std::max(1, env_int("TS_SC_CMAX", 16)));
    const int max_c = std::max(1, std::min(cmax, (L->max_pages + 63) / 64));  // >= 64 pages per CTA
    auto chunk_of = [&](int c) {
        int ch = (L->max_pages + c - 1) / c;
        return (ch + kSsStagePages - 1) / kSsStagePages * kSsStagePages;
    };
    if (two_ok) {  // two-level select: every CTA keeps only its chunk's scores
        for (int c = max_c; c >= 2; --c) {
            const int ch = chunk_of(c), cc = (L->max_pages + ch - 1) / ch;
            if (kmax % 4 != 0 || (two_env != 1 && L->max_pages < 4 * cc * kmax)) continue;
            const size_t smc = 1024 + ScSmem<W, R>::bytes(kmax, L->max_pages, fl | 2, cc, ch);
            if (smc > 227 * 1024 || !allow(smc)) continue;
            if (max_active_clusters(kern, (W + 1) * 32, smc, cc) >= rows) {
                pl.ok = true;
                pl.C = cc;
                pl.chunk = ch;
                pl.sm = smc;
                pl.flags = fl | 2;
                return pl;
            }
        }
    }
    // one-level select: every CTA selects over the whole row's keys; the largest C whose
    // clusters are all co-resident (one wave)
    size_t sm = 1024 + ScSmem<W, R>::bytes(kmax, L->max_pages, fl, 1, 0);
    if (sm > 227 * 1024 || !allow(sm)) return pl;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (W + 1) * 32, sm);
    const int target = device_sms() * std::max(1, per_sm);
    for (int C = std::max(1, std::min(max_c, target / std::max(1, rows)));; --C) {
        const int chunk = chunk_of(C);
        const int c = (L->max_pages + chunk - 1) / chunk;
        const size_t smc = c == 1 ? sm : 1024 + ScSmem<W, R>::bytes(kmax, L->max_pages, fl, c, chunk);
        if (c == 1 || (smc <= 227 * 1024 && allow(smc) &&
                       max_active_clusters(kern, (W + 1) * 32, smc, c) >= rows)) {
            pl.ok = true;
            pl.C = c;
            pl.chunk = chunk;
            pl.sm = smc;
            pl.flags = fl;
            return pl;
        }
    }
}

template <int W, int R, bool DSM, bool APP, bool F8>
ts_status launch_step(const ts_layout *L, ScoreSelParams &sp, const AttnParams &ap,
                      const StepPlan &pl, cudaStream_t st) {
    auto kern = decode_cluster_kernel<W, R, DSM, APP, F8>;
    const int rows = L->batch * L->num_kv_heads;
    CUtensorMap tmK, tmV;
    // (FP8 tiles are 1-D bulk copies; the maps are then unused placeholders)
    if (!make_pool_map(&tmK, ap.k_pool, L, 16) || !make_pool_map(&tmV, ap.v_pool, L, 16))
        return TS_ERR_CUDA;
    sp.C = pl.C;
    sp.chunk = pl.chunk;
    sp.flags = pl.flags;
    // PDL trigger for the next kernel in the stream (its prologue overlaps our tail): after
    // the attention loop (bit 4) with clusters of <= 8 CTAs — measured 0.9 % faster than at
    // kernel start (bit 3, TS_SC_TRIGGER=1) on C2 / C4, equal on C3; none with C5's 13-CTA
    // clusters (either trigger: 23 -> 28-32 us)
    static const int trig_env = env_int("TS_SC_TRIGGER", -1);
    if (trig_env == 1) sp.flags |= 8;
    if (trig_env == 2 || (trig_env < 0 && pl.C <= 8)) sp.flags |= 16;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(rows * pl.C);
    cfg.blockDim = dim3((W + 1) * 32);
    cfg.dynamicSmemBytes = pl.sm;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = pl.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    static const bool pdl = env_int("TS_NO_PDL", 0) == 0;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, kern, tmK, tmV, sp, ap) != cudaSuccess) return TS_ERR_CUDA;
    ++g_launches;
    return launch_status();
}

template <int W, int R, bool APP, bool F8>
ts_status launch_step_cluster_app(const ts_layout *L, ScoreSelParams &sp, const AttnParams &ap,
                                 cudaStream_t st) {
    // DSMEM merge when its merge area costs no cluster width and C <= 8 (measured: faster at
    // C = 4 (C3); at C = 13 (C5) one SM receiving 13 partials loses to the L2 ticket merge)
    static const int dsm_env = env_int("TS_SC_DSM", -1);  // dev knob
    const StepPlan b = plan_step<W, R, false, APP, F8>(L, sp.kmax);
    if constexpr (R == 8) {
        const StepPlan a = plan_step<W, R, true, APP, F8>(L, sp.kmax);
        if (dsm_env != 0 && a.ok && a.C > 1 && (dsm_env == 1 || !b.ok || (a.C >= b.C && a.C <= 8)))
            return launch_step<W, R, true, APP, F8>(L, sp, ap, a, st);
    }
    if (!b.ok) return TS_ERR_UNSUPPORTED;
    return launch_step<W, R, false, APP, F8>(L, sp, ap, b, st);
}

// the fused-append instantiation (APP) only when the call appends: the plain step keeps the
// leaner kernel (measured ~3 % on every config)
template <int W, int R>
ts_status launch_step_cluster_t(const ts_layout *L, ScoreSelParams &sp, const AttnParams &ap,
                                cudaStream_t st) {
    if (L->kv_dtype == TS_FP8E4M3)
        return sp.k_new ? launch_step_cluster_app<W, R, true, true>(L, sp, ap, st)
                        : launch_step_cluster_app<W, R, false, true>(L, sp, ap, st);
    return sp.k_new ? launch_step_cluster_app<W, R, true, false>(L, sp, ap, st)
                    : launch_step_cluster_app<W, R, false, false>(L, sp, ap, st);
}


ts_status launch_score_select(const ts_layout *L, const void *q, const void *meta, const int *pt,
                              const int *sl, int *ids, int *blk, int *cnt, int kmax,
                              cudaStream_t st, float *sel_scores = nullptr) {
    const int rows = L->batch * L->num_kv_heads;
    if (rows == 0) return TS_OK;
    ScoreSelParams p{};
    p.q = static_cast<const uint16_t *>(q);
    p.meta = static_cast<const uint16_t *>(meta);
    p.page_table = pt;
    p.seq_lens = sl;
    p.sel_ids = ids;
    p.sel_blk = blk;
    p.sel_count = cnt;
    p.B = L->batch;
    p.Hq = L->num_q_heads;
    p.Hkv = L->num_kv_heads;
    p.G = group_of(L);
    p.S = L->page_size;
    p.max_pages = L->max_pages;
    p.kmax = kmax;
    p.dbg = g_dbg_ss;
    p.stride = L->shard_stride;
    p.offset = L->shard_offset;
    p.sel_scores = sel_scores;
    static const int per_sm = env_int("TS_SS_PER_SM", 3);
    static const int cmax = std::min(kMaxClusterC, std::max(1, env_int("TS_SS_CMAX", 16)));
    const int target = device_sms() * per_sm;
    const int max_c = std::max(1, std::min(cmax, (L->max_pages + 63) / 64));  // >= 64 pages per CTA
    const int C = std::max(1, std::min(max_c, (target + rows - 1) / rows));
    return launch_ss_t<4, 4>(p, rows, C, st);
}

AttnParams attn_params(const ts_layout *L, const void *q, const void *k_pool, const void *v_pool,
                       const int *pt, const int *sl, const int *sel_ids, const int *sel_count,
                       int sel_stride, float scale, float *o, float *lse, void *ws) {
    const AttnWs w = attn_ws_layout(L, sel_stride);
    AttnParams p{};
    p.q = q;
    p.k_pool = k_pool;
    p.v_pool = v_pool;
    p.page_table = pt;
    p.seq_lens = sl;
    p.sel_ids = sel_ids;
    p.sel_count = sel_count;
    p.sel_blk = nullptr;
    p.sel_stride = sel_stride;
    p.B = L->batch;
    p.Hq = L->num_q_heads;
    p.Hkv = L->num_kv_heads;
    p.G = group_of(L);
    p.D = L->head_dim;
    p.S = L->page_size;
    p.max_pages = L->max_pages;
    p.stride = L->shard_stride;
    p.offset = L->shard_offset;
    p.num_blocks = L->num_blocks;
    p.scale = scale;
    p.o = o;
    p.lse = lse;
    p.tickets = reinterpret_cast<unsigned *>(static_cast<char *>(ws) + w.tickets);
    p.part = reinterpret_cast<float *>(static_cast<char *>(ws) + w.part);
    p.splits = 1;
    p.items = L->batch * L->num_kv_heads;
    p.dbg = g_dbg_ts;
    return p;
}

ts_status launch_attn(const ts_layout *L, const void *q, const void *k_pool, const void *v_pool,
                      const int *pt, const int *sl, const int *sel_ids, const int *sel_count,
                      int sel_stride, float scale, float *o, float *lse, void *ws, cudaStream_t st) {
    const int rows = L->batch * L->num_kv_heads;
    if (rows == 0) return TS_OK;
    AttnParams p = attn_params(L, q, k_pool, v_pool, pt, sl, sel_ids, sel_count, sel_stride, scale,
                               o, lse, ws);
    if (L->kv_dtype == TS_BF16) {
        if (!bf16_attn_supported(L) || sel_stride > kMaxSelAttn) return TS_ERR_UNSUPPORTED;
        return launch_sparse_attn(L, p, true, st);
    }
    if (L->kv_dtype == TS_FP8E4M3) {  // the TMA-ring kernel's F8 instantiation
        if (L->page_size % 16 != 0 || group_of(L) > 8 || sel_stride > kMaxSelAttn) return TS_ERR_UNSUPPORTED;
        // 2 KB stages (16 in the bf16 ring's bytes), 8 consumer warps: the FP8 tile chain is
        // consumer-bound (measured FullCache C3 86.7 -> 80.5 us with 8 warps instead of 4)
        return launch_sat<8, 16, true>(L, p, true, st);
    }
    const int threads = 32 * std::min(p.G, 8);
    if (L->head_dim == 64)
        launch_pdl(attn_simt_kernel<64>, dim3(rows), dim3(threads), 0, st, p, (const float *)k_pool, (const float *)v_pool);
    else
        launch_pdl(attn_simt_kernel<128>, dim3(rows), dim3(threads), 0, st, p, (const float *)k_pool, (const float *)v_pool);
    ++g_launches;
    return launch_status();
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char *ts_status_str(ts_status s) {
    switch (s) {
        case TS_OK: return "TS_OK";
        case TS_ERR_CONFIG: return "TS_ERR_CONFIG: invalid size, budget or dtype";
        case TS_ERR_SHAPE: return "TS_ERR_SHAPE: inconsistent shapes (heads, k, sharding)";
        case TS_ERR_ALIGN: return "TS_ERR_ALIGN: tensor pointer not 16-byte aligned";
        case TS_ERR_UNSUPPORTED: return "TS_ERR_UNSUPPORTED: shape outside the compiled set";
        case TS_ERR_CUDA: return "TS_ERR_CUDA: CUDA launch failure";
        case TS_ERR_WORKSPACE: return "TS_ERR_WORKSPACE: workspace missing or too small";
    }
    return "unknown ts_status";
}

const char *ts_version(void) { return "tinyserve-b200 0.1 (sm_100a)"; }

int32_t ts_last_launch_count(void) { return g_launches; }

#ifdef TS_DEV_KNOBS
// TS_DEBUG error word (common.cuh, dev build only): synchronises the device, returns the
// OR of the fault bits raised since the last reset (bit 0 seq_len out of range, bit 1
// page-table entry out of range), and clears it if `reset` != 0.
int32_t ts_debug_error_word(int32_t reset) {
    cudaDeviceSynchronize();
    unsigned v = 0;
    if (cudaMemcpyFromSymbol(&v, g_ts_debug_err, sizeof(v)) != cudaSuccess) return -1;
    if (reset) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(g_ts_debug_err, &z, sizeof(z));
    }
    return (int32_t)v;
}
// development hooks of the dev build only (not in the public header): device buffers for
// per-CTA globaltimer phase stamps (scripts/step_stamps.py)
void ts_debug_timestamps(void *buf) { g_dbg_ts = static_cast<unsigned long long *>(buf); }
void ts_debug_ss_timestamps(void *buf) { g_dbg_ss = static_cast<unsigned long long *>(buf); }
#endif

void ts_profile_events(void *const *events, int32_t n) {
    for (int i = 0; i < 4; ++i)
        g_phase_ev[i] = (events && i < n) ? static_cast<cudaEvent_t>(events[i]) : nullptr;
}

size_t ts_attn_workspace_bytes(const ts_layout *L, int32_t sel_stride) {
    if (check_layout(L) != TS_OK || sel_stride < 1) return 0;
    return attn_ws_layout(L, sel_stride).total;
}

size_t ts_workspace_bytes(const ts_layout *L, int32_t budget_tokens) {
    if (check_layout(L) != TS_OK || budget_tokens < 1) return 0;
    return step_ws_layout(L, kmax_of(L, budget_tokens)).total;
}

static ts_status meta_append_impl(const ts_layout *L, const void *k_new, const void *v_new,
                                  int32_t *seq_lens, int32_t advance, const int32_t *page_table,
                                  void *k_pool, void *v_pool, void *meta, void *stream);

ts_status ts_meta_append(const ts_layout *L, const void *k_new, const void *v_new,
                         int32_t *seq_lens, int32_t advance, const int32_t *page_table,
                         void *k_pool, void *v_pool, void *meta, void *stream) {
    g_launches = 0;
    return meta_append_impl(L, k_new, v_new, seq_lens, advance != 0 ? 1 : 0, page_table, k_pool,
                            v_pool, meta, stream);
}

static ts_status meta_append_impl(const ts_layout *L, const void *k_new, const void *v_new,
                                  int32_t *seq_lens, int32_t advance, const int32_t *page_table,
                                  void *k_pool, void *v_pool, void *meta, void *stream) {
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (!aligned16(k_new) || !aligned16(v_new) || !aligned16(k_pool) || !aligned16(v_pool) ||
        !aligned16(meta))
        return TS_ERR_ALIGN;
    if (L->batch == 0) return TS_OK;
    MetaParams p{L->batch, L->num_kv_heads, L->head_dim, L->page_size, L->max_pages,
                 L->shard_stride, L->shard_offset, L->num_blocks};
    if (L->kv_dtype == TS_FP8E4M3) {  // bf16 token -> E4M3 codes + row exponent (reading R21)
        if (L->num_kv_heads * 8 > 1024) return TS_ERR_UNSUPPORTED;
        launch_pdl(meta_append_f8_kernel, dim3(L->batch), dim3(L->num_kv_heads * 8), 0, as_stream(stream),
                   p, (const uint16_t *)k_new, (const uint16_t *)v_new, seq_lens, advance, page_table,
                   (uint8_t *)k_pool, (uint8_t *)v_pool, (uint16_t *)meta);
        ++g_launches;
        return launch_status();
    }
    const int threads = L->num_kv_heads * L->head_dim / (L->kv_dtype == TS_BF16 ? 8 : 4);
    if (threads > 1024) return TS_ERR_UNSUPPORTED;
    if (L->kv_dtype == TS_BF16)
        launch_pdl(meta_append_kernel<uint16_t>, dim3(L->batch), dim3(threads), 0, as_stream(stream), 
            p, (const uint16_t *)k_new, (const uint16_t *)v_new, seq_lens, advance, page_table,
            (uint16_t *)k_pool, (uint16_t *)v_pool, (uint16_t *)meta);
    else
        launch_pdl(meta_append_kernel<float>, dim3(L->batch), dim3(threads), 0, as_stream(stream), 
            p, (const float *)k_new, (const float *)v_new, seq_lens, advance, page_table,
            (float *)k_pool, (float *)v_pool, (float *)meta);
    ++g_launches;
    return launch_status();
}

ts_status ts_meta_build(const ts_layout *L, const void *k_pool, const int32_t *page_table,
                        const int32_t *seq_lens, void *meta, void *stream) {
    g_launches = 0;
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (!aligned16(k_pool) || !aligned16(meta)) return TS_ERR_ALIGN;
    if (L->batch == 0) return TS_OK;
    MetaParams p{L->batch, L->num_kv_heads, L->head_dim, L->page_size, L->max_pages,
                 L->shard_stride, L->shard_offset, L->num_blocks};
    const long long work = (long long)L->batch * L->max_pages * L->num_kv_heads *
                           (L->head_dim / (L->kv_dtype == TS_F32 ? 4 : 8));
    const int grid = (int)std::min<long long>((work + 255) / 256, (long long)device_sms() * 16);
    if (L->kv_dtype == TS_FP8E4M3)
        launch_pdl(meta_build_f8_kernel, dim3(grid), dim3(256), 0, as_stream(stream), p,
                   (const uint8_t *)k_pool, page_table, seq_lens, (uint16_t *)meta);
    else if (L->kv_dtype == TS_BF16)
        launch_pdl(meta_build_kernel<uint16_t>, dim3(grid), dim3(256), 0, as_stream(stream), 
            p, (const uint16_t *)k_pool, page_table, seq_lens, (uint16_t *)meta);
    else
        launch_pdl(meta_build_kernel<float>, dim3(grid), dim3(256), 0, as_stream(stream), 
            p, (const float *)k_pool, page_table, seq_lens, (float *)meta);
    ++g_launches;
    return launch_status();
}

ts_status ts_score_pages(const ts_layout *L, const void *q, const void *meta,
                         const int32_t *page_table, const int32_t *seq_lens, float *scores,
                         void *stream) {
    g_launches = 0;
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (!aligned16(q) || !aligned16(meta)) return TS_ERR_ALIGN;
    const ts_layout v = score_view(L);  // FP8 cache: q and metadata are bf16
    return launch_score(&v, q, meta, page_table, seq_lens, scores, as_stream(stream));
}

ts_status ts_select_topk(const float *scores, int32_t rows, int32_t stride, const int32_t *row_len,
                         const int32_t *ids_in, int32_t id_stride, int32_t id_offset, int32_t k,
                         int32_t *sel_ids, float *sel_scores, int32_t *sel_count, void *stream) {
    g_launches = 0;
    if (rows < 0 || stride < 1) return TS_ERR_CONFIG;
    if (k < 1 || id_stride < 1) return TS_ERR_SHAPE;
    return launch_select(scores, rows, stride, row_len, ids_in, id_stride, id_offset, k, sel_ids,
                         sel_scores, sel_count, as_stream(stream));
}

ts_status ts_sparse_decode_attn(const ts_layout *L, const void *q, const void *k_pool,
                                const void *v_pool, const int32_t *page_table,
                                const int32_t *seq_lens, const int32_t *sel_ids,
                                const int32_t *sel_count, int32_t sel_stride, float scale,
                                float *o, float *lse, void *ws, size_t ws_bytes, void *stream) {
    g_launches = 0;
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (sel_stride < 1) return TS_ERR_SHAPE;
    if (!aligned16(q) || !aligned16(k_pool) || !aligned16(v_pool) || !aligned16(o))
        return TS_ERR_ALIGN;
    if (!ws || ws_bytes < attn_ws_layout(L, sel_stride).total) return TS_ERR_WORKSPACE;
    return launch_attn(L, q, k_pool, v_pool, page_table, seq_lens, sel_ids, sel_count, sel_stride,
                       scale, o, lse, ws, as_stream(stream));
}

static ts_status decode_step_impl(const ts_layout *L, const void *q, const void *k_new,
                                  const void *v_new, const void *k_pool, const void *v_pool,
                                  const void *meta, const int32_t *page_table,
                                  const int32_t *seq_lens, int32_t budget_tokens, float scale,
                                  float *o, float *lse, int32_t *sel_ids_out,
                                  int32_t *sel_count_out, void *ws, size_t ws_bytes, void *stream,
                                  bool prefetch_prev = false);

ts_status ts_decode_step(const ts_layout *L, const void *q, const void *k_pool, const void *v_pool,
                         const void *meta, const int32_t *page_table, const int32_t *seq_lens,
                         int32_t budget_tokens, float scale, float *o, float *lse,
                         int32_t *sel_ids_out, int32_t *sel_count_out, void *ws, size_t ws_bytes,
                         void *stream) {
    g_launches = 0;
    return decode_step_impl(L, q, nullptr, nullptr, k_pool, v_pool, meta, page_table, seq_lens,
                            budget_tokens, scale, o, lse, sel_ids_out, sel_count_out, ws, ws_bytes,
                            stream);
}

ts_status ts_decode_step_append(const ts_layout *L, const void *q, const void *k_new,
                                const void *v_new, void *k_pool, void *v_pool, void *meta,
                                const int32_t *page_table, const int32_t *seq_lens,
                                int32_t budget_tokens, float scale, float *o, float *lse,
                                int32_t *sel_ids_out, int32_t *sel_count_out, void *ws,
                                size_t ws_bytes, void *stream) {
    g_launches = 0;
    if (!k_new || !v_new) return TS_ERR_CONFIG;
    if (!aligned16(k_new) || !aligned16(v_new)) return TS_ERR_ALIGN;
    return decode_step_impl(L, q, k_new, v_new, k_pool, v_pool, meta, page_table, seq_lens,
                            budget_tokens, scale, o, lse, sel_ids_out, sel_count_out, ws, ws_bytes,
                            stream);
}

ts_status ts_decode_step_prefetch(const ts_layout *L, const void *q, const void *k_pool,
                                  const void *v_pool, const void *meta, const int32_t *page_table,
                                  const int32_t *seq_lens, int32_t budget_tokens, float scale,
                                  float *o, float *lse, int32_t *sel_ids, int32_t *sel_count,
                                  void *ws, size_t ws_bytes, void *stream) {
    g_launches = 0;
    if (!sel_ids || !sel_count) return TS_ERR_CONFIG;  // they carry the previous selection in
    return decode_step_impl(L, q, nullptr, nullptr, k_pool, v_pool, meta, page_table, seq_lens,
                            budget_tokens, scale, o, lse, sel_ids, sel_count, ws, ws_bytes, stream,
                            true);
}

static ts_status decode_step_impl(const ts_layout *L, const void *q, const void *k_new,
                                  const void *v_new, const void *k_pool, const void *v_pool,
                                  const void *meta, const int32_t *page_table,
                                  const int32_t *seq_lens, int32_t budget_tokens, float scale,
                                  float *o, float *lse, int32_t *sel_ids_out,
                                  int32_t *sel_count_out, void *ws, size_t ws_bytes, void *stream,
                                  bool prefetch_prev) {
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (budget_tokens < 1) return TS_ERR_CONFIG;
    if (L->shard_stride != 1) return TS_ERR_UNSUPPORTED;
    if (!aligned16(q) || !aligned16(k_pool) || !aligned16(v_pool) || !aligned16(meta) ||
        !aligned16(o))
        return TS_ERR_ALIGN;
    const int kmax = kmax_of(L, budget_tokens);
    const StepWs w = step_ws_layout(L, kmax);
    if (!ws || ws_bytes < w.total) return TS_ERR_WORKSPACE;
    if (L->kv_dtype == TS_BF16 && (!bf16_attn_supported(L) || kmax > kMaxSel))
        return TS_ERR_UNSUPPORTED;
    // FP8 KV (reading R21): the one-launch cluster kernel only (d 64, S % 16 == 0, G <= 8)
    const bool f8 = L->kv_dtype == TS_FP8E4M3;
    if (f8 && (L->page_size % 16 != 0 || group_of(L) > 8 || kmax > kMaxSel)) return TS_ERR_UNSUPPORTED;
    char *wb = static_cast<char *>(ws);
    float *scores = reinterpret_cast<float *>(wb + w.scores);
    int *ids = sel_ids_out ? sel_ids_out : reinterpret_cast<int *>(wb + w.sel_ids);
    int *cnt = sel_count_out ? sel_count_out : reinterpret_cast<int *>(wb + w.sel_count);
    const cudaStream_t st = as_stream(stream);
    const int rows = L->batch * L->num_kv_heads;
    static const int two_kernels = env_int("TS_TWO_KERNELS", 0);
    if ((f8 || (L->kv_dtype == TS_BF16 && !two_kernels)) && group_of(L) <= 8 && L->head_dim == 64 &&
        L->page_size % 16 == 0 && rows > 0) {
        // the whole step in one cluster-per-row kernel (step_cluster.cuh)
        ScoreSelParams sp{};
        sp.q = static_cast<const uint16_t *>(q);
        sp.meta = static_cast<const uint16_t *>(meta);
        sp.page_table = page_table;
        sp.seq_lens = seq_lens;
        sp.sel_ids = ids;
        sp.sel_blk = nullptr;
        sp.sel_count = cnt;
        sp.B = L->batch;
        sp.Hq = L->num_q_heads;
        sp.Hkv = L->num_kv_heads;
        sp.G = group_of(L);
        sp.S = L->page_size;
        sp.max_pages = L->max_pages;
        sp.kmax = kmax;
        sp.dbg = g_dbg_ss;
        sp.k_new = static_cast<const uint16_t *>(k_new);  // fused append (nullable)
        sp.v_new = static_cast<const uint16_t *>(v_new);
        sp.prev_ids = prefetch_prev ? ids : nullptr;  // NEXT-2: the previous selection -> L2
        sp.prev_count = prefetch_prev ? cnt : nullptr;

        sp.k_pool = static_cast<const uint16_t *>(k_pool);
        sp.v_pool = static_cast<const uint16_t *>(v_pool);

        AttnParams ap = attn_params(L, q, k_pool, v_pool, page_table, seq_lens, ids, cnt, kmax, scale,
                                    o, lse, ws);
        phase_mark(0, st);
        // ring depth: 8 stages (64 KB in flight per CTA) when the rows leave SMs for wide
        // clusters (measured: C3 / C5 faster); 4 stages when many rows need >= 3 CTAs per SM
        static const int ring_env = env_int("TS_SC_R", 0);  // dev knob
        const int ring = ring_env ? ring_env : (L->batch * L->num_kv_heads <= device_sms() ? 8 : 4);
        s = ring == 8 ? launch_step_cluster_t<4, 8>(L, sp, ap, st) : launch_step_cluster_t<4, 4>(L, sp, ap, st);
        phase_mark(3, st);
        if (s != TS_ERR_UNSUPPORTED || f8) {
            g_launches = 1;
            return s;
        }
    }
    if (k_new) {  // not fused here: append first (slot seq_len - 1), then the plain step
        if ((s = meta_append_impl(L, k_new, v_new, const_cast<int32_t *>(seq_lens), -1, page_table,
                                  const_cast<void *>(k_pool), const_cast<void *>(v_pool),
                                  const_cast<void *>(meta), stream)) != TS_OK)
            return s;
    }
    const int pre = k_new ? 1 : 0;  // launches so far
    if (L->kv_dtype == TS_BF16 && group_of(L) <= 8 && L->head_dim == 64) {
        // score + select (cluster per row) -> sparse attention (PDL, blocks pre-resolved)
        int *blk = reinterpret_cast<int *>(wb + w.sel_blk);
        phase_mark(0, st);
        if ((s = launch_score_select(L, q, meta, page_table, seq_lens, ids, blk, cnt, kmax, st)) !=
            TS_OK)
            return s;
        phase_mark(1, st);
        phase_mark(2, st);
        if (rows > 0) {
            AttnParams p = attn_params(L, q, k_pool, v_pool, page_table, seq_lens, ids, cnt, kmax,
                                       scale, o, lse, ws);
            p.sel_blk = blk;
            static const bool pdl = env_int("TS_NO_PDL", 0) == 0;
            if ((s = launch_sparse_attn(L, p, pdl, st)) != TS_OK) return s;
        }
        phase_mark(3, st);
        g_launches = pre + (rows > 0 ? 2 : 1);
        return TS_OK;
    }
    int launches = pre;
    g_launches = 0;
    phase_mark(0, st);
    if ((s = launch_score(L, q, meta, page_table, seq_lens, scores, st)) != TS_OK) return s;
    phase_mark(1, st);
    launches += g_launches;
    g_launches = 0;
    if ((s = launch_select(scores, rows, L->max_pages, nullptr, nullptr, 1, 0, kmax, ids, nullptr,
                           cnt, st)) != TS_OK)
        return s;
    phase_mark(2, st);
    launches += g_launches;
    g_launches = 0;
    if ((s = launch_attn(L, q, k_pool, v_pool, page_table, seq_lens, ids, cnt, kmax, scale, o, lse,
                         ws, st)) != TS_OK)
        return s;
    phase_mark(3, st);
    g_launches += launches;
    return TS_OK;
}

// FullCache baseline: dense paged decode attention over every page
// j < P_b, same pool / layout / kernels as the sparse path.
size_t ts_dense_workspace_bytes(const ts_layout *L) {
    if (check_layout(L) != TS_OK) return 0;
    return attn_ws_layout(L, L->max_pages).total;
}

ts_status ts_dense_decode_attn(const ts_layout *L, const void *q, const void *k_pool,
                               const void *v_pool, const int32_t *page_table,
                               const int32_t *seq_lens, float scale, float *o, float *lse,
                               void *ws, size_t ws_bytes, void *stream) {
    g_launches = 0;
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (L->shard_stride != 1) return TS_ERR_UNSUPPORTED;
    if (!aligned16(q) || !aligned16(k_pool) || !aligned16(v_pool) || !aligned16(o))
        return TS_ERR_ALIGN;
    const bool f8 = L->kv_dtype == TS_FP8E4M3;
    if ((!f8 && !bf16_attn_supported(L)) || L->page_size % 16 != 0 || group_of(L) > 8)
        return TS_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < attn_ws_layout(L, L->max_pages).total) return TS_ERR_WORKSPACE;
    if (L->batch == 0) return TS_OK;
    AttnParams p = attn_params(L, q, k_pool, v_pool, page_table, seq_lens, nullptr, nullptr,
                               L->max_pages, scale, o, lse, ws);
    p.dense = 1;
    if (f8) return launch_sat<8, 16, true>(L, p, true, as_stream(stream));
    static const int rr = env_int("TS_SA_R", 8);
    if (rr == 16) return launch_sat<4, 16>(L, p, true, as_stream(stream));
    return launch_sat<4, 8>(L, p, true, as_stream(stream));
}

// FP8 KV storage (reading R21): quantise `rows` bf16 rows of head_dim 64.
ts_status ts_kv_quantize(int64_t rows, int32_t head_dim, const void *src, void *pool, void *stream) {
    g_launches = 0;
    if (rows < 0 || head_dim < 1) return TS_ERR_CONFIG;
    if (head_dim != 64) return TS_ERR_UNSUPPORTED;
    if (rows % 16) return TS_ERR_SHAPE;  // whole sub-page records
    if (!aligned16(src) || !aligned16(pool)) return TS_ERR_ALIGN;
    if (rows == 0) return TS_OK;
    const long long thr = rows * 8;
    const int grid = (int)std::min<long long>((thr + 255) / 256, (long long)device_sms() * 16);
    launch_pdl(kv_quantize_kernel, dim3(grid), dim3(256), 0, as_stream(stream), (long long)rows,
               (const uint16_t *)src, (uint8_t *)pool);
    ++g_launches;
    return launch_status();
}

size_t ts_pool_bytes(const ts_layout *L) {
    if (check_layout(L) != TS_OK) return 0;
    const size_t n = (size_t)L->num_blocks * L->num_kv_heads * L->page_size;
    if (L->kv_dtype == TS_FP8E4M3) return n * (L->head_dim + 1);
    return n * L->head_dim * (L->kv_dtype == TS_BF16 ? 2 : 4);
}

// The two halves of one rank's sequence-sharded step, one launch each.
ts_status ts_select_candidates(const ts_layout *L, const void *q, const void *meta,
                               const int32_t *page_table, const int32_t *seq_lens, int32_t k,
                               float *cand_scores, int32_t *cand_ids, int32_t *cand_count,
                               void *stream) {
    g_launches = 0;
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (k < 1) return TS_ERR_SHAPE;
    if (!aligned16(q) || !aligned16(meta)) return TS_ERR_ALIGN;
    if (L->kv_dtype == TS_F32 || group_of(L) > 8 || L->head_dim != 64 || k > kMaxSel)
        return TS_ERR_UNSUPPORTED;  // (the composed ts_score_pages + ts_select_topk cover these)
    const ts_layout v = score_view(L);
    return launch_score_select(&v, q, meta, page_table, seq_lens, cand_ids, nullptr, cand_count, k,
                               as_stream(stream), cand_scores);
}

ts_status ts_shard_attend(const ts_layout *L, const void *q, const void *k_pool, const void *v_pool,
                          const int32_t *page_table, const int32_t *seq_lens,
                          const float *cand_scores, const int32_t *cand_ids, int32_t parts,
                          int64_t part_stride, int32_t k, float scale, float *o, float *lse,
                          int32_t *sel_ids_out, int32_t *sel_count_out, void *ws, size_t ws_bytes,
                          void *stream) {
    g_launches = 0;
    ts_status s = check_layout(L);
    if (s != TS_OK) return s;
    if (parts < 1 || k < 1 || part_stride < 0) return TS_ERR_SHAPE;
    if (!aligned16(q) || !aligned16(k_pool) || !aligned16(v_pool) || !aligned16(o)) return TS_ERR_ALIGN;
    const bool f8 = L->kv_dtype == TS_FP8E4M3;
    if ((!f8 && !bf16_attn_supported(L)) || L->page_size % 16 != 0 || group_of(L) > 8 || k > kMaxSel)
        return TS_ERR_UNSUPPORTED;
    const long long pg = (long long)L->max_pages * L->shard_stride;  // global pages of a row
    const size_t scratch = (size_t)((parts * k + 3) & ~3) * 8 + (size_t)((pg + 31) / 32 + 4) * 8 +
                           (kSsHistM + 64 + 128 + (size_t)k) * 4;
    if (scratch > (size_t)8 * SatSmem<4, 8>::kStage || (long long)parts * k > 4096) return TS_ERR_UNSUPPORTED;
    if (!ws || ws_bytes < attn_ws_layout(L, k).total) return TS_ERR_WORKSPACE;
    if (L->batch == 0) return TS_OK;
    AttnParams p = attn_params(L, q, k_pool, v_pool, page_table, seq_lens, nullptr, nullptr, k, scale,
                               o, lse, ws);
    p.cand_scores = cand_scores;
    p.cand_ids = cand_ids;
    p.cand_parts = parts;
    p.cand_k = k;
    p.cand_part_stride = part_stride ? part_stride : (long long)L->batch * L->num_kv_heads * k;
    p.sel_out = sel_ids_out;
    p.sel_cnt_out = sel_count_out;
    return f8 ? launch_sat<8, 16, true>(L, p, true, as_stream(stream)) : launch_sat<4, 8>(L, p, true, as_stream(stream));
}

ts_status ts_select_merge(const float *cand_scores, const int32_t *cand_ids, int32_t parts,
                          int64_t part_stride, int32_t rows, int32_t k_part, int32_t k,
                          int32_t *sel_ids, float *sel_scores, int32_t *sel_count, void *stream) {
    g_launches = 0;
    if (rows < 0 || parts < 1 || k_part < 1 || part_stride < 0) return TS_ERR_CONFIG;
    if (k < 1 || !cand_ids) return TS_ERR_SHAPE;
    if (part_stride == 0) part_stride = (int64_t)rows * k_part;
    return launch_select(cand_scores, rows, k_part, nullptr, cand_ids, 1, 0, k, sel_ids, sel_scores,
                         sel_count, as_stream(stream), parts, part_stride);
}

ts_status ts_lse_merge(int32_t parts, int32_t rows, int32_t d, const float *o_parts,
                       const float *lse_parts, int64_t part_stride, float *o, float *lse,
                       void *stream) {
    g_launches = 0;
    if (parts < 1 || rows < 0 || d < 1 || part_stride < 0) return TS_ERR_CONFIG;
    if (rows == 0) return TS_OK;
    const long long so = part_stride ? part_stride : (long long)rows * d;
    const long long sl = part_stride ? part_stride : (long long)rows;
    launch_pdl(lse_merge_kernel, dim3(rows), dim3(64), 0, as_stream(stream), parts, rows, d, o_parts, lse_parts, so, sl,
                                                         o, lse);
    ++g_launches;
    return launch_status();
}

}  // extern "C"
