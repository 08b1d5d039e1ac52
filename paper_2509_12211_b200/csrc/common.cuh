// common.cuh — sm_100a device helpers shared by the TinyServe kernels (product path only).
// PTX wrappers: mbarrier, TMA tile loads (cp.async.bulk.tensor), legacy-tensor-core
// mma.sync (bf16 m16n8k16 / m16n8k8, f16 m16n8k16), bf16 / f16 <-> fp32 conversions.
#pragma once
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define TS_DEV __device__ __forceinline__

namespace ts {

namespace cg = cooperative_groups;

constexpr float kNegInf = -__builtin_huge_valf();
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ---------------------------------------------------------------- bf16 bit helpers
// A bf16 is the top 16 bits of an fp32: widening is a shift, exact.
TS_DEV float bf16lo_to_f32(uint32_t packed) { return __uint_as_float(packed << 16); }
TS_DEV float bf16hi_to_f32(uint32_t packed) { return __uint_as_float(packed & 0xffff0000u); }
TS_DEV float bf16_to_f32(uint16_t h) { return __uint_as_float(uint32_t(h) << 16); }

// bf16 pair helpers on packed registers (lo = lower address / lower index)
TS_DEV uint32_t bf16x2_max0(uint32_t x) {  // elementwise max(x, 0)   (exact)
    uint32_t r;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(0u));
    return r;
}
TS_DEV uint32_t bf16x2_min0(uint32_t x) {  // elementwise min(x, 0)   (exact)
    uint32_t r;
    asm("min.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(0u));
    return r;
}
TS_DEV uint32_t bf16x2_min(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
TS_DEV uint32_t bf16x2_max(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// ---------------------------------------------------------------- 128-bit global loads
TS_DEV uint4 ldg_nc_v4(const void *p) {  // streaming read-only, no L1 allocation
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
TS_DEV uint4 ldg_v4(const void *p) {
    uint4 r;
    asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
TS_DEV uint4 lds_v4(uint32_t saddr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(saddr));
    return r;
}
TS_DEV uint2 lds_v2(uint32_t saddr) {
    uint2 r;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(saddr));
    return r;
}
TS_DEV int lds_s8(uint32_t saddr) {
    int r;
    asm volatile("ld.shared.s8 %0, [%1];" : "=r"(r) : "r"(saddr));
    return r;
}
TS_DEV void sts_v4(uint32_t saddr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w));
}
TS_DEV uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

// ---------------------------------------------------------------- mbarrier
TS_DEV void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
TS_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
TS_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// generic-proxy writes (shared or global) ordered before this thread's later async-proxy
// (TMA / bulk copy) accesses
TS_DEV void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
TS_DEV void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// expect `bytes` more transaction bytes in the current phase, WITHOUT an arrive
TS_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
TS_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

TS_DEV void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// ---------------------------------------------------------------- sync / ordering
TS_DEV void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
TS_DEV uint32_t ld_acquire_u32(const unsigned *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
TS_DEV uint32_t ld_relaxed_u32(const unsigned *p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// ticket: atomic add with acquire-release semantics at GPU scope (after a CTA barrier, the
// release is cumulative over the CTA's prior writes; no separate membar round trip)
TS_DEV uint32_t atom_add_acq_rel_gpu(unsigned *p, unsigned v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
TS_DEV void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
TS_DEV void st_release_u32(unsigned *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
TS_DEV void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
TS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
TS_DEV void nanosleep_ns(uint32_t ns) { asm volatile("nanosleep.u32 %0;" ::"r"(ns)); }
TS_DEV uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------- TMA
TS_DEV uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 2-D tile load: box at (x = column, y = row) of the tensor map into smem, completing
// `bytes` transaction bytes on the mbarrier.
TS_DEV void tma_load_2d(uint32_t dst, const CUtensorMap *map, int32_t x, int32_t y, uint32_t bar,
                        uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::"
        "cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(map), "r"(x), "r"(y), "r"(bar), "l"(policy)
        : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, multiple of 16 bytes).
TS_DEV void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
// 1-D bulk copy with an L2 cache-policy hint (streaming data: evict_first).
TS_DEV void bulk_load_hint(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                           uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
}
// Ampere-style async copy, 16 B global -> shared (L2 only), and its mbarrier hook: the
// barrier receives one arrival from this thread once all its prior cp.async complete.
TS_DEV void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
TS_DEV void cp_async_mbar_arrive(uint32_t bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
// L2 prefetch of a contiguous run (16-byte aligned, multiple of 16 bytes); no smem, no barrier
TS_DEV void prefetch_l2_bulk(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
TS_DEV void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ---------------------------------------------------------------- mma.sync
// D[16x8] += A[16x16] * B[16x8], bf16 inputs, fp32 accumulate.
TS_DEV void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D[16x8] += A[16x8] * B[8x8], bf16 inputs, fp32 accumulate.
TS_DEV void mma_bf16_1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(b0));
}
// D[16x8] += A[16x16] * B[16x8], f16 inputs, fp32 accumulate (the FP8 KV path: E4M3 codes
// widen exactly to f16).
TS_DEV void mma_f16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                          uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// two fp32 -> packed bf16x2 (lo = element 0), round to nearest even
TS_DEV uint32_t bf16x2_pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// word i of a uint4 (i a compile-time constant after unrolling)
TS_DEV uint32_t u4_word(const uint4 &v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }
// two fp32 -> packed f16x2 (lo = element 0), round to nearest even
TS_DEV uint32_t f16x2_pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}
// ---------------------------------------------------------------- misc
TS_DEV float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
TS_DEV float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- TS_DEBUG error word
// Data-dependent faults the host cannot see without a sync (include/tinyserve.h "ERRORS"):
// in the dev build (-DTS_DEV_KNOBS, libtinyserve_dev.so) the kernels OR a bit into a device
// word, read back by ts_debug_error_word(); the release build compiles the checks away.
//   bit 0: seq_len < 0 or beyond the page-table row's capacity (max_pages * stride * S)
//   bit 1: a page-table entry the kernel dereferences is outside [0, num_blocks)
constexpr unsigned kDbgSeqLen = 1u, kDbgBlock = 2u;
#ifdef TS_DEV_KNOBS
__device__ unsigned g_ts_debug_err = 0u;
TS_DEV void debug_flag(bool bad, unsigned bit) {
    if (bad) atomicOr(&g_ts_debug_err, bit);
}
#else
TS_DEV void debug_flag(bool, unsigned) {}
#endif
// a physical block read from the page table (checked in the dev build)
TS_DEV int checked_block(int blk, int num_blocks) {
    debug_flag(blk < 0 || blk >= num_blocks, kDbgBlock);
    return blk;
}

// Sequence length as the kernels see it: at most the capacity of the page-table row
// (global pages < max_pages * stride).  seq_len beyond it is a caller error (undefined per
// include/tinyserve.h); clamping keeps every read inside the row and the pools' pages.
TS_DEV int clamp_len(int L, int max_pages, int stride, int S) {
    const long long cap = (long long)max_pages * stride * S;
    debug_flag(L < 0 || L > cap, kDbgSeqLen);
    return L < cap ? L : (int)cap;
}

// local page count of a sequence of L tokens under block-cyclic ownership:
// global pages j < ceil(L / S) with j % stride == offset
TS_DEV int local_pages(int L, int S, int stride, int offset) {
    const int P = (L + S - 1) / S;
    return P > offset ? (P - offset + stride - 1) / stride : 0;
}

// Orderable key of an fp32 score: larger score <-> larger unsigned key; -0.0 == +0.0.
TS_DEV uint32_t score_key(float s) {
    uint32_t u = __float_as_uint(s + 0.0f);  // -0.0 + 0.0 = +0.0 (round-to-nearest)
    return (u >> 31) ? ~u : (u | 0x80000000u);
}
TS_DEV float key_score(uint32_t k) {
    return __uint_as_float((k >> 31) ? (k & 0x7fffffffu) : ~k);
}
constexpr uint32_t kKeyNegInf = 0x007fffffu;  // score_key(-inf)

}  // namespace ts
