// score_select.cuh — Alg. 1 Steps 1-2 fused for ts_decode_step: page
// scoring, then the top-K of the row by the LAST CTA to finish scoring it (atomic ticket;
// "last finisher runs the successor"), which publishes the selection with a per-row
// release flag.  The attention kernel (attn_stream.cuh) is launched with programmatic
// dependent launch and grabs rows in order as their flags are released, so KV streaming
// of selected rows overlaps the scoring of later rows.  The kernel triggers its dependents
// at entry: the attention grid becomes resident as soon as every scoring CTA has started.
#pragma once
#include "common.cuh"
#include "score.cuh"
#include "select.cuh"

namespace ts {

struct FusedSelect {
    int *sel_ids;         // [rows][k]
    int *sel_count;       // [rows]
    unsigned *tickets;    // [rows] scoring tickets (self re-arming)
    unsigned *ready;      // [rows] released after the selection is written
    int k;
};

template <int D>
__global__ void __launch_bounds__(kScoreWarps * 32)
    score_select_kernel(ScoreParams p, const uint16_t *__restrict__ q,
                        const uint16_t *__restrict__ meta, const int *__restrict__ page_table,
                        const int *__restrict__ seq_lens, float *__restrict__ scores, FusedSelect fs) {
    extern __shared__ uint32_t keys[];  // [max_pages]
    __shared__ SelectSmem<kScoreWarps * 32> S;
    __shared__ int s_last;
    pdl_launch_dependents();
    const int row = blockIdx.y;
    score_mma_block<D>(p, q, meta, page_table, seq_lens, scores, row, blockIdx.x);
    if (gridDim.x > 1) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) s_last = atomicAdd(fs.tickets + row, 1u) == gridDim.x - 1;
        __syncthreads();
        if (!s_last) return;
        __threadfence();
    } else {
        __syncthreads();
    }
    SelectParams sp{scores, 0, p.max_pages, nullptr, nullptr, 1, 0, fs.k, p.max_pages, 0,
                    fs.sel_ids, nullptr, fs.sel_count};
    select_row<kScoreWarps * 32>(sp, row, keys, S);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (gridDim.x > 1) fs.tickets[row] = 0u;
        st_release_u32(fs.ready + row, 1u);
    }
}

}  // namespace ts
