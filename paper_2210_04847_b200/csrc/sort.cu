// sort.cu — in-tree stable LSD radix sort of (u32 key, u32 value) pairs.
//
// Used by the deterministic voxel-field backward (voxfield.cu), which needs each
// vertex's records in sample order (the reference's left fold, fields.hpp:76-81).
// 8-bit digits, tiles of kSortThreads x kSortRounds items; per pass:
//   1. k_digit_hist   per tile, the count of each digit -> hist[digit][tile]
//   2. scan_counts    exclusive scan of hist in digit-major order (scan.cu) = the
//                     first output position of (digit, tile)
//   3. k_digit_scatter per tile, in the tile's item order (round-major: item
//                     r * kSortThreads + t), each item's rank among the equal
//                     digits before it — warp match + per-warp digit counts in
//                     shared memory — so equal keys keep their input order.
// ceil(end_bit / 8) passes ping-pong between the two buffers.
#include "vm_internal.h"

namespace vmb {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortRounds = 8;
constexpr int kSortTile = kSortThreads * kSortRounds;
constexpr int kSortWarps = kSortThreads / 32;

__global__ void __launch_bounds__(kSortThreads) k_digit_hist(const uint32_t* __restrict__ keys, uint64_t m,
                                                             int shift, uint32_t* __restrict__ hist,
                                                             uint64_t n_tiles) {
    __shared__ uint32_t cnt[256];
    const int t = threadIdx.x;
    cnt[t] = 0u;
    __syncthreads();
    const uint64_t base = uint64_t(blockIdx.x) * kSortTile;
#pragma unroll
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t e = base + uint64_t(r) * kSortThreads + t;
        if (e < m) atomicAdd(&cnt[(keys[e] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[uint64_t(t) * n_tiles + blockIdx.x] = cnt[t];
}

__global__ void __launch_bounds__(kSortThreads) k_digit_scatter(
    const uint32_t* __restrict__ k_in, const uint32_t* __restrict__ v_in, uint32_t* __restrict__ k_out,
    uint32_t* __restrict__ v_out, uint64_t m, int shift, const uint32_t* __restrict__ pos, uint64_t n_tiles) {
    __shared__ uint32_t run[256];                    // items of each digit placed so far in this tile
    __shared__ uint32_t wcnt[kSortWarps][256];      // this round: items of each digit per warp
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    run[t] = 0u;
#pragma unroll
    for (int q = 0; q < kSortWarps; ++q) wcnt[q][t] = 0u;
    __syncthreads();
    const uint64_t base = uint64_t(blockIdx.x) * kSortTile;
    for (int r = 0; r < kSortRounds; ++r) {
        const uint64_t e = base + uint64_t(r) * kSortThreads + t;
        const bool in = e < m;
        const uint32_t key = in ? k_in[e] : 0u;
        const uint32_t val = in ? v_in[e] : 0u;
        const uint32_t dg = in ? (key >> shift) & 255u : 256u + uint32_t(lane);  // unique dummy digits
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const uint32_t rank_w = __popc(peers & ((1u << lane) - 1u));
        if (in && rank_w == 0) wcnt[w][dg] = __popc(peers);
        __syncthreads();
        if (in) {
            uint32_t before = run[dg];
            for (int q = 0; q < w; ++q) before += wcnt[q][dg];
            const uint32_t p = pos[uint64_t(dg) * n_tiles + blockIdx.x] + before + rank_w;
            k_out[p] = key;
            v_out[p] = val;
        }
        __syncthreads();
        uint32_t add = 0u;
#pragma unroll
        for (int q = 0; q < kSortWarps; ++q) {
            add += wcnt[q][t];
            wcnt[q][t] = 0u;
        }
        run[t] += add;
        __syncthreads();
    }
}

}  // namespace

// Sorts m pairs by the low end_bit bits of the keys, stably. The pairs start in
// (k0, v0); (k1, v1) is the other buffer; on return *k_res / *v_res point at the
// sorted pairs (one of the two buffers).
int radix_sort_pairs(vmb_ctx* ctx, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint64_t m, int end_bit,
                     uint32_t** k_res, uint32_t** v_res) {
    *k_res = k0;
    *v_res = v0;
    if (m == 0) return VMB_OK;
    const uint64_t n_tiles = (m + kSortTile - 1) / kSortTile;
    auto* hist = static_cast<uint32_t*>(scratch(ctx, SCRATCH_MISC, size_t(2) * 256 * n_tiles * sizeof(uint32_t) + 64));
    if (!hist) return VMB_CUDA;
    uint32_t* pos = hist + 256 * n_tiles;
    uint32_t *ki = k0, *vi = v0, *ko = k1, *vo = v1;
    for (int shift = 0; shift < end_bit; shift += 8) {
        k_digit_hist<<<unsigned(n_tiles), kSortThreads, 0, ctx->stream>>>(ki, m, shift, hist, n_tiles);
        int rc = scan_counts(ctx, hist, 256 * n_tiles, pos, ctx->d_u64 + 2);
        if (rc) return rc;
        k_digit_scatter<<<unsigned(n_tiles), kSortThreads, 0, ctx->stream>>>(ki, vi, ko, vo, m, shift, pos,
                                                                             n_tiles);
        uint32_t* tk = ki;
        ki = ko;
        ko = tk;
        uint32_t* tv = vi;
        vi = vo;
        vo = tv;
    }
    *k_res = ki;
    *v_res = vi;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "radix sort");
}

}  // namespace vmb
