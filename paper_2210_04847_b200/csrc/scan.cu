// scan.cu — CUB-free exclusive scans (packing: counts -> offsets; compaction).
//
// Three phases, each a bandwidth-bound pass: (1) per-tile local exclusive scan
// staged through padded shared memory with warp-shuffle sums, (2) a single-CTA
// scan of the tile totals (u64, so an overflow of the 32-bit sample index is
// detectable exactly as pack() does, core_types.cpp:33-36), (3) tile prefixes
// added back. 4096 elements per tile => 1024 tiles at 2^22 rays.
#include "vm_internal.h"

namespace vmb {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;

__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }

template <typename In>
__global__ void __launch_bounds__(kThreads) k_scan_tiles(const In* __restrict__ in, uint64_t n,
                                                         uint32_t* __restrict__ out,
                                                         unsigned long long* __restrict__ tile_sums) {
    __shared__ uint32_t sm[kTile + kTile / 32];
    __shared__ unsigned long long warp_tot[kThreads / 32];
    griddep_wait();
    const uint64_t base = uint64_t(blockIdx.x) * kTile;
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int i = k * kThreads + t;
        uint64_t g = base + i;
        sm[pad(i)] = g < n ? uint32_t(in[g]) : 0u;
    }
    __syncthreads();
    unsigned long long local = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) local += sm[pad(t * kItems + k)];
    // block-wide exclusive scan of `local`
    const int lane = t & 31, warp = t >> 5;
    unsigned long long incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    unsigned long long warp_prefix = 0, block_total = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
        if (w < warp) warp_prefix += warp_tot[w];
        block_total += warp_tot[w];
    }
    unsigned long long run = warp_prefix + incl - local;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int i = pad(t * kItems + k);
        uint32_t v = sm[i];
        sm[i] = uint32_t(run);
        run += v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        int i = k * kThreads + t;
        uint64_t g = base + i;
        if (g < n) out[g] = sm[pad(i)];
    }
    if (t == 0) tile_sums[blockIdx.x] = block_total;
}

// Exclusive scan of the tile totals in place (single CTA, chunked with carry).
__global__ void __launch_bounds__(1024) k_scan_sums(unsigned long long* sums, uint64_t n_tiles,
                                                    unsigned long long* d_total) {
    __shared__ unsigned long long warp_tot[32];
    __shared__ unsigned long long carry;
    griddep_wait();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < n_tiles; base += 1024) {
        uint64_t i = base + t;
        unsigned long long v = i < n_tiles ? sums[i] : 0ull;
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) warp_tot[warp] = incl;
        __syncthreads();
        unsigned long long wp = 0, tot = 0;
        for (int w = 0; w < 32; ++w) {
            if (w < warp) wp += warp_tot[w];
            tot += warp_tot[w];
        }
        if (i < n_tiles) sums[i] = carry + wp + incl - v;
        __syncthreads();
        if (t == 0) carry += tot;
        __syncthreads();
    }
    if (t == 0) *d_total = carry;
}

__global__ void k_scan_add(uint32_t* __restrict__ out, uint64_t n,
                           const unsigned long long* __restrict__ sums) {
    griddep_wait();
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] += uint32_t(sums[i / kTile]);
}

template <typename In>
int scan_impl(vmb_ctx* ctx, const In* in, uint64_t n, uint32_t* out,
              unsigned long long* d_total) {
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(d_total, 0, sizeof(unsigned long long), ctx->stream);
        return e == cudaSuccess ? VMB_OK : cuda_fail(e, "scan");
    }
    uint64_t tiles = (n + kTile - 1) / kTile;
    auto* sums = static_cast<unsigned long long*>(scratch(ctx, SCRATCH_SCAN, tiles * sizeof(unsigned long long)));
    if (!sums) return VMB_CUDA;
    launch_pdl(k_scan_tiles<In>, dim3(unsigned(tiles)), dim3(kThreads), 0, ctx->stream, in, n, out, sums);
    launch_pdl(k_scan_sums, dim3(1), dim3(1024), 0, ctx->stream, sums, tiles, d_total);
    if (tiles > 1) launch_pdl(k_scan_add, dim3(grid_blocks(ctx, n, 256)), dim3(256), 0, ctx->stream, out, n, sums);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "scan");
}

// Single-pass exclusive scan (decoupled look-back) for the march's per-chunk totals:
// each CTA takes the next tile in start order (ticket, so it only ever waits on
// tiles whose CTAs already run), scans it, publishes its aggregate, then sums its
// predecessors' published aggregates / inclusive prefixes from the nearest one back
// and publishes its own inclusive prefix. Status word: flag << 62 | value (1 =
// aggregate, 2 = inclusive prefix). Ticket and status words are zeroed by the caller.
__global__ void __launch_bounds__(kThreads) k_scan_onepass(const uint32_t* __restrict__ in, uint64_t n,
                                                           uint32_t* __restrict__ out, unsigned int* ticket,
                                                           unsigned long long* status, uint64_t n_tiles,
                                                           unsigned long long* __restrict__ d_total) {
    __shared__ uint32_t sm[kTile + kTile / 32];
    __shared__ unsigned long long warp_tot[kThreads / 32];
    __shared__ unsigned int tile_s;
    __shared__ unsigned long long prefix_s;
    griddep_wait();
    const int t = threadIdx.x;
    if (t == 0) tile_s = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = tile_s;
    const uint64_t base = tile * kTile;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int i = k * kThreads + t;
        const uint64_t g = base + i;
        sm[pad(i)] = g < n ? in[g] : 0u;
    }
    __syncthreads();
    unsigned long long local = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) local += sm[pad(t * kItems + k)];
    const int lane = t & 31, warp = t >> 5;
    unsigned long long incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    unsigned long long warp_prefix = 0, block_total = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
        if (w < warp) warp_prefix += warp_tot[w];
        block_total += warp_tot[w];
    }
    constexpr unsigned long long kAgg = 1ull << 62, kIncl = 2ull << 62, kVal = (1ull << 62) - 1;
    if (t == 0) {
        unsigned long long prefix = 0;
        if (tile == 0) {
            atomicExch(status, kIncl | block_total);
        } else {
            atomicExch(status + tile, kAgg | block_total);
            for (uint64_t k = tile; k-- > 0;) {
                unsigned long long w;
                do {
                    w = atomicAdd(status + k, 0ull);
                } while ((w >> 62) == 0);
                prefix += w & kVal;
                if ((w >> 62) == 2) break;
            }
            atomicExch(status + tile, kIncl | (prefix + block_total));
        }
        prefix_s = prefix;
        if (tile == n_tiles - 1) *d_total = prefix + block_total;
    }
    __syncthreads();
    unsigned long long run = prefix_s + warp_prefix + incl - local;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int i = pad(t * kItems + k);
        const uint32_t v = sm[i];
        sm[i] = uint32_t(run);
        run += v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const int i = k * kThreads + t;
        const uint64_t g = base + i;
        if (g < n) out[g] = sm[pad(i)];
    }
}

}  // namespace

uint64_t scan_onepass_tiles(uint64_t n) { return (n + kTile - 1) / kTile; }

// the chunk totals' scan in one kernel; ticket + status: 1 + 2 n_tiles zeroed words
int scan_counts_onepass(vmb_ctx* ctx, const uint32_t* counts, uint64_t n, uint32_t* offsets,
                        unsigned long long* d_total, unsigned int* ticket, unsigned long long* status) {
    if (n == 0) return scan_counts(ctx, counts, n, offsets, d_total);
    const uint64_t tiles = scan_onepass_tiles(n);
    launch_pdl(k_scan_onepass, dim3(unsigned(tiles)), dim3(kThreads), 0, ctx->stream, counts, n, offsets, ticket,
               status, tiles, d_total);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "scan");
}

int scan_counts(vmb_ctx* ctx, const uint32_t* counts, uint64_t n, uint32_t* offsets,
                unsigned long long* d_total) {
    return scan_impl<uint32_t>(ctx, counts, n, offsets, d_total);
}

int scan_flags(vmb_ctx* ctx, const uint8_t* flags, uint64_t n, uint32_t* pos,
               unsigned long long* d_total) {
    return scan_impl<uint8_t>(ctx, flags, n, pos, d_total);
}

}  // namespace vmb
