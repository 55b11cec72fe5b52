// grid.cu — device-resident OccupancyGrid (occupancy_grid.cpp).
//
// HBM layout per grid (R = resolution, n = R^3):
//   cache  f64[n]            density EMA (occupancy_grid.hpp:87)
//   bits   u32[ceil(n/32)]   packed occupancy, cell c -> word c/32 bit c%32;
//                            byte-for-byte the OGRD bit section (LSB-first, x-fastest)
//   coarse u32[..]           1-cell-dilated occupancy of 8^3-cell blocks for the
//                            empty-space-skipping marcher (see march.cu)
// Update is one fused, bandwidth-bound pass per cell word: probe (splitmix64 jitter,
// inverse contraction, analytic density, max over timestamps) -> EMA -> threshold ->
// warp ballot into the bit word. 16.125 B of HBM traffic per cell.
#include <cstring>
#include <string>

#include <algorithm>

#include "vm_internal.h"

namespace vmb {

int check_contraction(const vmb_contraction* c);

namespace {

struct GridDev {
    Contract k;
    uint32_t res;
    uint64_t n;
    double thr, ref_step;
};

GridDev dev_of(const vmb_grid* g) { return GridDev{g->k, g->res, g->n_cells, g->thr, g->ref_step}; }

// refresh_bits (occupancy_grid.cpp:58-61) for one cell
__device__ __forceinline__ bool occupied_bit(double cache, double ref_step, double thr) {
    return (1.0 - exp(-cache * ref_step)) > thr;
}

constexpr int kMaxTimestamps = 64;
struct Timestamps {
    double t[kMaxTimestamps];
    int n;
};

// Probe of one cell with an analytic field over all timestamps
// (occupancy_grid.cpp:106-140). Returns the max density (0 when the cell has no
// preimage); sets *bad to the first timestamp index with an invalid density.
template <bool VOX>
__device__ __forceinline__ double probe_cell(const GridDev& g, const vmb_field& f,
                                             const Timestamps& ts, uint64_t cell, bool has_seed,
                                             uint64_t seed, int* bad) {
    D3 w;
    *bad = -1;
    if (!invert(g.k, probe_point(cell, g.res, has_seed, seed), &w)) return 0.0;
    double probed = 0.0;
    for (int i = 0; i < ts.n; ++i) {
        double d = field_density_t<VOX>(f, time_shift(f, w, ts.t[i]));
        if (!isfinite(d) || d < 0.0) {
            *bad = i;
            return probed;
        }
        if (d > probed) probed = d;
    }
    return probed;
}

// Fused update for a field that cannot produce invalid densities.
template <bool VOX>
__global__ void __launch_bounds__(256) k_update_fused(GridDev g, vmb_field f, Timestamps ts,
                                                      bool has_seed, uint64_t seed, double decay,
                                                      double* __restrict__ cache,
                                                      uint32_t* __restrict__ bits, uint64_t n_words) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = warp; w < n_words; w += n_warps) {
        uint64_t cell = w * 32 + lane;
        bool bit = false;
        if (cell < g.n) {
            int bad;
            double probed = probe_cell<VOX>(g, f, ts, cell, has_seed, seed, &bad);
            double c = max_ref(cache[cell] * decay, probed);
            cache[cell] = c;
            bit = occupied_bit(c, g.ref_step, g.thr);
        }
        unsigned word = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) bits[w] = word;
    }
}

// Error scan for fields whose sigma is invalid: first (timestamp, cell) wins.
template <bool VOX>
__global__ void k_update_errors(GridDev g, vmb_field f, Timestamps ts, bool has_seed,
                                uint64_t seed, DevError* err) {
    for (uint64_t cell = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < g.n;
         cell += uint64_t(gridDim.x) * blockDim.x) {
        int bad;
        probe_cell<VOX>(g, f, ts, cell, has_seed, seed, &bad);
        if (bad >= 0) atomicMin(&err->key, (unsigned long long)((uint64_t(bad) << 40) | cell));
    }
}

// Sharded probe (multi-GPU): cells [c0, c1) of this rank, zero elsewhere.
template <bool VOX>
__global__ void k_probe_range(GridDev g, vmb_field f, Timestamps ts, bool has_seed, uint64_t seed,
                              uint64_t c0, uint64_t c1, double* __restrict__ probed) {
    for (uint64_t cell = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < g.n;
         cell += uint64_t(gridDim.x) * blockDim.x) {
        double v = 0.0;
        if (cell >= c0 && cell < c1) {
            int bad;
            v = probe_cell<VOX>(g, f, ts, cell, has_seed, seed, &bad);
        }
        probed[cell] = v;
    }
}

// The cells [c0, c1) only, each at its own index (the block of an all-gather).
template <bool VOX>
__global__ void k_probe_block(GridDev g, vmb_field f, Timestamps ts, bool has_seed, uint64_t seed, uint64_t c0,
                              uint64_t c1, double* __restrict__ probed) {
    for (uint64_t cell = c0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < c1;
         cell += uint64_t(gridDim.x) * blockDim.x) {
        int bad;
        probed[cell] = probe_cell<VOX>(g, f, ts, cell, has_seed, seed, &bad);
    }
}

// cache = max(cache * decay, probed); bits (occupancy_grid.cpp:142-143)
__global__ void __launch_bounds__(256) k_apply(GridDev g, const double* __restrict__ probed,
                                               double decay, double* __restrict__ cache,
                                               uint32_t* __restrict__ bits, uint64_t n_words) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = warp; w < n_words; w += n_warps) {
        uint64_t cell = w * 32 + lane;
        bool bit = false;
        if (cell < g.n) {
            double c = max_ref(cache[cell] * decay, probed[cell]);
            cache[cell] = c;
            bit = occupied_bit(c, g.ref_step, g.thr);
        }
        unsigned word = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) bits[w] = word;
    }
}

// bits from cache only (constructor, seed_occupancy)
__global__ void __launch_bounds__(256) k_refresh(GridDev g, const double* __restrict__ cache,
                                                 uint32_t* __restrict__ bits, uint64_t n_words) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t w = warp; w < n_words; w += n_warps) {
        uint64_t cell = w * 32 + lane;
        bool bit = cell < g.n && occupied_bit(cache[cell], g.ref_step, g.thr);
        unsigned word = __ballot_sync(0xffffffffu, bit);
        if (lane == 0) bits[w] = word;
    }
}

__global__ void k_fill(double* __restrict__ p, uint64_t n, double v) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        p[i] = v;
}

__global__ void k_seed_mask(const uint8_t* __restrict__ mask, uint64_t n, double high,
                            double* __restrict__ cache) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        cache[i] = mask[i] ? high : 0.0;
}

// Dilated coarse occupancy: block K covers fine cells [K*B-1, (K+1)*B] per axis.
__global__ void k_coarse(const uint32_t* __restrict__ bits, uint32_t res, uint32_t block,
                         uint32_t res_c, uint32_t* __restrict__ coarse, uint64_t coarse_words) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t nc = uint64_t(res_c) * res_c * res_c;
    for (uint64_t w = warp; w < coarse_words; w += n_warps) {
        uint64_t kc = w * 32 + lane;
        bool any = false;
        if (kc < nc) {
            int kx = int(kc % res_c), ky = int((kc / res_c) % res_c), kz = int(kc / (uint64_t(res_c) * res_c));
            int x0 = max(kx * int(block) - 1, 0), x1 = min((kx + 1) * int(block), int(res) - 1);
            int y0 = max(ky * int(block) - 1, 0), y1 = min((ky + 1) * int(block), int(res) - 1);
            int z0 = max(kz * int(block) - 1, 0), z1 = min((kz + 1) * int(block), int(res) - 1);
            for (int z = z0; z <= z1 && !any; ++z)
                for (int y = y0; y <= y1 && !any; ++y) {
                    // cells [row + x0, row + x1] of one x-row: OR of masked words
                    uint64_t row = (uint64_t(y) + uint64_t(res) * uint64_t(z)) * res;
                    uint64_t c0 = row + x0, c1 = row + x1;
                    for (uint64_t w = c0 >> 5; w <= (c1 >> 5); ++w) {
                        uint32_t lo = w == (c0 >> 5) ? uint32_t(c0 & 31) : 0u;
                        uint32_t hi = w == (c1 >> 5) ? uint32_t(c1 & 31) : 31u;
                        uint32_t mask = (hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u)) & ~((1u << lo) - 1u);
                        if (__ldg(bits + w) & mask) {
                            any = true;
                            break;
                        }
                    }
                }
        }
        unsigned word = __ballot_sync(0xffffffffu, any);
        if (lane == 0) coarse[w] = word;
    }
}

// Bounding box of the occupied cells (min and max+1 per axis) by warp reductions
// and one atomic per warp and axis; bbox is preset to {~0 x3, 0 x3}.
__global__ void k_bbox(const uint32_t* __restrict__ bits, uint32_t res, uint64_t n_words,
                       uint32_t* __restrict__ bbox) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < n_words; w += stride) {
        uint32_t m = __ldg(bits + w);
        if (m && res % 32 == 0) {  // the word is one piece of an x-row: O(1)
            const uint64_t c0 = w * 32;
            const uint32_t xb = uint32_t(c0 % res), y = uint32_t((c0 / res) % res), z = uint32_t(c0 / (uint64_t(res) * res));
            lo[0] = min(lo[0], xb + uint32_t(__ffs(m) - 1)), hi[0] = max(hi[0], xb + 32u - uint32_t(__clz(m)));
            lo[1] = min(lo[1], y), lo[2] = min(lo[2], z);
            hi[1] = max(hi[1], y + 1), hi[2] = max(hi[2], z + 1);
            m = 0;
        }
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1u;
            const uint64_t c = w * 32 + uint64_t(b);
            const uint32_t x = uint32_t(c % res), y = uint32_t((c / res) % res), z = uint32_t(c / (uint64_t(res) * res));
            lo[0] = min(lo[0], x), lo[1] = min(lo[1], y), lo[2] = min(lo[2], z);
            hi[0] = max(hi[0], x + 1), hi[1] = max(hi[1], y + 1), hi[2] = max(hi[2], z + 1);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __reduce_min_sync(0xffffffffu, lo[a]);
        hi[a] = __reduce_max_sync(0xffffffffu, hi[a]);
    }
    if ((threadIdx.x & 31) == 0 && hi[0]) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(bbox + a, lo[a]);
            atomicMax(bbox + 3 + a, hi[a]);
        }
    }
}

__global__ void k_popcount(const uint32_t* __restrict__ bits, uint64_t n_words,
                           unsigned long long* out) {
    unsigned long long local = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n_words;
         i += uint64_t(gridDim.x) * blockDim.x)
        local += __popc(bits[i]);
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

__global__ void k_query(GridDev g, const uint32_t* __restrict__ bits, const double* __restrict__ pts,
                        uint64_t n, uint8_t* __restrict__ out, DevError* err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        D3 p = d3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        if (!finite3(p)) {
            atomicMin(&err->key, (unsigned long long)i);
            out[i] = 0;
            continue;
        }
        int64_t c = cell_of_point(g.k, g.res, p);
        out[i] = c >= 0 && ((bits[uint64_t(c) >> 5] >> (uint64_t(c) & 31)) & 1u);
    }
}

// Probe points of the generic callback path: flags + world points per cell.
__global__ void k_probe_points(GridDev g, bool has_seed, uint64_t seed, double* __restrict__ world,
                               uint8_t* __restrict__ valid) {
    for (uint64_t cell = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < g.n;
         cell += uint64_t(gridDim.x) * blockDim.x) {
        D3 w = d3(0, 0, 0);
        bool ok = invert(g.k, probe_point(cell, g.res, has_seed, seed), &w);
        valid[cell] = ok;
        world[3 * cell] = w.x;
        world[3 * cell + 1] = w.y;
        world[3 * cell + 2] = w.z;
    }
}

__global__ void k_compact_points(uint64_t n, const double* __restrict__ world,
                                 const uint8_t* __restrict__ valid, const uint32_t* __restrict__ pos,
                                 double* __restrict__ points, uint32_t* __restrict__ cells) {
    for (uint64_t cell = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; cell < n;
         cell += uint64_t(gridDim.x) * blockDim.x) {
        if (!valid[cell]) continue;
        uint32_t k = pos[cell];
        points[3 * uint64_t(k)] = world[3 * cell];
        points[3 * uint64_t(k) + 1] = world[3 * cell + 1];
        points[3 * uint64_t(k) + 2] = world[3 * cell + 2];
        cells[k] = uint32_t(cell);
    }
}

__global__ void k_accumulate(const double* __restrict__ dens, const uint32_t* __restrict__ cells,
                             uint64_t n, double* __restrict__ probed, DevError* err) {
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        double d = dens[k];
        uint32_t c = cells[k];
        if (!isfinite(d) || d < 0.0) {
            atomicMin(&err->key, (unsigned long long)k);
            continue;
        }
        if (d > probed[c]) probed[c] = d;
    }
}

std::string cell_name(const vmb_grid* g, uint64_t c) {
    uint32_t R = g->res;
    return "occupancy grid: invalid density at cell (" + std::to_string(c % R) + "," +
           std::to_string((c / R) % R) + "," + std::to_string(c / (uint64_t(R) * R)) + ")";
}

int launch_check(const char* where) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, where);
}

int grid_alloc(vmb_grid* g) {
    g->n_cells = uint64_t(g->res) * g->res * g->res;
    g->n_words = (g->n_cells + 31) / 32;
    g->res_c = (g->res + g->block - 1) / g->block;
    g->coarse_words = (uint64_t(g->res_c) * g->res_c * g->res_c + 31) / 32;
    cudaError_t e = cudaMalloc(&g->cache, g->n_cells * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&g->bits, g->n_words * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&g->coarse, g->coarse_words * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc(&g->dist, g->n_cells);
    if (e == cudaSuccess) e = cudaMalloc(&g->dist_tmp, g->n_cells);
    if (e == cudaSuccess) e = cudaMalloc(&g->bbox, 6 * sizeof(uint32_t));
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "grid allocation");
}

double domain_diagonal(const vmb_contraction& c) {  // occupancy_grid.cpp:16-21
    if (c.kind == VMB_CONTRACT_AABB) {
        D3 s = d3(c.box_max[0] - c.box_min[0], c.box_max[1] - c.box_min[1],
                  c.box_max[2] - c.box_min[2]);
        return norm(s);
    }
    return 2.0 * c.radius * std::sqrt(3.0);
}

int make_timestamps(const double* h_ts, uint64_t n, Timestamps* ts) {
    if (n == 0) return fail(VMB_INVALID_ARGUMENT, "occupancy grid: timestamps must be non-empty");
    if (n > uint64_t(kMaxTimestamps))
        return fail(VMB_NOT_SUPPORTED, "occupancy grid: at most 64 timestamps per device update");
    ts->n = int(n);
    for (uint64_t i = 0; i < n; ++i) ts->t[i] = h_ts[i];
    return VMB_OK;
}

// Capped Chebyshev distance transform, separable (x, then y, then z):
//   D_x(c)   = min |dx| over occupied cells on the x-line (cap if none within cap-1)
//   D_y(c)   = min over |dy| < cap of max(|dy|, D_x(c + dy e_y)),  same for z.
// The composition is exactly the L-inf distance to the nearest occupied cell,
// capped at kDistCap.
static_assert(kDistCap >= 1 && kDistCap <= 16, "the x pass reads a 2 * kDistCap - 1 bit window");

// bits [lo, lo + 63] of the packed bitfield (cells outside [0, n) read as 0)
__device__ __forceinline__ uint64_t bits64(const uint32_t* __restrict__ bits, int64_t lo, uint64_t n_words) {
    const int64_t neg = lo < 0 ? -lo : 0;  // cells before 0 read as 0 (|lo| < 16 here)
    const uint64_t start = uint64_t(lo + neg);
    const uint64_t q = start >> 5, sh = start & 31;
    const uint64_t w0 = q < n_words ? __ldg(bits + q) : 0u;
    const uint64_t w1 = q + 1 < n_words ? __ldg(bits + q + 1) : 0u;
    const uint64_t w2 = q + 2 < n_words ? __ldg(bits + q + 2) : 0u;
    const uint64_t w = ((w0 | (w1 << 32)) >> sh) | (sh ? (w2 << (64 - sh)) : 0ull);
    return w << neg;
}

// x pass: the window [c - (cap-1), c + (cap-1)] of the row, clipped to the row,
// nearest set bit on each side by clz / ffs.
__global__ void k_dist_x(const uint32_t* __restrict__ bits, uint32_t res, uint64_t n, uint64_t n_words,
                         uint8_t* __restrict__ out) {
    griddep_wait();
    constexpr int W = kDistCap - 1;
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < n;
         c += uint64_t(gridDim.x) * blockDim.x) {
        const int x = int(c % res);
        const int64_t lo = int64_t(c) - W;
        uint64_t w = bits64(bits, lo, n_words);
        // keep bit positions p <= 2W with lo + p inside this row [c - x, c - x + res)
        const int pmin = x < W ? W - x : 0;                        // row start
        const int pmax = min(2 * W, W + (int(res) - 1 - x));        // row end / window end
        const uint64_t keep = (pmax >= 63 ? ~0ull : ((1ull << (pmax + 1)) - 1)) & (~0ull << pmin);
        w &= keep;
        int best = kDistCap;
        const uint64_t left = w & ((2ull << W) - 1);  // positions 0..W: cells c-W .. c
        if (left) best = W - (63 - __clzll(left));
        const uint64_t right = w >> W;                 // cell c at bit 0
        if (right) best = min(best, __ffsll(right) - 1);
        out[c] = uint8_t(best);
    }
}

// y / z pass over shared-memory tiles: a block holds one full line of 32
// neighbouring x columns (tile[t][x]); each cell scans |dd| < its current best.
__global__ void k_dist_axis_tiled(const uint8_t* __restrict__ in, uint32_t res, uint64_t stride,
                                  uint64_t ostride, uint8_t* __restrict__ out) {
    extern __shared__ uint8_t tile[];  // [res][32]
    griddep_wait();
    const uint32_t ntx = (res + 31) / 32;
    const uint32_t other = blockIdx.x / ntx, x0 = (blockIdx.x % ntx) * 32;
    const int lane = threadIdx.x & 31, row = threadIdx.x >> 5, rows = blockDim.x >> 5;
    const uint32_t x = x0 + lane;
    const bool valid = x < res;
    const uint64_t base = x + uint64_t(other) * ostride;
    for (uint32_t t = row; t < res; t += rows) tile[t * 32 + lane] = valid ? __ldg(in + base + t * stride) : kDistCap;
    __syncthreads();
    if (!valid) return;
    for (int t = row; t < int(res); t += rows) {
        int best = tile[t * 32 + lane];
        for (int dd = 1; dd < best; ++dd) {
            if (t - dd >= 0) best = min(best, max(dd, int(tile[(t - dd) * 32 + lane])));
            if (t + dd < int(res)) best = min(best, max(dd, int(tile[(t + dd) * 32 + lane])));
        }
        out[base + t * stride] = uint8_t(best);
    }
}

}  // namespace

// The dilated coarse bits serve only walk_skip (the fp64 DDA used when the fp32
// fast walk does not apply), so they are built on that path's first use after a
// change of the bits, synchronously (any context may then read them).
int grid_ensure_coarse(vmb_ctx* ctx, const vmb_grid* cg) {
    auto* g = const_cast<vmb_grid*>(cg);
    if (g->coarse_valid) return VMB_OK;
    k_coarse<<<grid_blocks(ctx, g->coarse_words * 32, 256), 256, 0, ctx->stream>>>(
        g->bits, g->res, g->block, g->res_c, g->coarse, g->coarse_words);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "grid coarse");
    g->coarse_valid = true;
    return VMB_OK;
}

int grid_rebuild_coarse(vmb_ctx* ctx, vmb_grid* g) {
    g->coarse_valid = false;
    const int blocks = grid_blocks(ctx, g->n_cells, 256);
    launch_pdl(k_dist_x, dim3(blocks), dim3(256), 0, ctx->stream, g->bits, g->res, g->n_cells, g->n_words, g->dist);
    const uint64_t r = g->res, plane = r * r;
    const uint32_t tiles = uint32_t(r * ((r + 31) / 32));
    const size_t smem = size_t(r) * 32;  // one line of 32 columns
    static const bool opted = [] {      // lines beyond 48 KB of shared memory (res > 1536)
        return cudaFuncSetAttribute(k_dist_axis_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) ==
               cudaSuccess;
    }();
    (void)opted;
    launch_pdl(k_dist_axis_tiled, dim3(tiles), dim3(256), smem, ctx->stream, g->dist, g->res, r, plane, g->dist_tmp);
    launch_pdl(k_dist_axis_tiled, dim3(tiles), dim3(256), smem, ctx->stream, g->dist_tmp, g->res, plane, r, g->dist);
    cudaMemsetAsync(g->bbox, 0xff, 3 * sizeof(uint32_t), ctx->stream);
    cudaMemsetAsync(g->bbox + 3, 0, 3 * sizeof(uint32_t), ctx->stream);
    k_bbox<<<grid_blocks(ctx, g->n_words, 256, 4), 256, 0, ctx->stream>>>(g->bits, g->res, g->n_words, g->bbox);
    return launch_check("grid coarse/dist");
}

int grid_refresh(vmb_ctx* ctx, vmb_grid* g) {
    launch_pdl(k_refresh, dim3(grid_blocks(ctx, g->n_words * 32, 256)), dim3(256), 0, ctx->stream, dev_of(g), g->cache,
                                                                                g->bits, g->n_words);
    int rc = launch_check("grid refresh");
    return rc ? rc : grid_rebuild_coarse(ctx, g);
}

}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_comm_allreduce_max_f64(vmb_ctx* ctx, double* d_buf, uint64_t n);

int vmb_grid_create(vmb_ctx* ctx, uint32_t res, const vmb_contraction* c, double thr,
                    double ref_step, double init, vmb_grid** out) {
    int rc = check_contraction(c);
    if (rc) return rc;
    if (res == 0) return fail(VMB_INVALID_ARGUMENT, "occupancy grid: resolution must be > 0");
    if (!(thr > 0.0 && thr < 1.0))
        return fail(VMB_INVALID_ARGUMENT, "occupancy grid: alpha_threshold must be in (0,1)");
    if (!(init >= 0.0))
        return fail(VMB_INVALID_ARGUMENT, "occupancy grid: initial density must be >= 0");
    cudaSetDevice(ctx->device);
    auto* g = new vmb_grid();
    g->device = ctx->device;
    g->res = res;
    g->con = *c;
    g->k = make_contract(*c);
    g->thr = thr;
    g->ref_step = ref_step > 0.0 ? ref_step : domain_diagonal(*c) / 1024.0;
    rc = grid_alloc(g);
    if (rc) {
        vmb_grid_destroy(g);
        return rc;
    }
    k_fill<<<grid_blocks(ctx, g->n_cells, 256), 256, 0, ctx->stream>>>(g->cache, g->n_cells, init);
    rc = grid_refresh(ctx, g);
    if (rc) {
        vmb_grid_destroy(g);
        return rc;
    }
    *out = g;
    return VMB_OK;
}

int vmb_grid_destroy(vmb_grid* g) {
    if (!g) return VMB_OK;
    cudaDeviceSynchronize();
    cudaFree(g->cache);
    cudaFree(g->bits);
    cudaFree(g->coarse);
    cudaFree(g->dist);
    cudaFree(g->dist_tmp);
    cudaFree(g->bbox);
    cudaFree(g->probed);
    delete g;
    return VMB_OK;
}

int vmb_grid_clone(vmb_ctx* ctx, const vmb_grid* src, vmb_grid** out) {
    auto* g = new vmb_grid();
    g->device = src->device;
    g->res = src->res;
    g->con = src->con;
    g->k = src->k;
    g->thr = src->thr;
    g->ref_step = src->ref_step;
    g->block = src->block;
    int rc = grid_alloc(g);
    if (rc) {
        vmb_grid_destroy(g);
        return rc;
    }
    cudaMemcpyAsync(g->cache, src->cache, g->n_cells * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(g->bits, src->bits, g->n_words * 4, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(g->coarse, src->coarse, g->coarse_words * 4, cudaMemcpyDeviceToDevice, ctx->stream);
    g->coarse_valid = src->coarse_valid;
    cudaMemcpyAsync(g->dist, src->dist, g->n_cells, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(g->bbox, src->bbox, 6 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream);
    rc = launch_check("grid clone");
    if (rc) {
        vmb_grid_destroy(g);
        return rc;
    }
    *out = g;
    return VMB_OK;
}

int vmb_grid_info(const vmb_grid* g, uint32_t* res, vmb_contraction* c, double* thr,
                  double* ref_step, double* thr_density) {
    if (res) *res = g->res;
    if (c) *c = g->con;
    if (thr) *thr = g->thr;
    if (ref_step) *ref_step = g->ref_step;
    if (thr_density) *thr_density = -std::log1p(-g->thr) / g->ref_step;  // occupancy_grid.cpp:63-65
    return VMB_OK;
}

int vmb_grid_update_field(vmb_ctx* ctx, vmb_grid* g, const vmb_field* f, const double* h_ts,
                          uint64_t n_ts, double decay, int has_seed, uint64_t seed) {
    Timestamps ts;
    int rc = make_timestamps(h_ts, n_ts, &ts);
    if (rc) return rc;
    if (!(decay >= 0.0 && decay <= 1.0))
        return fail(VMB_INVALID_ARGUMENT, "occupancy grid: ema_decay must be in [0,1]");
    if (int frc = check_field(f)) return frc;
    GridDev gd = dev_of(g);
    if (f->kind == VMB_FIELD_VOXEL || !(std::isfinite(f->sigma) && f->sigma >= 0.0)) {
        // Only analytic fields with an invalid sigma, or a voxel field (its
        // parameters may be non-finite), can fail; find the first bad probe
        // (timestamp-major, then cell order) before touching the cache.
        rc = reset_error(ctx);
        if (rc) return rc;
        (f->kind == VMB_FIELD_VOXEL ? k_update_errors<true> : k_update_errors<false>)<<<grid_blocks(ctx, g->n_cells, 256), 256, 0, ctx->stream>>>(
            gd, *f, ts, has_seed != 0, seed, ctx->d_err);
        DevError err;
        rc = read_error(ctx, &err);
        if (rc) return rc;
        if (err.key != ~0ull) return fail(VMB_RUNTIME, cell_name(g, err.key & ((1ull << 40) - 1)));
    }
    if (ctx->nccl_comm) {  // a communicator attached (any size): block probe + all-gather
        // rank k probes cells [k B, (k + 1) B), B = ceil(n / nranks), into their own
        // positions; the in-place all-gather gives every rank every block
        const uint64_t B = (g->n_cells + ctx->nranks - 1) / ctx->nranks;
        if (!g->probed || g->probed_words < B * ctx->nranks) {
            if (g->probed) cudaFree(g->probed);
            g->probed = nullptr;
            cudaError_t e = cudaMalloc(&g->probed, B * ctx->nranks * sizeof(double));
            if (e != cudaSuccess) return cuda_fail(e, "probe buffer");
            g->probed_words = B * ctx->nranks;
        }
        const uint64_t c0 = B * ctx->rank, c1 = std::min(g->n_cells, c0 + B);
        if (c1 > c0)
            (f->kind == VMB_FIELD_VOXEL ? k_probe_block<true> : k_probe_block<false>)<<<grid_blocks(ctx, c1 - c0, 256), 256, 0, ctx->stream>>>(
                gd, *f, ts, has_seed != 0, seed, c0, c1, g->probed);
        rc = launch_check("grid probe");
        if (rc) return rc;
        rc = vmb_comm_allgather_f64(ctx, g->probed, B);
        if (rc) return rc;
        k_apply<<<grid_blocks(ctx, g->n_words * 32, 256), 256, 0, ctx->stream>>>(
            gd, g->probed, decay, g->cache, g->bits, g->n_words);
    } else {
        launch_pdl(f->kind == VMB_FIELD_VOXEL ? k_update_fused<true> : k_update_fused<false>,
                   dim3(grid_blocks(ctx, g->n_words * 32, 256)), dim3(256), 0, ctx->stream, gd, *f, ts, has_seed != 0,
                   seed, decay, g->cache, g->bits, g->n_words);
    }
    rc = launch_check("grid update");
    return rc ? rc : grid_rebuild_coarse(ctx, g);
}

int vmb_grid_probe_field_range(vmb_ctx* ctx, const vmb_grid* g, const vmb_field* f,
                               const double* h_ts, uint64_t n_ts, int has_seed, uint64_t seed,
                               uint64_t c0, uint64_t c1, double* d_probed) {
    Timestamps ts;
    int rc = make_timestamps(h_ts, n_ts, &ts);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    if (c1 > g->n_cells) c1 = g->n_cells;
    (f->kind == VMB_FIELD_VOXEL ? k_probe_range<true> : k_probe_range<false>)<<<grid_blocks(ctx, g->n_cells, 256), 256, 0, ctx->stream>>>(
        dev_of(g), *f, ts, has_seed != 0, seed, c0, c1, d_probed);
    return launch_check("grid probe range");
}

int vmb_grid_probe_points(vmb_ctx* ctx, const vmb_grid* g, int has_seed, uint64_t seed,
                          double* d_points, uint32_t* d_cells, uint64_t* h_count) {
    uint64_t n = g->n_cells;
    char* tmp = static_cast<char*>(scratch(ctx, SCRATCH_GRID, n * (24 + 1 + 4) + 256));
    if (!tmp) return VMB_CUDA;
    auto* world = reinterpret_cast<double*>(tmp);
    auto* pos = reinterpret_cast<uint32_t*>(tmp + n * 24);
    auto* valid = reinterpret_cast<uint8_t*>(tmp + n * 28);
    int blocks = grid_blocks(ctx, n, 256);
    k_probe_points<<<blocks, 256, 0, ctx->stream>>>(dev_of(g), has_seed != 0, seed, world, valid);
    int rc = scan_flags(ctx, valid, n, pos, ctx->d_u64);
    if (rc) return rc;
    k_compact_points<<<blocks, 256, 0, ctx->stream>>>(n, world, valid, pos, d_points, d_cells);
    rc = launch_check("probe points");
    if (rc) return rc;
    cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "probe points");
    *h_count = ctx->h_u64[0];
    return VMB_OK;
}

int vmb_grid_accumulate(vmb_ctx* ctx, const vmb_grid* g, const double* dens, const uint32_t* cells,
                        uint64_t n, double* probed) {
    if (!n) return VMB_OK;
    int rc = reset_error(ctx);
    if (rc) return rc;
    k_accumulate<<<grid_blocks(ctx, n, 256), 256, 0, ctx->stream>>>(dens, cells, n, probed, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull) {
        uint32_t c;
        cudaMemcpy(&c, cells + err.key, 4, cudaMemcpyDeviceToHost);
        return fail(VMB_RUNTIME, cell_name(g, c));
    }
    return VMB_OK;
}

int vmb_grid_apply(vmb_ctx* ctx, vmb_grid* g, double* probed, double decay) {
    if (!(decay >= 0.0 && decay <= 1.0))
        return fail(VMB_INVALID_ARGUMENT, "occupancy grid: ema_decay must be in [0,1]");
    if (ctx->nccl_comm) {  // a communicator attached (any size): combine the ranks' probes
        int rc = vmb_comm_allreduce_max_f64(ctx, probed, g->n_cells);
        if (rc) return rc;
    }
    k_apply<<<grid_blocks(ctx, g->n_words * 32, 256), 256, 0, ctx->stream>>>(dev_of(g), probed, decay,
                                                                              g->cache, g->bits, g->n_words);
    int rc = launch_check("grid apply");
    return rc ? rc : grid_rebuild_coarse(ctx, g);
}

int vmb_grid_seed_mask(vmb_ctx* ctx, vmb_grid* g, const uint8_t* mask) {
    if (g->con.kind != VMB_CONTRACT_AABB)
        return fail(VMB_INVALID_ARGUMENT, "seed_occupancy: supported for AabbNormalize grids only");
    double high = 2.0 * (-std::log1p(-g->thr) / g->ref_step);
    k_seed_mask<<<grid_blocks(ctx, g->n_cells, 256), 256, 0, ctx->stream>>>(mask, g->n_cells, high, g->cache);
    int rc = launch_check("seed mask");
    return rc ? rc : grid_refresh(ctx, g);
}

int vmb_grid_occupied_count(vmb_ctx* ctx, const vmb_grid* g, uint64_t* count) {
    cudaMemsetAsync(ctx->d_u64, 0, 8, ctx->stream);
    k_popcount<<<grid_blocks(ctx, g->n_words, 256), 256, 0, ctx->stream>>>(g->bits, g->n_words, ctx->d_u64);
    cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "occupied count");
    *count = ctx->h_u64[0];
    return VMB_OK;
}

int vmb_grid_query(vmb_ctx* ctx, const vmb_grid* g, const double* pts, uint64_t n, uint8_t* out) {
    if (!n) return VMB_OK;
    int rc = reset_error(ctx);
    if (rc) return rc;
    k_query<<<grid_blocks(ctx, n, 256), 256, 0, ctx->stream>>>(dev_of(g), g->bits, pts, n, out, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull) return fail(VMB_INVALID_ARGUMENT, "non-finite coordinate");
    return VMB_OK;
}

int vmb_grid_read(vmb_ctx* ctx, const vmb_grid* g, uint8_t* h_bits, double* h_cache) {
    if (h_bits)
        cudaMemcpyAsync(h_bits, g->bits, (g->n_cells + 7) / 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (h_cache)
        cudaMemcpyAsync(h_cache, g->cache, g->n_cells * 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "grid read");
}

int vmb_grid_occupied_bbox(vmb_ctx* ctx, const vmb_grid* g, uint32_t* h_box) {
    cudaError_t e = cudaMemcpyAsync(h_box, g->bbox, 6 * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "grid bbox");
}

int vmb_grid_read_distance(vmb_ctx* ctx, const vmb_grid* g, uint8_t* h_dist, uint32_t* h_cap) {
    if (h_cap) *h_cap = uint32_t(kDistCap);
    if (h_dist) cudaMemcpyAsync(h_dist, g->dist, g->n_cells, cudaMemcpyDeviceToHost, ctx->stream);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "grid read distance");
}

int vmb_grid_write(vmb_ctx* ctx, vmb_grid* g, const uint8_t* h_bits, const double* h_cache) {
    if (h_bits) {
        cudaMemsetAsync(g->bits, 0, g->n_words * 4, ctx->stream);
        cudaMemcpyAsync(g->bits, h_bits, (g->n_cells + 7) / 8, cudaMemcpyHostToDevice, ctx->stream);
    }
    if (h_cache)
        cudaMemcpyAsync(g->cache, h_cache, g->n_cells * 8, cudaMemcpyHostToDevice, ctx->stream);
    int rc = launch_check("grid write");
    if (rc) return rc;
    rc = grid_rebuild_coarse(ctx, g);
    if (rc) return rc;
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "grid write");
}

const uint32_t* vmb_grid_device_bits(const vmb_grid* g) { return g->bits; }
const double* vmb_grid_device_cache(const vmb_grid* g) { return g->cache; }

}  // extern "C"
