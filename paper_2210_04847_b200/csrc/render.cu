// render.cu — differentiable compositing along rays (rendering.cpp:19-134).
//
// Layout: packed samples are ray-contiguous (offsets = exclusive scan of counts),
// so the samples of 32 consecutive rays form one contiguous range. Each warp owns
// 32 rays and streams their range through its shared-memory tile:
//   1. cp.async (LDGSTS) copies t_starts/t_ends (f64), sigma and rgb (AoS) of up to
//      CH samples into the tile — every element in flight at once, no registers;
//   2. alpha = 1 - exp(-sigma * delta) is computed sample-parallel (all lanes,
//      independent exps), so the per-ray loops below never wait on an exp;
//   3. each lane runs its own ray's recurrence sequentially from shared memory in
//      the reference's operation order and in fp64 (T *= 1 - alpha; fp32 is not
//      accurate enough);
//   4. per-sample outputs are staged back into the tile and written coalesced.
// render_backward groups consecutive rays whose samples fit one tile. Within a
// group (k_backward_hy) only the two true recurrences run lane-serially: the
// forward transmittance (one dependent multiply per sample) and the reverse
// suffix sum (one dependent add per sample); everything else — alpha, v, the
// weights, d_rgb — runs sample-parallel over the tile with every lane busy.
// Only a single ray longer than a tile uses two forward sweeps with
// suffix_k = S - P_k. Warps whose rays
// are not contiguous (arbitrary user offsets) use per-lane global reads.
// Sample positions are 32-bit: packed offsets are u32 by construction (pack()
// rejects more than 2^32-1 samples, core_types.cpp:33-36).
#include <type_traits>

#include "vm_internal.h"
#include "vm_bulk.cuh"

namespace vmb {
namespace {

#ifndef VMB_RENDER_WARPS
#define VMB_RENDER_WARPS 4  // r2 (config 5 step, with 8 CTAs/SM): 4 warps 0.694 ms, 8 warps 0.707
#endif
constexpr int kWarps = VMB_RENDER_WARPS;  // threads per CTA / 32

template <typename T> struct Tile;
#ifndef VMB_TILE_F32
#define VMB_TILE_F32 128  // r2 A/B: 192 and 256 slower (config 5 0.706 / 0.796 ms), config 2 no better
#endif
template <> struct Tile<float> { static constexpr int CH = VMB_TILE_F32; };
template <> struct Tile<double> { static constexpr int CH = 64; };

template <typename T>
struct FwdSmem {
    double ts[Tile<T>::CH];
    double te[Tile<T>::CH];
    double al[Tile<T>::CH];   // alpha (or exp(-sigma*delta) for the transmittance)
    T rgb[3 * Tile<T>::CH];
    T sig[Tile<T>::CH];
};

// PAD (k_backward_hy, dynamic shared memory): room for a bulk copy that starts at
// the 16-byte boundary at or below a group's first sample and ends at the one at or
// above its last, and the copies' mbarrier
struct BulkBar {
    unsigned long long bar;   // the bulk copies' mbarrier
};
struct NoBar {};
template <typename T, int PAD = 0>
struct BwdSmem : std::conditional_t<(PAD > 0), BulkBar, NoBar> {
    alignas(16) double ts[Tile<T>::CH + PAD];
    alignas(16) double te[Tile<T>::CH + PAD];
    double al[Tile<T>::CH];
    double tr[Tile<T>::CH];   // transmittance before each sample
    alignas(16) T rgb[3 * Tile<T>::CH + PAD];   // input rgb, then d_rgb
    alignas(16) T sig[Tile<T>::CH + PAD];       // input sigma, then d_sigma
};
constexpr int kBulkPad = 8;

struct RayRange {
    uint64_t r;
    bool valid;
    uint32_t off, end;
    bool contiguous;  // warp-uniform
    uint32_t s0, s1;  // warp range when contiguous
};

__device__ __forceinline__ RayRange ray_range(const uint32_t* __restrict__ offsets,
                                              const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
                                              uint64_t warp_id, int lane) {
    RayRange rr;
    rr.r = warp_id * 32 + lane;
    rr.valid = rr.r < n_rays;
    // samples at or beyond n_samples (the buffers' length) are ignored: a ray range
    // is clamped into [0, n_samples), which keeps the ranges contiguous
    const uint64_t ns = n_samples < 0xffffffffull ? n_samples : 0xffffffffull;
    const uint64_t o64 = rr.valid ? __ldg(offsets + rr.r) : 0u;
    const uint64_t e64 = rr.valid ? o64 + __ldg(counts + rr.r) : 0u;
    rr.off = uint32_t(o64 < ns ? o64 : ns);
    rr.end = uint32_t(e64 < ns ? e64 : ns);
    const uint32_t next_off = __shfl_down_sync(0xffffffffu, rr.off, 1);
    const bool next_valid = __shfl_down_sync(0xffffffffu, int(rr.valid), 1);
    const bool ok = !(rr.valid && lane < 31 && next_valid) || rr.end == next_off;
    rr.contiguous = __all_sync(0xffffffffu, ok);
    rr.s0 = __shfl_sync(0xffffffffu, rr.off, 0);
    const unsigned vmask = __ballot_sync(0xffffffffu, rr.valid);
    rr.s1 = __shfl_sync(0xffffffffu, rr.end, vmask ? 31 - __clz(vmask) : 0);
    return rr;
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES)
                 : "memory");
}

// Stage samples [cs, cs+n) into a tile and compute alpha (kTransmittance: the
// factor exp(-sigma*delta) of rendering.cpp:29 instead) for each of them.
template <typename T, bool kTransmittance, typename S>
__device__ __forceinline__ void stage_in(S& sm, int lane, uint32_t cs, uint32_t n,
                                         const double* __restrict__ ts, const double* __restrict__ te,
                                         const T* __restrict__ rgb, const T* __restrict__ sig) {
    // fully unrolled rounds of 32 (n <= CH): per-lane base pointers + constant
    // offsets, no loop-carried address arithmetic
    constexpr int R = Tile<T>::CH / 32;
    const double* pts = ts + cs + lane;
    const double* pte = te + cs + lane;
    const T* psg = sig + cs + lane;
#pragma unroll
    for (int k = 0; k < R; ++k)
        if (32u * k + lane < n) {
            cp_async<8>(&sm.ts[32 * k + lane], pts + 32 * k);
            cp_async<8>(&sm.te[32 * k + lane], pte + 32 * k);
            cp_async<sizeof(T)>(&sm.sig[32 * k + lane], psg + 32 * k);
        }
    if (rgb) {
        const T* prgb = rgb + 3 * uint64_t(cs) + lane;
#pragma unroll
        for (int k = 0; k < 3 * R; ++k)
            if (32u * k + lane < 3 * n) cp_async<sizeof(T)>(&sm.rgb[32 * k + lane], prgb + 32 * k);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const uint32_t i = 32u * k + lane;
        if (i < n) {
            double e = exp(-double(sm.sig[i]) * (sm.te[i] - sm.ts[i]));
            sm.al[i] = kTransmittance ? e : 1.0 - e;
        }
    }
    __syncwarp();
}

// k_backward_hy's staging by the bulk-copy engine: lane 0 issues one
// cp.async.bulk per array (t_starts, t_ends, sigma, rgb) of the group's samples
// [cs, cs + n), each from the 16-byte boundary at or below its first byte to the one
// at or above its end, completed on the warp's mbarrier; the group's sample i then
// sits at index i + shift of the array's tile (TileView). Returns false (nothing
// issued) when a pointer is not 16-byte aligned or a rounded span would pass
// n_samples: the caller stages that group with stage_in.
template <typename T>
struct TileView {
    double* ts;
    double* te;
    T* rgb;
    T* sig;
};
template <typename T>
__device__ __forceinline__ bool stage_bulk(BwdSmem<T, kBulkPad>& sm, int lane, uint32_t cs, uint32_t n, uint64_t n_samples,
                                           const double* __restrict__ ts, const double* __restrict__ te,
                                           const T* __restrict__ rgb, const T* __restrict__ sig, uint32_t& phase,
                                           TileView<T>& v) {
#ifndef VMB_BWD_BULK
#define VMB_BWD_BULK 1
#endif
    if (!VMB_BWD_BULK) return false;
    const uint64_t a_t0 = reinterpret_cast<uint64_t>(ts), a_t1 = reinterpret_cast<uint64_t>(te);
    const uint64_t a_c = reinterpret_cast<uint64_t>(rgb), a_s = reinterpret_cast<uint64_t>(sig);
    if (((a_t0 | a_t1 | a_c | a_s) & 15u) != 0u) return false;
    // byte spans [lo, hi) relative to each array, 16-byte aligned
    const uint64_t t_lo = (8ull * cs) & ~15ull, t_hi = (8ull * (cs + n) + 15ull) & ~15ull;
    const uint64_t c_lo = (3ull * sizeof(T) * cs) & ~15ull, c_hi = (3ull * sizeof(T) * (cs + n) + 15ull) & ~15ull;
    const uint64_t s_lo = (uint64_t(sizeof(T)) * cs) & ~15ull, s_hi = (uint64_t(sizeof(T)) * (cs + n) + 15ull) & ~15ull;
    if (t_hi > 8ull * n_samples || c_hi > 3ull * sizeof(T) * n_samples || s_hi > uint64_t(sizeof(T)) * n_samples)
        return false;
    __syncwarp();  // every lane's accesses of the tile so far precede the copies
    if (lane == 0) {
        fence_proxy_async();
        mbar_expect(&sm.bar, uint32_t(2 * (t_hi - t_lo) + (c_hi - c_lo) + (s_hi - s_lo)));
        bulk_g2s(sm.ts, reinterpret_cast<const char*>(ts) + t_lo, uint32_t(t_hi - t_lo), &sm.bar);
        bulk_g2s(sm.te, reinterpret_cast<const char*>(te) + t_lo, uint32_t(t_hi - t_lo), &sm.bar);
        bulk_g2s(sm.rgb, reinterpret_cast<const char*>(rgb) + c_lo, uint32_t(c_hi - c_lo), &sm.bar);
        bulk_g2s(sm.sig, reinterpret_cast<const char*>(sig) + s_lo, uint32_t(s_hi - s_lo), &sm.bar);
    }
    v.ts = sm.ts + (8ull * cs - t_lo) / 8;
    v.te = sm.te + (8ull * cs - t_lo) / 8;
    v.rgb = sm.rgb + (3ull * sizeof(T) * cs - c_lo) / sizeof(T);
    v.sig = sm.sig + (uint64_t(sizeof(T)) * cs - s_lo) / sizeof(T);
    mbar_wait(&sm.bar, phase);
    phase ^= 1u;
    return true;
}

// ------------------------------------------------------------------ forward
struct Fwd {
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, op = 0.0, dep = 0.0;
    // rendering.cpp:51-58 (alpha precomputed with the same expression)
    __device__ __forceinline__ void add(double ts, double te, double r, double g, double b,
                                        double alpha) {
        double w = T * alpha;
        cr = cr + r * w;
        cg = cg + g * w;
        cb = cb + b * w;
        op += w;
        dep += w * 0.5 * (ts + te);
        T *= 1.0 - alpha;
    }
};

#ifndef VMB_FWD_LANE_AVG
#define VMB_FWD_LANE_AVG 16
#endif
constexpr uint32_t kFwdLaneAvg = VMB_FWD_LANE_AVG;

template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 24 / kWarps) k_forward(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ rgb,
    const T* __restrict__ sig, T* __restrict__ color, T* __restrict__ opacity, T* __restrict__ depth) {
    __shared__ FwdSmem<T> smem[kWarps];
    const int lane = threadIdx.x & 31;
    FwdSmem<T>& sm = smem[threadIdx.x >> 5];
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const RayRange rr = ray_range(offsets, counts, n_rays, n_samples, w, lane);
        Fwd acc;
        // Long rays (more than kFwdLaneAvg samples per ray on average, e.g. growth
        // lattices): one tile then holds the samples of one or two rays, so the
        // tile loop would run on one lane in 32; each lane streams its own ray
        // from global memory instead (same expressions, same order).
        if (rr.contiguous && rr.s1 - rr.s0 <= 32u * kFwdLaneAvg) {
            for (uint32_t cs = rr.s0; cs < rr.s1; cs += Tile<T>::CH) {
                const uint32_t n = min(uint32_t(Tile<T>::CH), rr.s1 - cs);
                stage_in<T, false>(sm, lane, cs, n, ts, te, rgb, sig);
                const uint32_t a = max(rr.off, cs), b = min(rr.end, cs + n);
                for (uint32_t s = a; s < b; ++s) {
                    const uint32_t i = s - cs;
                    acc.add(sm.ts[i], sm.te[i], double(sm.rgb[3 * i]), double(sm.rgb[3 * i + 1]),
                            double(sm.rgb[3 * i + 2]), sm.al[i]);
                }
                __syncwarp();
            }
        } else {
#pragma unroll 4
            for (uint32_t s = rr.off; s < rr.end; ++s)
                acc.add(ts[s], te[s], double(rgb[3 * uint64_t(s)]), double(rgb[3 * uint64_t(s) + 1]),
                        double(rgb[3 * uint64_t(s) + 2]), 1.0 - exp(-double(sig[s]) * (te[s] - ts[s])));
        }
        if (rr.valid) {
            color[3 * rr.r] = T(acc.cr);
            color[3 * rr.r + 1] = T(acc.cg);
            color[3 * rr.r + 2] = T(acc.cb);
            opacity[rr.r] = T(acc.op);
            depth[rr.r] = T(acc.dep);
        }
    }
}

// render_forward for long rays (render_forward picks it when the batch averages
// more than kFwdLaneAvg samples per ray, e.g. growth lattices): one lane per ray,
// every lane active, and the samples reach shared memory coalesced: the warp
// stages a window of the next W samples of each of its 32 rays (32 / W rays per
// load instruction, W = 16 consecutive samples each for f32 attributes, 8 for f64) into a [sample][ray] tile, then
// each lane composites its own ray's window from it (rendering.cpp:47-58, the
// tile kernel's expressions in the same order: bit-identical).
constexpr int kWinWarps = 2, kWinPad = 33;
#ifndef VMB_WIN_W32
#define VMB_WIN_W32 16
#endif
template <typename T> struct Win { static constexpr int W = sizeof(T) == 4 ? VMB_WIN_W32 : 8; };

template <typename T>
struct WinSmem {
    static constexpr int kWinW = Win<T>::W;
    double ts[kWinW][kWinPad];
    double te[kWinW][kWinPad];
    T r[kWinW][kWinPad], g[kWinW][kWinPad], b[kWinW][kWinPad], sig[kWinW][kWinPad];
};

template <typename T>
__global__ void __launch_bounds__(kWinWarps * 32) k_forward_win(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ rgb,
    const T* __restrict__ sig, T* __restrict__ color, T* __restrict__ opacity, T* __restrict__ depth) {
    __shared__ WinSmem<T> smem[kWinWarps];
    const int lane = threadIdx.x & 31;
    constexpr int kWinW = Win<T>::W, kRq = 32 / kWinW;  // rays per load instruction
    const int half = lane / kWinW, j = lane % kWinW;
    WinSmem<T>& sm = smem[threadIdx.x >> 5];
    const uint64_t ns = n_samples < 0xffffffffull ? n_samples : 0xffffffffull;
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t r = w * 32 + lane;
        const bool valid = r < n_rays;
        const uint64_t o64 = valid ? __ldg(offsets + r) : 0u;
        const uint64_t e64 = valid ? o64 + __ldg(counts + r) : 0u;
        uint32_t pos = uint32_t(o64 < ns ? o64 : ns);
        const uint32_t end = uint32_t(e64 < ns ? e64 : ns);
        Fwd acc;
        while (__any_sync(0xffffffffu, pos < end)) {
#pragma unroll 4
            for (int q0 = 0; q0 < 32; q0 += kRq) {
                const int q = q0 + half;
                const uint32_t p = __shfl_sync(0xffffffffu, pos, q);
                const uint32_t e = __shfl_sync(0xffffffffu, end, q);
                if (p + uint32_t(j) < e) {
                    const uint64_t x = uint64_t(p) + j;
                    cp_async<8>(&sm.ts[j][q], ts + x);
                    cp_async<8>(&sm.te[j][q], te + x);
                    cp_async<sizeof(T)>(&sm.sig[j][q], sig + x);
                    cp_async<sizeof(T)>(&sm.r[j][q], rgb + 3 * x);
                    cp_async<sizeof(T)>(&sm.g[j][q], rgb + 3 * x + 1);
                    cp_async<sizeof(T)>(&sm.b[j][q], rgb + 3 * x + 2);
                }
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncwarp();
            const uint32_t n = pos < end ? min(uint32_t(kWinW), end - pos) : 0u;
            for (uint32_t i = 0; i < n; ++i) {
                const double t0 = sm.ts[i][lane], t1 = sm.te[i][lane];
                const double e = exp(-double(sm.sig[i][lane]) * (t1 - t0));
                acc.add(t0, t1, double(sm.r[i][lane]), double(sm.g[i][lane]), double(sm.b[i][lane]), 1.0 - e);
            }
            pos += n;
            __syncwarp();
        }
        if (valid) {
            color[3 * r] = T(acc.cr);
            color[3 * r + 1] = T(acc.cg);
            color[3 * r + 2] = T(acc.cb);
            opacity[r] = T(acc.op);
            depth[r] = T(acc.dep);
        }
    }
}

// march_render for long-ray batches on the two-pass march path (growth lattices):
// k_shade and k_forward_win in one pass. Each lane keeps its ray's origin and
// direction, stages windows of t0/t1 coalesced, shades every sample of its ray
// at the midpoint (k_shade's expressions: voxmarch.cpp:243-244), composites it
// (rendering.cpp:47-58) and the window's rgb/sigma go out coalesced per ray.
// Bit-identical to k_shade -> render_forward; t0/t1/ray_indices are read once
// instead of twice and rgb/sigma are never re-read.
template <typename RT, typename T, bool VOX>
__global__ void __launch_bounds__(kWinWarps * 32) k_shade_forward_win(
    const RT* __restrict__ orig, const RT* __restrict__ dirs, vmb_field f, double time,
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, T* __restrict__ rgb, T* __restrict__ sig,
    T* __restrict__ color, T* __restrict__ opacity, T* __restrict__ depth) {
    __shared__ WinSmem<T> smem[kWinWarps];
    griddep_wait();
    const int lane = threadIdx.x & 31;
    constexpr int kWinW = Win<T>::W, kRq = 32 / kWinW;
    const int half = lane / kWinW, j = lane % kWinW;
    WinSmem<T>& sm = smem[threadIdx.x >> 5];
    const uint64_t ns = n_samples < 0xffffffffull ? n_samples : 0xffffffffull;
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t r = w * 32 + lane;
        const bool valid = r < n_rays;
        const uint64_t o64 = valid ? __ldg(offsets + r) : 0u;
        const uint64_t e64 = valid ? o64 + __ldg(counts + r) : 0u;
        uint32_t pos = uint32_t(o64 < ns ? o64 : ns);
        const uint32_t end = uint32_t(e64 < ns ? e64 : ns);
        const uint64_t rr = valid ? r : 0;
        const D3 o = d3(double(orig[3 * rr]), double(orig[3 * rr + 1]), double(orig[3 * rr + 2]));
        const D3 d = d3(double(dirs[3 * rr]), double(dirs[3 * rr + 1]), double(dirs[3 * rr + 2]));
        Fwd acc;
        while (__any_sync(0xffffffffu, pos < end)) {
#pragma unroll 4
            for (int q0 = 0; q0 < 32; q0 += kRq) {
                const int q = q0 + half;
                const uint32_t p = __shfl_sync(0xffffffffu, pos, q);
                const uint32_t e = __shfl_sync(0xffffffffu, end, q);
                if (p + uint32_t(j) < e) {
                    const uint64_t x = uint64_t(p) + j;
                    cp_async<8>(&sm.ts[j][q], ts + x);
                    cp_async<8>(&sm.te[j][q], te + x);
                }
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncwarp();
            const uint32_t m = pos < end ? min(uint32_t(kWinW), end - pos) : 0u;
            for (uint32_t i = 0; i < m; ++i) {
                const double t0 = sm.ts[i][lane], t1 = sm.te[i][lane];
                const D3 x = o + d * (0.5 * (t0 + t1));
                D3 c;
                const double sigma = field_rgb_sigma_t<VOX>(f, time_shift(f, x, time), &c);
                const T cr = T(c.x), cg = T(c.y), cb = T(c.z), sg = T(sigma);
                sm.r[i][lane] = cr;
                sm.g[i][lane] = cg;
                sm.b[i][lane] = cb;
                sm.sig[i][lane] = sg;
                const double ex = exp(-double(sg) * (t1 - t0));
                acc.add(t0, t1, double(cr), double(cg), double(cb), 1.0 - ex);
            }
            __syncwarp();
#pragma unroll 4
            for (int q0 = 0; q0 < 32; q0 += kRq) {
                const int q = q0 + half;
                const uint32_t p = __shfl_sync(0xffffffffu, pos, q);
                const uint32_t e = __shfl_sync(0xffffffffu, end, q);
                if (p + uint32_t(j) < e) {
                    const uint64_t x = uint64_t(p) + j;
                    sig[x] = sm.sig[j][q];
                    rgb[3 * x] = sm.r[j][q];
                    rgb[3 * x + 1] = sm.g[j][q];
                    rgb[3 * x + 2] = sm.b[j][q];
                }
            }
            __syncwarp();
            pos += m;
        }
        if (valid) {
            color[3 * r] = T(acc.cr);
            color[3 * r + 1] = T(acc.cg);
            color[3 * r + 2] = T(acc.cb);
            opacity[r] = T(acc.op);
            depth[r] = T(acc.dep);
        }
    }
}

// ------------------------------------------------------------------ backward
struct Up {
    double dcx, dcy, dcz, dop, ddep;
    // v = dot(d_color, rgb) + d_opacity + d_depth * mid   (rendering.cpp:102)
    __device__ __forceinline__ double value(double r, double g, double b, double mid) const {
        return (dcx * r + dcy * g + dcz * b) + dop + ddep * mid;
    }
};

template <typename T>
__device__ __forceinline__ Up load_up(const T* dc, const T* dop, const T* ddep, uint64_t r, bool valid) {
    Up u{0, 0, 0, 0, 0};
    if (valid) {
        u.dcx = double(dc[3 * r]);
        u.dcy = double(dc[3 * r + 1]);
        u.dcz = double(dc[3 * r + 2]);
        u.dop = double(dop[r]);
        u.ddep = double(ddep[r]);
    }
    return u;
}

template <typename T, typename S>
__device__ __forceinline__ void write_out(S& sm, int lane, uint32_t cs, uint32_t n,
                                          T* __restrict__ g_rgb, T* __restrict__ g_sig) {
    constexpr int R = Tile<T>::CH / 32;
    __syncwarp();
    T* psg = g_sig + cs + lane;
    T* prgb = g_rgb + 3 * uint64_t(cs) + lane;
#pragma unroll
    for (int k = 0; k < R; ++k)
        if (32u * k + lane < n) psg[32 * k] = sm.sig[32 * k + lane];
#pragma unroll
    for (int k = 0; k < 3 * R; ++k)
        if (32u * k + lane < 3 * n) prgb[32 * k] = sm.rgb[32 * k + lane];
    __syncwarp();
}

// One ray [s0, s1) by the whole warp (a ray longer than a tile, or a ray of a warp
// whose rays are not stored contiguously), rendering.cpp:85-108 with the
// reference's directions: T by a product scan over the lanes carried forward
// across rounds and tiles, and the suffix of w v accumulated from the ray's END —
// a reverse sum scan carried backwards across rounds and tiles — so the tail
// gradients never come from a difference of two large sums. A forward sweep over
// the tiles stores the transmittance carried into each tile (kCarryTiles per
// super-block; longer rays repeat it per super-block), then the tiles are
// processed last to first. Per sample the same expressions as the reference, up
// to the association order of the scans' products and sums.
constexpr int kCarryTiles = 32;  // one per lane: lane k holds the T carried into tile sb_start + k

template <typename T, typename S>
__device__ void bwd_long_ray(S& sm, int lane, uint32_t s0, uint32_t s1, const Up& u,
                             const double* __restrict__ ts, const double* __restrict__ te,
                             const T* __restrict__ rgb, const T* __restrict__ sig,
                             T* __restrict__ g_rgb, T* __restrict__ g_sig) {
    constexpr uint32_t CH = Tile<T>::CH;
    const uint32_t nt = (s1 - s0 + CH - 1) / CH;
    double carryS = 0.0;  // sum of w v over the samples after the current round
    for (uint32_t sb_end = nt; sb_end > 0;) {
        const uint32_t sb_start = sb_end > uint32_t(kCarryTiles) ? sb_end - kCarryTiles : 0u;
        // forward sweep: T carried into every tile of the super-block (the last tile's
        // own product is never needed: a ray within one tile has no forward sweep)
        double carryT = 1.0, my_carry = 1.0;
        for (uint32_t t = 0; t + 1 < sb_end; ++t) {
            if (t >= sb_start && uint32_t(lane) == t - sb_start) my_carry = carryT;
            const uint32_t cs = s0 + t * CH, n = min(CH, s1 - cs);
            stage_in<T, false>(sm, lane, cs, n, ts, te, static_cast<const T*>(nullptr), sig);
            for (uint32_t r0 = 0; r0 < n; r0 += 32) {
                double x = r0 + lane < n ? 1.0 - sm.al[r0 + lane] : 1.0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) x *= __shfl_xor_sync(0xffffffffu, x, d);
                carryT *= x;
            }
            __syncwarp();
        }
        if (uint32_t(lane) == sb_end - 1 - sb_start) my_carry = carryT;
        __syncwarp();
        for (uint32_t t = sb_end; t-- > sb_start;) {
            const uint32_t cs = s0 + t * CH, n = min(CH, s1 - cs);
            stage_in<T, false>(sm, lane, cs, n, ts, te, rgb, sig);
            double cT = __shfl_sync(0xffffffffu, my_carry, int(t - sb_start));
            for (uint32_t r0 = 0; r0 < n; r0 += 32) {  // T before each sample of the tile
                const uint32_t i = r0 + uint32_t(lane);
                double x = i < n ? 1.0 - sm.al[i] : 1.0;  // inclusive product of (1 - alpha)
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double y = __shfl_up_sync(0xffffffffu, x, d);
                    if (lane >= d) x *= y;
                }
                double tr = __shfl_up_sync(0xffffffffu, x, 1);
                tr = (lane == 0 ? 1.0 : tr) * cT;
                cT *= __shfl_sync(0xffffffffu, x, 31);
                if (i < n) sm.tr[i] = tr;
            }
            __syncwarp();
            for (uint32_t r0 = (n - 1) / 32 * 32 + 32; r0 > 0;) {  // rounds last to first
                r0 -= 32;
                const uint32_t i = r0 + uint32_t(lane);
                const bool in = i < n;
                double t0 = 0.0, t1 = 0.0, a = 0.0, tr = 0.0, v = 0.0;
                if (in) {
                    t0 = sm.ts[i], t1 = sm.te[i], a = sm.al[i], tr = sm.tr[i];
                    v = u.value(double(sm.rgb[3 * i]), double(sm.rgb[3 * i + 1]), double(sm.rgb[3 * i + 2]),
                                0.5 * (t0 + t1));
                }
                const double wgt = tr * a;
                const double x = in ? wgt * v : 0.0;
                double incl = x;  // sum of x over this lane and the later ones
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const double y = __shfl_down_sync(0xffffffffu, incl, d);
                    if (lane + d < 32) incl += y;
                }
                double later = __shfl_down_sync(0xffffffffu, incl, 1);
                if (lane == 31) later = 0.0;
                const double suffix = later + carryS;
                carryS += __shfl_sync(0xffffffffu, incl, 0);
                if (in) {
                    sm.rgb[3 * i] = T(u.dcx * wgt);
                    sm.rgb[3 * i + 1] = T(u.dcy * wgt);
                    sm.rgb[3 * i + 2] = T(u.dcz * wgt);
                    sm.sig[i] = T((t1 - t0) * (tr * (1.0 - a) * v - suffix));
                }
            }
            write_out<T>(sm, lane, cs, n, g_rgb, g_sig);
        }
        sb_end = sb_start;
    }
}

// The rays k_backward_hy set aside (longer than a tile), one warp each.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 32 / kWarps) k_backward_long(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ rgb,
    const T* __restrict__ sig, const T* __restrict__ dc, const T* __restrict__ dop,
    const T* __restrict__ ddep, T* __restrict__ g_rgb, T* __restrict__ g_sig,
    const uint32_t* __restrict__ long_rays, const unsigned int* __restrict__ n_long) {
    __shared__ BwdSmem<T> smem[kWarps];
    griddep_wait();
    const int lane = threadIdx.x & 31;
    BwdSmem<T>& sm = smem[threadIdx.x >> 5];
    const unsigned int n = *n_long;
    const uint64_t ns = n_samples < 0xffffffffull ? n_samples : 0xffffffffull;
    const uint64_t stride = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    // Software pipeline over the warp's rays: the next ray's offset, count and upstream
    // gradients, and the index of the one after, are in flight while a ray is processed
    // (its chain was list -> offsets -> samples, three dependent global round trips).
    uint64_t k = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    struct Meta {
        uint32_t o = 0, c = 0;
        T u[5] = {};
    };
    auto ray_at = [&](uint64_t q) { return q < n ? __ldg(long_rays + q) : 0u; };
    auto fetch = [&](uint64_t q, uint32_t r, Meta& m) {
        if (q >= n) return;
        m.o = __ldg(offsets + r), m.c = __ldg(counts + r);
        m.u[0] = dc[3 * uint64_t(r)], m.u[1] = dc[3 * uint64_t(r) + 1], m.u[2] = dc[3 * uint64_t(r) + 2];
        m.u[3] = dop[r], m.u[4] = ddep[r];
    };
    Meta cur;
    fetch(k, ray_at(k), cur);
    uint32_t r_next = ray_at(k + stride);
    for (; k < n; k += stride) {
        const uint32_t r_after = ray_at(k + 2 * stride);
        Meta nxt;
        fetch(k + stride, r_next, nxt);
        const uint64_t o = cur.o, e = o + cur.c;
        const Up u{double(cur.u[0]), double(cur.u[1]), double(cur.u[2]), double(cur.u[3]), double(cur.u[4])};
        bwd_long_ray(sm, lane, uint32_t(o < ns ? o : ns), uint32_t(e < ns ? e : ns), u,
                     ts, te, rgb, sig, g_rgb, g_sig);
        cur = nxt;
        r_next = r_after;
    }
}

// render_backward: greedy groups of consecutive rays whose samples fit one tile;
// each group is staged once and every lane runs the reference's exact forward-T /
// reverse-suffix recurrence (rendering.cpp:85-108) from shared memory.
#ifndef VMB_BWD_MINB
#define VMB_BWD_MINB 8
#endif


template <typename T>
__global__ void __launch_bounds__(kWarps * 32, VMB_BWD_MINB) k_backward_hy(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ rgb,
    const T* __restrict__ sig, const T* __restrict__ dc, const T* __restrict__ dop,
    const T* __restrict__ ddep, T* __restrict__ g_rgb, T* __restrict__ g_sig,
    uint32_t* __restrict__ long_rays, unsigned int* __restrict__ n_long) {
    extern __shared__ __align__(16) unsigned char bwd_dyn_smem[];  // kWarps x BwdSmem<T, kBulkPad>
    griddep_wait();
    const int lane = threadIdx.x & 31;
    BwdSmem<T, kBulkPad>& sm = reinterpret_cast<BwdSmem<T, kBulkPad>*>(bwd_dyn_smem)[threadIdx.x >> 5];
    if (lane == 0) {
        mbar_init(&sm.bar);
        mbar_fence_init();
    }
    __syncwarp();
    uint32_t bphase = 0u;  // parity of the bulk-copy barrier's next phase
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const RayRange rr = ray_range(offsets, counts, n_rays, n_samples, w, lane);
        if (rr.contiguous && rr.s0 == rr.s1) continue;  // no sample in the chunk (half of config 5's)
        const Up u = load_up(dc, dop, ddep, rr.r, rr.valid);
        if (!rr.contiguous) {  // rays not stored one after the other: each by the whole warp
            for (int q = 0; q < 32; ++q) {
                const uint32_t a = __shfl_sync(0xffffffffu, rr.off, q), b = __shfl_sync(0xffffffffu, rr.end, q);
                const Up uq{__shfl_sync(0xffffffffu, u.dcx, q), __shfl_sync(0xffffffffu, u.dcy, q),
                            __shfl_sync(0xffffffffu, u.dcz, q), __shfl_sync(0xffffffffu, u.dop, q),
                            __shfl_sync(0xffffffffu, u.ddep, q)};
                if (__shfl_sync(0xffffffffu, int(rr.valid), q) && a < b)
                    bwd_long_ray<T>(sm, lane, a, b, uq, ts, te, rgb, sig, g_rgb, g_sig);
            }
            continue;
        }
        const unsigned vmask = __ballot_sync(0xffffffffu, rr.valid);  // valid lanes: a prefix
        // Rays longer than half a tile go to k_backward_long (one warp per ray, lane
        // scans): a group holding one or two such rays would run its recurrences on
        // one or two lanes (the cascade's ~120-sample rays). One list append per warp.
#ifndef VMB_BWD_SERIAL_DIV
#define VMB_BWD_SERIAL_DIV 2  // rays above CH / this go to k_backward_long (config 2, 27-sample rays: /2 0.211 ms, /4 0.210, /8 0.237)
#endif
        const unsigned lm =
            __ballot_sync(0xffffffffu, rr.valid && rr.end - rr.off > uint32_t(Tile<T>::CH / VMB_BWD_SERIAL_DIV));
        {
            if (lm) {
                unsigned at = 0;
                if (lane == 0) at = atomicAdd(n_long, unsigned(__popc(lm)));
                at = __shfl_sync(0xffffffffu, at, 0);
                if ((lm >> lane) & 1u)
                    long_rays[at + __popc(lm & ((1u << lane) - 1u))] = uint32_t(rr.r);
            }
        }
        int g0 = 0;
        while (g0 < 32 && ((vmask >> g0) & 1u)) {
            const uint32_t base = __shfl_sync(0xffffffffu, rr.off, g0);
            if ((lm >> g0) & 1u) {  // ray g0 is listed for k_backward_long
                ++g0;
                continue;
            }
            const bool fits = rr.valid && lane >= g0 && rr.end - base <= uint32_t(Tile<T>::CH);
            const unsigned fm = __ballot_sync(0xffffffffu, fits);  // monotone: ends ascend
            // the group: from g0 while the rays fit the tile, up to the next listed ray
            const unsigned later_long = lm & ~((2u << g0) - 1u);
            const int g1 = min(31 - __clz(fm), later_long ? __ffs(later_long) - 2 : 31);
            const uint32_t n = __shfl_sync(0xffffffffu, rr.end, g1) - base;
            if (n) {
                TileView<T> tv;
                if (stage_bulk(sm, lane, base, n, n_samples, ts, te, rgb, sig, bphase, tv)) {
#pragma unroll
                    for (int k = 0; k < Tile<T>::CH / 32; ++k) {
                        const uint32_t i = 32u * k + lane;
                        if (i < n) sm.al[i] = 1.0 - exp(-double(tv.sig[i]) * (tv.te[i] - tv.ts[i]));
                    }
                    __syncwarp();
                } else {
                    stage_in<T, false>(sm, lane, base, n, ts, te, rgb, sig);
                    tv = TileView<T>{sm.ts, sm.te, sm.rgb, sm.sig};
                }
                // owner lane of each staged sample: bytes of the sigma tile, free
                // between the alpha phase and phase D (which writes d_sigma there)
                uint8_t* own = reinterpret_cast<uint8_t*>(tv.sig);
                // B (lane-serial): T before each sample, rendering.cpp:89-96 — one
                // dependent DMUL per sample; the owner map for the parallel phase
                if (lane >= g0 && lane <= g1) {
                    double t = 1.0;
                    uint32_t i = rr.off - base;
                    const uint32_t e = rr.end - base;
                    for (; i + 4 <= e; i += 4) {  // the 4 loads issue before the chain
                        const double f0 = 1.0 - sm.al[i], f1 = 1.0 - sm.al[i + 1];
                        const double f2 = 1.0 - sm.al[i + 2], f3 = 1.0 - sm.al[i + 3];
                        sm.tr[i] = t;
                        t *= f0;
                        sm.tr[i + 1] = t;
                        t *= f1;
                        sm.tr[i + 2] = t;
                        t *= f2;
                        sm.tr[i + 3] = t;
                        t *= f3;
                        own[i] = own[i + 1] = own[i + 2] = own[i + 3] = uint8_t(lane);
                    }
                    for (; i < e; ++i) {
                        sm.tr[i] = t;
                        own[i] = uint8_t(lane);
                        t *= 1.0 - sm.al[i];
                    }
                }
                __syncwarp();
                // C (sample-parallel, every lane): w, v, d_rgb = d_color w (stored
                // coalesced), and in place delta (ts), w v (te), T (1 - alpha) v (tr)
#pragma unroll
                for (int k = 0; k < Tile<T>::CH / 32; ++k) {
                    const uint32_t i = 32u * k + uint32_t(lane);
                    if (32u * k >= n) break;  // warp-uniform
                    const bool in = i < n;
                    const int o = in ? int(own[i]) : 0;
                    const Up uo{__shfl_sync(0xffffffffu, u.dcx, o), __shfl_sync(0xffffffffu, u.dcy, o),
                                __shfl_sync(0xffffffffu, u.dcz, o), __shfl_sync(0xffffffffu, u.dop, o),
                                __shfl_sync(0xffffffffu, u.ddep, o)};
                    if (in) {
                        const double t0 = tv.ts[i], t1 = tv.te[i], a = sm.al[i], tr = sm.tr[i];
                        const double v = uo.value(double(tv.rgb[3 * i]), double(tv.rgb[3 * i + 1]),
                                                  double(tv.rgb[3 * i + 2]), 0.5 * (t0 + t1));
                        const double wgt = tr * a;
                        T* gr = g_rgb + 3 * uint64_t(base) + 3 * i;
                        gr[0] = T(uo.dcx * wgt);
                        gr[1] = T(uo.dcy * wgt);
                        gr[2] = T(uo.dcz * wgt);
                        tv.ts[i] = t1 - t0;
                        tv.te[i] = wgt * v;
                        sm.tr[i] = tr * (1.0 - a) * v;
                    }
                }
                __syncwarp();
                // D (lane-serial, reverse): suffix sum, rendering.cpp:99-108 — one
                // dependent DADD per sample
                if (lane >= g0 && lane <= g1) {
                    double suffix = 0.0;
                    uint32_t i = rr.end - base;
                    const uint32_t b = rr.off - base;
                    for (; i >= b + 4; i -= 4) {  // loads first, then the chain
                        const double d3_ = tv.ts[i - 1], a3 = sm.tr[i - 1], w3 = tv.te[i - 1];
                        const double d2_ = tv.ts[i - 2], a2 = sm.tr[i - 2], w2 = tv.te[i - 2];
                        const double d1_ = tv.ts[i - 3], a1 = sm.tr[i - 3], w1 = tv.te[i - 3];
                        const double d0_ = tv.ts[i - 4], a0 = sm.tr[i - 4], w0 = tv.te[i - 4];
                        tv.sig[i - 1] = T(d3_ * (a3 - suffix));
                        suffix += w3;
                        tv.sig[i - 2] = T(d2_ * (a2 - suffix));
                        suffix += w2;
                        tv.sig[i - 3] = T(d1_ * (a1 - suffix));
                        suffix += w1;
                        tv.sig[i - 4] = T(d0_ * (a0 - suffix));
                        suffix += w0;
                    }
                    while (i-- > b) {
                        tv.sig[i] = T(tv.ts[i] * (sm.tr[i] - suffix));
                        suffix += tv.te[i];
                    }
                }
                __syncwarp();
                T* psg = g_sig + base + lane;
#pragma unroll
                for (int k = 0; k < Tile<T>::CH / 32; ++k)
                    if (32u * k + lane < n) psg[32 * k] = tv.sig[32 * k + lane];
                __syncwarp();
            }
            g0 = g1 + 1;
        }
    }
}

// ------------------------------------------------------------------ transmittance
template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 32 / kWarps) k_transmittance(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ sig,
    T* __restrict__ out) {
    __shared__ BwdSmem<T> smem[kWarps];
    const int lane = threadIdx.x & 31;
    BwdSmem<T>& sm = smem[threadIdx.x >> 5];
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const RayRange rr = ray_range(offsets, counts, n_rays, n_samples, w, lane);
        double t = 1.0;  // rendering.cpp:26-31: out = T; T *= exp(-sigma * delta)
        if (rr.contiguous) {
            for (uint32_t cs = rr.s0; cs < rr.s1; cs += Tile<T>::CH) {
                const uint32_t n = min(uint32_t(Tile<T>::CH), rr.s1 - cs);
                stage_in<T, true>(sm, lane, cs, n, ts, te, static_cast<const T*>(nullptr), sig);
                for (uint32_t s = max(rr.off, cs); s < min(rr.end, cs + n); ++s) {
                    const uint32_t i = s - cs;
                    sm.tr[i] = t;
                    t *= sm.al[i];
                }
                __syncwarp();
                for (uint32_t i = lane; i < n; i += 32) out[cs + i] = T(sm.tr[i]);
                __syncwarp();
            }
        } else {
            for (uint32_t s = rr.off; s < rr.end; ++s) {
                out[s] = T(t);
                t *= exp(-double(sig[s]) * (te[s] - ts[s]));
            }
        }
    }
}

// ------------------------------------------------------------------ attribute
// render_attribute (rendering.cpp:114-134): dim-D values, thread per ray.
template <typename T>
__global__ void k_attribute(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts,
                            uint64_t n_rays, uint64_t n_samples, const double* __restrict__ ts, const double* __restrict__ te,
                            const T* __restrict__ sig, const T* __restrict__ values, uint64_t dim,
                            T* __restrict__ out) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rays;
         r += uint64_t(gridDim.x) * blockDim.x) {
        for (uint64_t k = 0; k < dim; ++k) out[r * dim + k] = T(0);
        uint64_t b = offsets[r], e = b + counts[r];
        b = b < n_samples ? b : n_samples;  // samples beyond the buffers are ignored
        e = e < n_samples ? e : n_samples;
        double trans = 1.0;
        for (uint64_t s = b; s < e; ++s) {
            double alpha = 1.0 - exp(-double(sig[s]) * (te[s] - ts[s]));
            double w = trans * alpha;
            for (uint64_t k = 0; k < dim; ++k)
                out[r * dim + k] = T(double(out[r * dim + k]) + w * double(values[s * dim + k]));
            trans *= 1.0 - alpha;
        }
    }
}

// ------------------------------------------------------------------ shading (harness)
template <typename RT, typename T, bool VOX>
__global__ void k_shade(const RT* __restrict__ orig, const RT* __restrict__ dirs, vmb_field f,
                        double time, const uint32_t* __restrict__ idx, const double* __restrict__ ts,
                        const double* __restrict__ te, uint64_t n, T* __restrict__ rgb,
                        T* __restrict__ sig) {
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < n;
         s += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t r = idx[s];
        D3 o = d3(double(orig[3 * r]), double(orig[3 * r + 1]), double(orig[3 * r + 2]));
        D3 d = d3(double(dirs[3 * r]), double(dirs[3 * r + 1]), double(dirs[3 * r + 2]));
        D3 p = o + d * (0.5 * (ts[s] + te[s]));  // voxmarch.cpp:243-244
        D3 c;
        double sigma = field_rgb_sigma_t<VOX>(f, time_shift(f, p, time), &c);
        rgb[3 * s] = T(c.x);
        rgb[3 * s + 1] = T(c.y);
        rgb[3 * s + 2] = T(c.z);
        sig[s] = T(sigma);
    }
}

int launched(const char* where) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, where);
}

#ifndef VMB_RENDER_CTAS
#define VMB_RENDER_CTAS 32
#endif
#ifndef VMB_FWD_WIN_CTAS
#define VMB_FWD_WIN_CTAS 6  // windowed forward CTAs per SM (r1 sweep: 6 best)
#endif
int render_blocks(vmb_ctx* ctx, uint64_t n_rays) {
    return grid_blocks(ctx, (n_rays + 31) / 32 * 32, kWarps * 32, VMB_RENDER_CTAS);
}

// render_backward: k_backward_hy (groups of whole rays per tile, the reference's
// sequential recurrences), then the rays it set aside (longer than a tile) by
// k_backward_long (one warp per ray, scans, suffix accumulated from the end).
template <typename T>
int launch_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* rgb, const void* sig, const void* dc,
                    const void* dop, const void* ddep, void* g_rgb, void* g_sig) {
    const int blocks = render_blocks(ctx, p->n_rays);
    auto* list = static_cast<uint32_t*>(scratch(ctx, SCRATCH_RENDER, 16 + 4 * p->n_rays));
    if (!list) return VMB_CUDA;
    auto* n_long = reinterpret_cast<unsigned int*>(list);
    zero_words_async(ctx, n_long, 1);
    constexpr size_t smem = kWarps * sizeof(BwdSmem<T, kBulkPad>);
    static const bool opted = [] {  // above the 48 KB default of dynamic shared memory
        return cudaFuncSetAttribute(k_backward_hy<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) ==
               cudaSuccess;
    }();
    (void)opted;
    launch_pdl(k_backward_hy<T>, dim3(blocks), dim3(kWarps * 32), smem, ctx->stream, p->d_offsets, p->d_counts,
               p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends, static_cast<const T*>(rgb),
               static_cast<const T*>(sig), static_cast<const T*>(dc), static_cast<const T*>(dop),
               static_cast<const T*>(ddep), static_cast<T*>(g_rgb), static_cast<T*>(g_sig), list + 4, n_long);
    launch_pdl(k_backward_long<T>, dim3(ctx->num_sms * (32 / kWarps)), dim3(kWarps * 32), 0, ctx->stream,
               p->d_offsets, p->d_counts, p->n_samples, p->d_t_starts, p->d_t_ends, static_cast<const T*>(rgb),
               static_cast<const T*>(sig), static_cast<const T*>(dc), static_cast<const T*>(dop),
               static_cast<const T*>(ddep), static_cast<T*>(g_rgb), static_cast<T*>(g_sig), list + 4, n_long);
    return launched("render_backward");
}

template <typename RT, typename T>
void launch_shade_forward(vmb_ctx* ctx, const vmb_rays* rays, const vmb_field* f, double time,
                          const vmb_packed_view* p, void* rgb, void* sig, void* color, void* opacity,
                          void* depth) {
    const int wb = grid_blocks(ctx, (p->n_rays + 31) / 32 * 32, kWinWarps * 32, VMB_FWD_WIN_CTAS);
    launch_pdl(f->kind == VMB_FIELD_VOXEL ? k_shade_forward_win<RT, T, true> : k_shade_forward_win<RT, T, false>,
               dim3(wb), dim3(kWinWarps * 32), 0, ctx->stream, static_cast<const RT*>(rays->d_origins),
               static_cast<const RT*>(rays->d_directions), *f, time, p->d_offsets, p->d_counts, p->n_rays,
               p->n_samples, p->d_t_starts, p->d_t_ends, static_cast<T*>(rgb), static_cast<T*>(sig),
               static_cast<T*>(color), static_cast<T*>(opacity), static_cast<T*>(depth));
}

}  // namespace
}  // namespace vmb

namespace vmb {
// render_backward of the listed rays only (one warp per ray): the fused training
// step's rays that its expansion could not differentiate (vm_internal.h).
int backward_listed(vmb_ctx* ctx, const vmb_packed_view* p, const void* rgb, const void* sig, const void* dc,
                    const void* dop, const void* ddep, void* g_rgb, void* g_sig, const uint32_t* list,
                    const unsigned int* n_list, int dtype) {
    auto go = [&](auto* t) {
        using T = std::remove_pointer_t<decltype(t)>;
        k_backward_long<T><<<ctx->num_sms * (32 / kWarps), kWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_samples, p->d_t_starts, p->d_t_ends, static_cast<const T*>(rgb),
            static_cast<const T*>(sig), static_cast<const T*>(dc), static_cast<const T*>(dop),
            static_cast<const T*>(ddep), static_cast<T*>(g_rgb), static_cast<T*>(g_sig), list, n_list);
    };
    if (dtype == VMB_F32)
        go(static_cast<float*>(nullptr));
    else
        go(static_cast<double*>(nullptr));
    return launched("render_backward");
}

// shade + render_forward in one pass for long-ray batches; returns 1 when the
// batch is not long-ray dominated (the caller runs k_shade -> render_forward).
int shade_forward_long(vmb_ctx* ctx, const vmb_rays* rays, const vmb_field* f, double time,
                       const vmb_packed_view* p, void* rgb, void* sig, void* color, void* opacity,
                       void* depth, int dtype) {
    if (!p->n_rays || p->n_samples <= uint64_t(kFwdLaneAvg) * p->n_rays) return 1;
    if (int frc = check_field(f)) return frc;
    if (rays->dtype == VMB_F32 && dtype == VMB_F32)
        launch_shade_forward<float, float>(ctx, rays, f, time, p, rgb, sig, color, opacity, depth);
    else if (rays->dtype == VMB_F32)
        launch_shade_forward<float, double>(ctx, rays, f, time, p, rgb, sig, color, opacity, depth);
    else if (dtype == VMB_F32)
        launch_shade_forward<double, float>(ctx, rays, f, time, p, rgb, sig, color, opacity, depth);
    else
        launch_shade_forward<double, double>(ctx, rays, f, time, p, rgb, sig, color, opacity, depth);
    return launched("shade_forward");
}
}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_render_forward(vmb_ctx* ctx, const vmb_packed_view* p, const void* rgb, const void* sig,
                       void* color, void* opacity, void* depth, int dtype) {
    if (!p->n_rays) return VMB_OK;
    if (p->n_samples > uint64_t(kFwdLaneAvg) * p->n_rays) {
        const int wb = grid_blocks(ctx, (p->n_rays + 31) / 32 * 32, kWinWarps * 32, VMB_FWD_WIN_CTAS);
        if (dtype == VMB_F32)
            k_forward_win<float><<<wb, kWinWarps * 32, 0, ctx->stream>>>(
                p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
                static_cast<const float*>(rgb), static_cast<const float*>(sig), static_cast<float*>(color),
                static_cast<float*>(opacity), static_cast<float*>(depth));
        else
            k_forward_win<double><<<wb, kWinWarps * 32, 0, ctx->stream>>>(
                p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
                static_cast<const double*>(rgb), static_cast<const double*>(sig),
                static_cast<double*>(color), static_cast<double*>(opacity), static_cast<double*>(depth));
        return launched("render_forward");
    }
    int blocks = render_blocks(ctx, p->n_rays);
    if (dtype == VMB_F32)
        k_forward<float><<<blocks, kWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
            static_cast<const float*>(rgb), static_cast<const float*>(sig), static_cast<float*>(color),
            static_cast<float*>(opacity), static_cast<float*>(depth));
    else
        k_forward<double><<<blocks, kWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
            static_cast<const double*>(rgb), static_cast<const double*>(sig), static_cast<double*>(color),
            static_cast<double*>(opacity), static_cast<double*>(depth));
    return launched("render_forward");
}

int vmb_render_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* rgb, const void* sig,
                        const void* dc, const void* dop, const void* ddep, void* g_rgb, void* g_sig,
                        int dtype) {
    if (!p->n_rays) return VMB_OK;
    return dtype == VMB_F32
               ? launch_backward<float>(ctx, p, rgb, sig, dc, dop, ddep, g_rgb, g_sig)
               : launch_backward<double>(ctx, p, rgb, sig, dc, dop, ddep, g_rgb, g_sig);
}

int vmb_transmittance(vmb_ctx* ctx, const vmb_packed_view* p, const void* sig, void* out, int dtype) {
    if (!p->n_rays) return VMB_OK;
    int blocks = render_blocks(ctx, p->n_rays);
    if (dtype == VMB_F32)
        k_transmittance<float><<<blocks, kWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
            static_cast<const float*>(sig), static_cast<float*>(out));
    else
        k_transmittance<double><<<blocks, kWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
            static_cast<const double*>(sig), static_cast<double*>(out));
    return launched("transmittance");
}

int vmb_render_attribute(vmb_ctx* ctx, const vmb_packed_view* p, const void* sig, const void* values,
                         uint64_t dim, void* out, int dtype) {
    if (dim == 0) return fail(VMB_INVALID_ARGUMENT, "rendering: value length mismatch");
    if (!p->n_rays) return VMB_OK;
    int blocks = grid_blocks(ctx, p->n_rays, 128, 16);
    if (dtype == VMB_F32)
        k_attribute<float><<<blocks, 128, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
            static_cast<const float*>(sig), static_cast<const float*>(values), dim, static_cast<float*>(out));
    else
        k_attribute<double><<<blocks, 128, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends,
            static_cast<const double*>(sig), static_cast<const double*>(values), dim,
            static_cast<double*>(out));
    return launched("render_attribute");
}

int vmb_shade_field(vmb_ctx* ctx, const vmb_rays* rays, const vmb_field* f, double time,
                    const uint32_t* idx, const double* ts, const double* te, uint64_t n, void* rgb,
                    void* sig, int dtype) {
    if (int frc = check_field(f)) return frc;
    if (!n) return VMB_OK;
    int blocks = grid_blocks(ctx, n, 256, 8);
    if (rays->dtype == VMB_F32 && dtype == VMB_F32)
        (f->kind == VMB_FIELD_VOXEL ? k_shade<float, float, true> : k_shade<float, float, false>)<<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const float*>(rays->d_origins), static_cast<const float*>(rays->d_directions), *f,
            time, idx, ts, te, n, static_cast<float*>(rgb), static_cast<float*>(sig));
    else if (rays->dtype == VMB_F32)
        (f->kind == VMB_FIELD_VOXEL ? k_shade<float, double, true> : k_shade<float, double, false>)<<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const float*>(rays->d_origins), static_cast<const float*>(rays->d_directions), *f,
            time, idx, ts, te, n, static_cast<double*>(rgb), static_cast<double*>(sig));
    else if (dtype == VMB_F32)
        (f->kind == VMB_FIELD_VOXEL ? k_shade<double, float, true> : k_shade<double, float, false>)<<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const double*>(rays->d_origins), static_cast<const double*>(rays->d_directions), *f,
            time, idx, ts, te, n, static_cast<float*>(rgb), static_cast<float*>(sig));
    else
        (f->kind == VMB_FIELD_VOXEL ? k_shade<double, double, true> : k_shade<double, double, false>)<<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const double*>(rays->d_origins), static_cast<const double*>(rays->d_directions), *f,
            time, idx, ts, te, n, static_cast<double*>(rgb), static_cast<double*>(sig));
    return launched("shade");
}

}  // extern "C"
