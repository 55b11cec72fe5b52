// ops.cu — NerfAcc's standalone compositing operators over packed samples, and
// ray_aabb_intersect.
//
// The reference has these only fused inside render_forward / render_backward
// (rendering.cpp:47-58, 67-112) and transmittance (rendering.cpp:19-33); the
// north_star names them as separate kernels with their own backward:
//
//   render_weight_from_density   alpha = 1 - exp(-sigma (t_end - t_start)),
//                                T = exclusive prod (1 - alpha), w = T alpha
//   render_weight_from_alpha     T = exclusive prod (1 - alpha), w = T alpha
//   render_transmittance_from_alpha  T only
//   accumulate_along_rays        out[ray] = sum w v (a segmented reduce)
//   ray_aabb_intersect           slab test per (ray, box)
//
// Layout: ray-contiguous packed samples (offsets = exclusive scan of counts), so
// the samples of 32 consecutive rays are one contiguous range. A warp owns 32
// rays and streams their range in rounds of 32 consecutive samples, one sample
// per lane (coalesced loads), with SEGMENTED warp-shuffle scans:
//   forward   exclusive product of (1 - alpha) with a head flag at each ray's
//             first sample, the running product carried across rounds;
//   backward  a reverse segmented scan of affine maps x -> c + m x (m = 1 - alpha),
//             tail flag at each ray's last sample, carried backwards across rounds:
//               W_j = sum_{i>j} (gw_i alpha_i + gT_i) prod_{j<k<i} (1 - alpha_k)
//             so that, division-free,
//               dL/dalpha_j = T_j (gw_j - W_j)                  (weights, T)
//               dL/dsigma_j = delta_j (1 - alpha_j) (g_alpha_j + T_j (gw_j - W_j))
//             The latter equals rendering.cpp:99-108's delta (T (1 - alpha) v - suffix)
//             with v = gw, suffix = sum_{k>j} w_k v_k, since T_j (1 - alpha_j) W_j is
//             that suffix (plus the gT terms, which render_backward does not have).
// The reverse sweep needs T at the start of each round: a forward sweep stores the
// carry-in of up to kCarry rounds in shared memory; longer ranges are processed in
// super-blocks of kCarry rounds from the end, each re-running the forward sweep.
// Products and sums are reassociated by the scans: results agree with the
// reference's sequential order to a few ulps (the contract is rel 1e-5).
// Warps whose rays are not contiguous run the same scans one ray at a time.
#include "vm_internal.h"
#include "vm_scan.cuh"

namespace vmb {
namespace {

constexpr int kOpsWarps = 8;
constexpr int kCarry = 32;  // rounds (x 32 samples) of carried T per super-block

// The warp's 32 rays: offsets/ends clamped into [0, n_samples); contiguous when
// every valid ray ends where the next valid ray begins (then [s0, s1) is theirs).
struct Warp32 {
    uint64_t ray;
    bool valid;
    uint32_t off, end;
    bool contiguous;
    uint32_t s0, s1;
};

__device__ __forceinline__ Warp32 warp_rays(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts,
                                            uint64_t n_rays, uint64_t n_samples, uint64_t w, int lane) {
    Warp32 r;
    r.ray = w * 32 + lane;
    r.valid = r.ray < n_rays;
    const uint64_t ns = n_samples < 0xffffffffull ? n_samples : 0xffffffffull;
    const uint64_t o = r.valid ? __ldg(offsets + r.ray) : 0u;
    const uint64_t e = r.valid ? o + __ldg(counts + r.ray) : 0u;
    r.off = uint32_t(o < ns ? o : ns);
    r.end = uint32_t(e < ns ? e : ns);
    const uint32_t next_off = __shfl_down_sync(0xffffffffu, r.off, 1);
    const int next_valid = __shfl_down_sync(0xffffffffu, int(r.valid), 1);
    const bool ok = !(r.valid && lane < 31 && next_valid) || r.end == next_off;
    r.contiguous = __all_sync(0xffffffffu, ok);
    const unsigned vm = __ballot_sync(0xffffffffu, r.valid);
    r.s0 = __shfl_sync(0xffffffffu, r.off, 0);
    r.s1 = __shfl_sync(0xffffffffu, r.end, vm ? 31 - __clz(vm) : 0);
    return r;
}

// A range of samples [a, b) and the rule that maps a position to its ray:
// single (one ray, lane `one`) or the warp's contiguous rays (owner search).
struct Range {
    uint32_t a, b;
    int one;           // >= 0: every sample belongs to this lane's ray
    uint32_t off, end; // this lane's ray (for the owner search)
    bool valid;
};

// Owner lane of position p (largest valid lane with off <= p), and whether p is
// the first / last sample of its ray.
__device__ __forceinline__ int owner(const Range& R, uint32_t p, bool* head, bool* tail) {
    int L;
    if (R.one >= 0) {
        L = R.one;
        *head = p == R.a;
        *tail = p + 1 == R.b;
        return L;
    }
    const uint32_t key = R.valid ? R.off : 0xffffffffu;
    L = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, key, (L + s) & 31);
        if (L + s < 32 && v <= p) L += s;
    }
    const uint32_t o = __shfl_sync(0xffffffffu, R.off, L);
    const uint32_t e = __shfl_sync(0xffffffffu, R.end, L);
    *head = p == o;
    *tail = p + 1 == e;
    return L;
}

// alpha of sample p: from sigma and the interval (density ops) or given.
template <typename T, bool DENS>
__device__ __forceinline__ double alpha_at(const T* __restrict__ x, const double* __restrict__ ts,
                                           const double* __restrict__ te, uint32_t p) {
    if (DENS) return 1.0 - exp(-double(x[p]) * (te[p] - ts[p]));  // rendering.cpp:47-49
    return double(x[p]);
}

// ------------------------------------------------------------------ forward
// weights / transmittance / alphas of one range (any output may be null).
template <typename T, bool DENS>
__device__ void fwd_range(const Range& R, const T* __restrict__ x, const double* __restrict__ ts,
                          const double* __restrict__ te, T* __restrict__ w_out, T* __restrict__ t_out,
                          T* __restrict__ a_out) {
    const int lane = threadIdx.x & 31;
    double carry = 1.0;
    for (uint32_t base = R.a; base < R.b; base += 32) {
        const uint32_t p = base + lane;
        const bool in = p < R.b;
        bool head = false, tail = false;
        owner(R, in ? p : R.b - 1, &head, &tail);
        head = head && in;
        const double a = in ? alpha_at<T, DENS>(x, ts, te, p) : 0.0;
        const double t = seg_excl_prod(in ? 1.0 - a : 1.0, head, carry);
        if (in) {
            if (w_out) w_out[p] = T(t * a);
            if (t_out) t_out[p] = T(t);
            if (a_out) a_out[p] = T(a);
        }
    }
}

template <typename T, bool DENS>
__global__ void __launch_bounds__(kOpsWarps * 32) k_weights(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ x, T* __restrict__ w_out,
    T* __restrict__ t_out, T* __restrict__ a_out) {
    const int lane = threadIdx.x & 31;
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const Warp32 wr = warp_rays(offsets, counts, n_rays, n_samples, w, lane);
        if (wr.contiguous) {
            fwd_range<T, DENS>(Range{wr.s0, wr.s1, -1, wr.off, wr.end, wr.valid}, x, ts, te, w_out, t_out, a_out);
        } else {
            for (int r = 0; r < 32; ++r) {
                const uint32_t a = __shfl_sync(0xffffffffu, wr.off, r), b = __shfl_sync(0xffffffffu, wr.end, r);
                if (__shfl_sync(0xffffffffu, int(wr.valid), r) && a < b)
                    fwd_range<T, DENS>(Range{a, b, r, 0, 0, true}, x, ts, te, w_out, t_out, a_out);
            }
        }
    }
}

// ------------------------------------------------------------------ backward
// gw / gT / ga: upstream gradients of weights, transmittance, alphas (nullable).
// DENS: out = dL/dsigma; else out = dL/dalpha.
template <typename T, bool DENS>
__device__ void bwd_range(const Range& R, double* s_carry, const T* __restrict__ x, const double* __restrict__ ts,
                          const double* __restrict__ te, const T* __restrict__ gw, const T* __restrict__ gT,
                          const T* __restrict__ ga, T* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint32_t nr = (R.b - R.a + 31) / 32;
    double carryV = 0.0;  // reverse carry, kept across super-blocks
    for (uint32_t sb_end = nr; sb_end > 0;) {
        const uint32_t sb_start = sb_end > uint32_t(kCarry) ? sb_end - kCarry : 0u;
        // forward sweep up to the super-block's end: T carried into each of its rounds
        double carryT = 1.0;
        for (uint32_t k = 0; k < sb_end; ++k) {
            if (k >= sb_start && lane == 0) s_carry[k - sb_start] = carryT;
            const uint32_t p = R.a + 32 * k + lane;
            const bool in = p < R.b;
            bool head = false, tail = false;
            owner(R, in ? p : R.b - 1, &head, &tail);
            head = head && in;
            const double a = in ? alpha_at<T, DENS>(x, ts, te, p) : 0.0;
            seg_excl_prod(in ? 1.0 - a : 1.0, head, carryT);
        }
        __syncwarp();
        // reverse sweep over the super-block's rounds
        for (uint32_t k = sb_end; k-- > sb_start;) {
            double cT = s_carry[k - sb_start];
            const uint32_t p = R.a + 32 * k + lane;
            const bool in = p < R.b;
            bool head = false, tail = false;
            owner(R, in ? p : R.b - 1, &head, &tail);
            head = head && in;
            tail = tail || !in;  // lanes past the range end close nothing open
            const double a = in ? alpha_at<T, DENS>(x, ts, te, p) : 0.0;
            const double t = seg_excl_prod(in ? 1.0 - a : 1.0, head, cT);
            const double g_w = in && gw ? double(gw[p]) : 0.0;
            const double g_t = in && gT ? double(gT[p]) : 0.0;
            const double W = seg_excl_affine_rev(in ? g_w * a + g_t : 0.0, in ? 1.0 - a : 1.0, tail, carryV);
            if (in) {
                const double g_alpha = t * (g_w - W);
                if (DENS) {
                    const double g_a = ga ? double(ga[p]) + g_alpha : g_alpha;
                    out[p] = T((te[p] - ts[p]) * (1.0 - a) * g_a);
                } else {
                    out[p] = T(g_alpha);
                }
            }
        }
        __syncwarp();
        sb_end = sb_start;
    }
}

template <typename T, bool DENS>
__global__ void __launch_bounds__(kOpsWarps * 32) k_weights_bwd(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const double* __restrict__ ts, const double* __restrict__ te, const T* __restrict__ x, const T* __restrict__ gw,
    const T* __restrict__ gT, const T* __restrict__ ga, T* __restrict__ out) {
    __shared__ double s_carry[kOpsWarps][kCarry];
    const int lane = threadIdx.x & 31;
    double* sc = s_carry[threadIdx.x >> 5];
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const Warp32 wr = warp_rays(offsets, counts, n_rays, n_samples, w, lane);
        if (wr.contiguous) {
            bwd_range<T, DENS>(Range{wr.s0, wr.s1, -1, wr.off, wr.end, wr.valid}, sc, x, ts, te, gw, gT, ga, out);
        } else {
            for (int r = 0; r < 32; ++r) {
                const uint32_t a = __shfl_sync(0xffffffffu, wr.off, r), b = __shfl_sync(0xffffffffu, wr.end, r);
                if (__shfl_sync(0xffffffffu, int(wr.valid), r) && a < b)
                    bwd_range<T, DENS>(Range{a, b, r, 0, 0, true}, sc, x, ts, te, gw, gT, ga, out);
            }
        }
    }
}

// ------------------------------------------------------------------ accumulate_along_rays
// out[ray][d] = sum over the ray's samples, in order, of w * v[d] (v = 1 when
// values is null: the ray's opacity). Segmented sum scan; the ray's last sample
// writes (rays without samples write 0 from their own lane).
template <typename T>
__device__ void acc_range(const Range& R, uint64_t ray0, const T* __restrict__ wts, const T* __restrict__ v,
                          uint64_t dim, uint64_t d, T* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    double carry = 0.0;
    for (uint32_t base = R.a; base < R.b; base += 32) {
        const uint32_t p = base + lane;
        const bool in = p < R.b;
        bool head = false, tail = false;
        const int L = owner(R, in ? p : R.b - 1, &head, &tail);
        head = head && in;
        double x = in ? double(wts[p]) * (v ? double(v[uint64_t(p) * dim + d]) : 1.0) : 0.0;
        int f = head;
#pragma unroll
        for (int s = 1; s < 32; s <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, s);
            const int g = __shfl_up_sync(0xffffffffu, f, s);
            if (lane >= s) {
                if (!f) x = y + x;
                f |= g;
            }
        }
        if (!f) x = carry + x;
        carry = __shfl_sync(0xffffffffu, x, 31);
        if (in && tail) out[(ray0 + uint64_t(L)) * dim + d] = T(x);
    }
}

template <typename T>
__global__ void __launch_bounds__(kOpsWarps * 32) k_accumulate(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const T* __restrict__ wts, const T* __restrict__ v, uint64_t dim, T* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const Warp32 wr = warp_rays(offsets, counts, n_rays, n_samples, w, lane);
        if (wr.valid && wr.off >= wr.end)
            for (uint64_t d = 0; d < dim; ++d) out[wr.ray * dim + d] = T(0);
        for (uint64_t d = 0; d < dim; ++d) {
            if (wr.contiguous) {
                acc_range<T>(Range{wr.s0, wr.s1, -1, wr.off, wr.end, wr.valid}, w * 32, wts, v, dim, d, out);
            } else {
                for (int r = 0; r < 32; ++r) {
                    const uint32_t a = __shfl_sync(0xffffffffu, wr.off, r), b = __shfl_sync(0xffffffffu, wr.end, r);
                    if (__shfl_sync(0xffffffffu, int(wr.valid), r) && a < b)
                        acc_range<T>(Range{a, b, r, 0, 0, true}, w * 32, wts, v, dim, d, out);
                }
            }
        }
    }
}

// backward: g_w[s] = sum_d g_out[ray][d] v[s][d]; g_v[s][d] = w[s] g_out[ray][d]
template <typename T>
__global__ void __launch_bounds__(kOpsWarps * 32) k_accumulate_bwd(
    const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ counts, uint64_t n_rays, uint64_t n_samples,
    const T* __restrict__ wts, const T* __restrict__ v, uint64_t dim, const T* __restrict__ g_out,
    T* __restrict__ g_w, T* __restrict__ g_v) {
    const int lane = threadIdx.x & 31;
    const uint64_t n_warps = (n_rays + 31) / 32;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < n_warps;
         w += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const Warp32 wr = warp_rays(offsets, counts, n_rays, n_samples, w, lane);
        auto one = [&](uint32_t p, uint64_t ray) {
            double s = 0.0;
            for (uint64_t d = 0; d < dim; ++d) {
                const double g = double(g_out[ray * dim + d]);
                s += g * (v ? double(v[uint64_t(p) * dim + d]) : 1.0);
                if (g_v) g_v[uint64_t(p) * dim + d] = T(double(wts[p]) * g);
            }
            if (g_w) g_w[p] = T(s);
        };
        if (wr.contiguous) {
            const Range R{wr.s0, wr.s1, -1, wr.off, wr.end, wr.valid};
            for (uint32_t base = R.a; base < R.b; base += 32) {
                const uint32_t p = base + lane;
                bool h, t;
                const int L = owner(R, p < R.b ? p : R.b - 1, &h, &t);
                if (p < R.b) one(p, w * 32 + L);
            }
        } else if (wr.valid) {
            for (uint32_t p = wr.off; p < wr.end; ++p) one(p, wr.ray);
        }
    }
}

// ------------------------------------------------------------------ ray_aabb_intersect
// NerfAcc's ray_aabb_intersect: per (ray, box) slab test in fp64,
//   t_min = max(near, max_a min(t1_a, t2_a)), t_max = min(far, min_a max(t1_a, t2_a)),
//   t_a = (box_a - o_a) / d_a  (IEEE: d_a = 0 gives +-inf, or NaN when o_a is on a
//   slab plane — then that axis does not constrain: fmax/fmin drop the NaN),
//   hit = t_max > t_min; a miss stores miss_value in both.
template <typename RT>
__global__ void k_ray_aabb(const RT* __restrict__ o, const RT* __restrict__ d, uint64_t n_rays,
                           const double* __restrict__ boxes, uint64_t n_boxes, double near_, double far_,
                           double miss, double* __restrict__ tmin, double* __restrict__ tmax,
                           uint8_t* __restrict__ hit) {
    const uint64_t n = n_rays * n_boxes;
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = k / n_boxes, b = k - r * n_boxes;
        double lo = near_, hi = far_;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double oa = double(o[3 * r + a]), da = double(d[3 * r + a]);
            const double t1 = (boxes[6 * b + a] - oa) / da, t2 = (boxes[6 * b + 3 + a] - oa) / da;
            lo = fmax(lo, fmin(t1, t2));
            hi = fmin(hi, fmax(t1, t2));
        }
        const bool h = hi > lo;
        tmin[k] = h ? lo : miss;
        tmax[k] = h ? hi : miss;
        if (hit) hit[k] = uint8_t(h);
    }
}

int ops_blocks(vmb_ctx* ctx, uint64_t n_rays) { return grid_blocks(ctx, (n_rays + 31) / 32 * 32, kOpsWarps * 32, 8); }

int launched(const char* where) {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, where);
}

int check_view(const vmb_packed_view* p, bool need_t) {
    if (!p) return fail(VMB_INVALID_ARGUMENT, "rendering: packed view required");
    if (p->n_rays && (!p->d_offsets || !p->d_counts))
        return fail(VMB_INVALID_ARGUMENT, "rendering: packed offsets/counts required");
    if (need_t && p->n_samples && (!p->d_t_starts || !p->d_t_ends))
        return fail(VMB_INVALID_ARGUMENT, "rendering: t_starts/t_ends required");
    return VMB_OK;
}

template <typename T>
int weights_fwd(vmb_ctx* ctx, const vmb_packed_view* p, bool dens, const void* x, void* w, void* t, void* a) {
    auto kern = dens ? k_weights<T, true> : k_weights<T, false>;
    kern<<<ops_blocks(ctx, p->n_rays), kOpsWarps * 32, 0, ctx->stream>>>(
        p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends, static_cast<const T*>(x),
        static_cast<T*>(w), static_cast<T*>(t), static_cast<T*>(a));
    return launched("render_weights");
}

template <typename T>
int weights_bwd(vmb_ctx* ctx, const vmb_packed_view* p, bool dens, const void* x, const void* gw, const void* gT,
                const void* ga, void* out) {
    auto kern = dens ? k_weights_bwd<T, true> : k_weights_bwd<T, false>;
    kern<<<ops_blocks(ctx, p->n_rays), kOpsWarps * 32, 0, ctx->stream>>>(
        p->d_offsets, p->d_counts, p->n_rays, p->n_samples, p->d_t_starts, p->d_t_ends, static_cast<const T*>(x),
        static_cast<const T*>(gw), static_cast<const T*>(gT), static_cast<const T*>(ga), static_cast<T*>(out));
    return launched("render_weights_backward");
}

}  // namespace
}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_render_weight_from_density(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_sigmas, void* d_weights,
                                   void* d_trans, void* d_alphas, int dtype) {
    if (int rc = check_view(p, true)) return rc;
    if (!p->n_rays || !p->n_samples) return VMB_OK;
    return dtype == VMB_F32 ? weights_fwd<float>(ctx, p, true, d_sigmas, d_weights, d_trans, d_alphas)
                            : weights_fwd<double>(ctx, p, true, d_sigmas, d_weights, d_trans, d_alphas);
}

int vmb_render_weight_from_density_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_sigmas,
                                            const void* d_grad_weights, const void* d_grad_trans,
                                            const void* d_grad_alphas, void* d_grad_sigmas, int dtype) {
    if (int rc = check_view(p, true)) return rc;
    if (!p->n_rays || !p->n_samples) return VMB_OK;
    return dtype == VMB_F32
               ? weights_bwd<float>(ctx, p, true, d_sigmas, d_grad_weights, d_grad_trans, d_grad_alphas, d_grad_sigmas)
               : weights_bwd<double>(ctx, p, true, d_sigmas, d_grad_weights, d_grad_trans, d_grad_alphas,
                                     d_grad_sigmas);
}

int vmb_render_weight_from_alpha(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas, void* d_weights,
                                 void* d_trans, int dtype) {
    if (int rc = check_view(p, false)) return rc;
    if (!p->n_rays || !p->n_samples) return VMB_OK;
    return dtype == VMB_F32 ? weights_fwd<float>(ctx, p, false, d_alphas, d_weights, d_trans, nullptr)
                            : weights_fwd<double>(ctx, p, false, d_alphas, d_weights, d_trans, nullptr);
}

int vmb_render_weight_from_alpha_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas,
                                          const void* d_grad_weights, const void* d_grad_trans, void* d_grad_alphas,
                                          int dtype) {
    if (int rc = check_view(p, false)) return rc;
    if (!p->n_rays || !p->n_samples) return VMB_OK;
    return dtype == VMB_F32
               ? weights_bwd<float>(ctx, p, false, d_alphas, d_grad_weights, d_grad_trans, nullptr, d_grad_alphas)
               : weights_bwd<double>(ctx, p, false, d_alphas, d_grad_weights, d_grad_trans, nullptr, d_grad_alphas);
}

int vmb_render_transmittance_from_alpha(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas, void* d_trans,
                                        int dtype) {
    return vmb_render_weight_from_alpha(ctx, p, d_alphas, nullptr, d_trans, dtype);
}

int vmb_render_transmittance_from_alpha_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas,
                                                 const void* d_grad_trans, void* d_grad_alphas, int dtype) {
    return vmb_render_weight_from_alpha_backward(ctx, p, d_alphas, nullptr, d_grad_trans, d_grad_alphas, dtype);
}

int vmb_accumulate_along_rays(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_weights, const void* d_values,
                              uint64_t dim, void* d_out, int dtype) {
    if (dim == 0) return fail(VMB_INVALID_ARGUMENT, "rendering: value length mismatch");
    if (int rc = check_view(p, false)) return rc;
    if (!p->n_rays) return VMB_OK;
    const int blocks = ops_blocks(ctx, p->n_rays);
    if (dtype == VMB_F32)
        k_accumulate<float><<<blocks, kOpsWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, static_cast<const float*>(d_weights),
            static_cast<const float*>(d_values), dim, static_cast<float*>(d_out));
    else
        k_accumulate<double><<<blocks, kOpsWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, static_cast<const double*>(d_weights),
            static_cast<const double*>(d_values), dim, static_cast<double*>(d_out));
    return launched("accumulate_along_rays");
}

int vmb_accumulate_along_rays_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_weights,
                                       const void* d_values, uint64_t dim, const void* d_grad_out,
                                       void* d_grad_weights, void* d_grad_values, int dtype) {
    if (dim == 0) return fail(VMB_INVALID_ARGUMENT, "rendering: value length mismatch");
    if (int rc = check_view(p, false)) return rc;
    if (!p->n_rays || !p->n_samples) return VMB_OK;
    const int blocks = ops_blocks(ctx, p->n_rays);
    if (dtype == VMB_F32)
        k_accumulate_bwd<float><<<blocks, kOpsWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, static_cast<const float*>(d_weights),
            static_cast<const float*>(d_values), dim, static_cast<const float*>(d_grad_out),
            static_cast<float*>(d_grad_weights), static_cast<float*>(d_grad_values));
    else
        k_accumulate_bwd<double><<<blocks, kOpsWarps * 32, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, p->n_rays, p->n_samples, static_cast<const double*>(d_weights),
            static_cast<const double*>(d_values), dim, static_cast<const double*>(d_grad_out),
            static_cast<double*>(d_grad_weights), static_cast<double*>(d_grad_values));
    return launched("accumulate_along_rays_backward");
}

int vmb_ray_aabb_intersect(vmb_ctx* ctx, const vmb_rays* rays, const double* d_aabbs, uint64_t n_aabbs,
                           double miss_value, double* d_t_min, double* d_t_max, uint8_t* d_hit) {
    if (!rays) return fail(VMB_INVALID_ARGUMENT, "ray_aabb_intersect: rays required");
    const uint64_t n = rays->n_rays * n_aabbs;
    if (!n) return VMB_OK;
    const int blocks = grid_blocks(ctx, n, 256, 8);
    if (rays->dtype == VMB_F32)
        k_ray_aabb<float><<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const float*>(rays->d_origins), static_cast<const float*>(rays->d_directions), rays->n_rays,
            d_aabbs, n_aabbs, rays->near_plane, rays->far_plane, miss_value, d_t_min, d_t_max, d_hit);
    else
        k_ray_aabb<double><<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const double*>(rays->d_origins), static_cast<const double*>(rays->d_directions), rays->n_rays,
            d_aabbs, n_aabbs, rays->near_plane, rays->far_plane, miss_value, d_t_min, d_t_max, d_hit);
    return launched("ray_aabb_intersect");
}

}  // extern "C"
