// voxfield.cu — field queries and the TrilinearVoxelField backward on the device
// (fields.cpp:75-93 query_density/query_rgb_sigma, :170-211 backward).
//
// Forward evaluation of every field kind lives in vm_exact.cuh (field_density /
// field_rgb_sigma), so march, shading and the grid update take a stored voxel
// field exactly like an analytic one. This file adds the batch queries and the
// parameter gradient.
//
// Backward. The reference accumulates accum[v] += w_k * g_i over samples i in
// order, so each vertex's sum is a left fold in sample order and the result is
// bitwise reproducible (fields.hpp:76-81). Two device modes:
//   VMB_GRAD_DETERMINISTIC — the same folds, bit for bit: every inside sample
//     emits 8 (vertex, record) pairs, record = 8 i + k; a stable LSD radix sort
//     by vertex (in-tree, sort.cu) orders each vertex's records by sample; one thread per
//     vertex segment then folds accum[v] + c_1 + c_2 + ... in that order.
//   VMB_GRAD_ATOMIC — fp64 atomicAdd per (sample, vertex); the fold order is
//     the hardware's, so sums differ from the reference in the last bits
//     (relative error ~ n_contributions * 2^-53; tests use rtol 1e-12).
#include "vm_internal.h"

namespace vmb {
namespace {

template <typename T>
__device__ __forceinline__ D3 ld3(const T* p, uint64_t i) {
    return d3(double(p[3 * i]), double(p[3 * i + 1]), double(p[3 * i + 2]));
}

// Position of sample i: an explicit point, or the midpoint o + d (0.5 (ts + te))
// of a packed sample (voxmarch.cpp:243-244), shifted by the field's velocity.
struct Positions {
    const double* points;  // [n][3] or null
    const void* orig;      // rays (when points is null)
    const void* dirs;
    int ray_dtype;
    const uint32_t* idx;
    const double* ts;
    const double* te;
    double time;
    __device__ __forceinline__ D3 at(const vmb_field& f, uint64_t i) const {
        D3 p;
        if (points) {
            p = ld3(points, i);
        } else {
            const uint64_t r = idx[i];
            const D3 o = ray_dtype == VMB_F32 ? ld3(static_cast<const float*>(orig), r)
                                              : ld3(static_cast<const double*>(orig), r);
            const D3 d = ray_dtype == VMB_F32 ? ld3(static_cast<const float*>(dirs), r)
                                              : ld3(static_cast<const double*>(dirs), r);
            p = o + d * (0.5 * (ts[i] + te[i]));
        }
        return time_shift(f, p, time);
    }
};

template <typename T>
__global__ void k_field_query(vmb_field f, Positions pos, uint64_t n, double* __restrict__ sig,
                              double* __restrict__ rgb, DevError* err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const D3 p = pos.at(f, i);
        if (!finite3(p)) {  // check_finite_positions (fields.cpp:14-19)
            atomicMin(&err->key, (unsigned long long)i);
            continue;
        }
        if (rgb) {
            D3 c;
            sig[i] = field_rgb_sigma(f, p, &c);
            rgb[3 * i] = c.x;
            rgb[3 * i + 1] = c.y;
            rgb[3 * i + 2] = c.z;
        } else {
            sig[i] = field_density(f, p);
        }
    }
}

// Per-sample chain rule through the activations (fields.cpp:189-197): returns
// false outside the box. g = {d_raw_density, d_raw_r, d_raw_g, d_raw_b}.
template <typename GT>
__device__ __forceinline__ bool sample_grad(const vmb_field& f, D3 p, const GT* d_rgbs, const GT* d_sigmas,
                                            uint64_t i, uint32_t c[3], double fr[3], double g[4]) {
    if (!vox_stencil(f, p, c, fr)) return false;
    double raw_d = 0.0, rr = 0.0, rg = 0.0, rb = 0.0;
    for (int k = 0; k < 8; ++k) {
        const double w = vox_weight(fr, k);
        const uint64_t v = vox_vertex(f, c, k);
        raw_d += w * f.vox_density[v];
        rr += w * f.vox_color[3 * v];
        rg += w * f.vox_color[3 * v + 1];
        rb += w * f.vox_color[3 * v + 2];
    }
    // softplus' = sigmoid; sigmoid' = s (1 - s), both at the interpolated raw value
    g[0] = double(d_sigmas[i]) * vox_sigmoid(raw_d);
    const double sr = vox_sigmoid(rr), sg = vox_sigmoid(rg), sb = vox_sigmoid(rb);
    g[1] = double(d_rgbs[3 * i]) * sr * (1.0 - sr);
    g[2] = double(d_rgbs[3 * i + 1]) * sg * (1.0 - sg);
    g[3] = double(d_rgbs[3 * i + 2]) * sb * (1.0 - sb);
    return true;
}

template <typename GT>
__global__ void k_vox_grad_atomic(vmb_field f, Positions pos, uint64_t n, const GT* __restrict__ d_rgbs,
                                  const GT* __restrict__ d_sigmas, double* __restrict__ acc_d,
                                  double* __restrict__ acc_c) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t c[3];
        double fr[3], g[4];
        if (!sample_grad(f, pos.at(f, i), d_rgbs, d_sigmas, i, c, fr, g)) continue;
        for (int k = 0; k < 8; ++k) {
            const double w = vox_weight(fr, k);
            const uint64_t v = vox_vertex(f, c, k);
            atomicAdd(acc_d + v, w * g[0]);
            atomicAdd(acc_c + 3 * v, w * g[1]);
            atomicAdd(acc_c + 3 * v + 1, w * g[2]);
            atomicAdd(acc_c + 3 * v + 2, w * g[3]);
        }
    }
}

// Deterministic mode, pass 1: per-sample gradient + stencil, and the 8 sort
// records (key = vertex, value = 8 i + k); outside samples emit sentinel keys.
template <typename GT>
__global__ void k_vox_grad_records(vmb_field f, Positions pos, uint64_t n, const GT* __restrict__ d_rgbs,
                                   const GT* __restrict__ d_sigmas, double4* __restrict__ sg,
                                   double4* __restrict__ sfr, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ vals, uint32_t sentinel) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t c[3];
        double fr[3], g[4];
        const bool in = sample_grad(f, pos.at(f, i), d_rgbs, d_sigmas, i, c, fr, g);
        sg[i] = make_double4(g[0], g[1], g[2], g[3]);
        sfr[i] = make_double4(fr[0], fr[1], fr[2], 0.0);
        for (int k = 0; k < 8; ++k) {
            keys[8 * i + k] = in ? uint32_t(vox_vertex(f, c, k)) : sentinel;
            vals[8 * i + k] = uint32_t(8 * i + k);
        }
    }
}

// Pass 3: one thread per segment head folds its vertex's records in order.
__global__ void k_vox_grad_fold(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                uint64_t m, uint32_t sentinel, const double4* __restrict__ sg,
                                const double4* __restrict__ sfr, double* __restrict__ acc_d,
                                double* __restrict__ acc_c) {
    for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
         j += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = keys[j];
        if (v == sentinel || (j > 0 && keys[j - 1] == v)) continue;
        double d = acc_d[v], r = acc_c[3 * uint64_t(v)], g = acc_c[3 * uint64_t(v) + 1],
               b = acc_c[3 * uint64_t(v) + 2];
        for (uint64_t q = j; q < m && keys[q] == v; ++q) {
            const uint32_t rec = vals[q];
            const uint64_t i = rec >> 3;
            const int k = int(rec & 7u);
            const double4 f4 = sfr[i];
            const double fr[3] = {f4.x, f4.y, f4.z};
            const double w = vox_weight(fr, k);
            const double4 g4 = sg[i];
            d += w * g4.x;  // accum[v] += w * d_raw (fields.cpp:198-205)
            r += w * g4.y;
            g += w * g4.z;
            b += w * g4.w;
        }
        acc_d[v] = d;
        acc_c[3 * uint64_t(v)] = r;
        acc_c[3 * uint64_t(v) + 1] = g;
        acc_c[3 * uint64_t(v) + 2] = b;
    }
}

int first_bad_position(vmb_ctx* ctx, const vmb_field& f, const Positions& pos, uint64_t n, double* sig,
                       double* rgb) {
    int rc = reset_error(ctx);
    if (rc) return rc;
    k_field_query<double><<<grid_blocks(ctx, n, 256, 8), 256, 0, ctx->stream>>>(f, pos, n, sig, rgb, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull)
        return fail(VMB_INVALID_ARGUMENT, "field: non-finite position at index " + std::to_string(err.key));
    return VMB_OK;
}

template <typename GT>
int vox_backward(vmb_ctx* ctx, const vmb_field& f, const Positions& pos, uint64_t n, const GT* d_rgbs,
                 const GT* d_sigmas, double* acc_d, double* acc_c, int mode) {
    if (!n) return VMB_OK;
    const uint64_t n_vert = uint64_t(f.vox_resolution) * f.vox_resolution * f.vox_resolution;
    if (mode == VMB_GRAD_ATOMIC) {
        k_vox_grad_atomic<GT><<<grid_blocks(ctx, n, 256, 8), 256, 0, ctx->stream>>>(f, pos, n, d_rgbs, d_sigmas,
                                                                                     acc_d, acc_c);
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? VMB_OK : cuda_fail(e, "voxel field backward");
    }
    if (8 * n > 0xffffffffull || n_vert >= 0xffffffffull)
        return fail(VMB_INVALID_ARGUMENT, "voxel field backward: more than 2^29 samples per call");
    const uint64_t m = 8 * n;
    const uint32_t sentinel = 0xffffffffu;
    int end_bit = 1;
    while (end_bit < 32 && (1ull << end_bit) <= n_vert) ++end_bit;  // keys < 2^end_bit except the sentinel
    // the sentinel must sort last: give it the top key within end_bit bits
    const uint32_t sent = end_bit >= 32 ? sentinel : uint32_t((1ull << end_bit) - 1);
    const size_t bytes = m * 16 + n * 64 + 256;
    char* base = static_cast<char*>(scratch(ctx, SCRATCH_VOXGRAD, bytes));
    if (!base) return VMB_CUDA;
    auto* k_in = reinterpret_cast<uint32_t*>(base);
    auto* k_out = k_in + m;
    auto* v_in = k_out + m;
    auto* v_out = v_in + m;
    auto* sg = reinterpret_cast<double4*>(base + ((m * 16 + 31) & ~size_t(31)));
    auto* sfr = sg + n;
    k_vox_grad_records<GT><<<grid_blocks(ctx, n, 256, 8), 256, 0, ctx->stream>>>(f, pos, n, d_rgbs, d_sigmas, sg,
                                                                                 sfr, k_in, v_in, sent);
    uint32_t *ks = nullptr, *vs = nullptr;
    if (int rc = radix_sort_pairs(ctx, k_in, v_in, k_out, v_out, m, end_bit, &ks, &vs)) return rc;
    k_vox_grad_fold<<<grid_blocks(ctx, m, 256, 8), 256, 0, ctx->stream>>>(ks, vs, m, sent, sg, sfr, acc_d, acc_c);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "voxel field backward");
}

// AdamOptimizer::step (fields.cpp:282-292): the reference's expressions per
// element; bias corrections come from the host (std::pow, as the reference).
__global__ void k_adam_check(const double* __restrict__ g, uint64_t n, DevError* err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        if (!isfinite(g[i])) atomicMin(&err->key, (unsigned long long)i);
}

__global__ void k_adam(double* __restrict__ p, const double* __restrict__ g, double* __restrict__ m,
                       double* __restrict__ v, uint64_t n, double lr, double b1, double b2, double eps,
                       double bias1, double bias2) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double gi = g[i];
        const double mi = b1 * m[i] + (1.0 - b1) * gi;
        const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const double m_hat = mi / bias1;
        const double v_hat = vi / bias2;
        p[i] -= lr * m_hat / (sqrt(v_hat) + eps);
    }
}

Positions sample_positions(const vmb_rays* rays, const uint32_t* idx, const double* ts, const double* te,
                           double time) {
    return Positions{nullptr, rays->d_origins, rays->d_directions, rays->dtype, idx, ts, te, time};
}

}  // namespace
}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_field_query(vmb_ctx* ctx, const vmb_field* f, const double* d_points, uint64_t n, double time,
                    double* d_sigmas, double* d_rgbs) {
    if (int rc = check_field(f)) return rc;
    if (!n) return VMB_OK;
    return first_bad_position(ctx, *f, Positions{d_points, nullptr, nullptr, 0, nullptr, nullptr, nullptr, time},
                              n, d_sigmas, d_rgbs);
}

int vmb_voxel_field_backward(vmb_ctx* ctx, const vmb_field* f, const double* d_points, uint64_t n,
                             const void* d_rgb_grads, const void* d_sigma_grads, int dtype,
                             double* d_accum_density, double* d_accum_color, int mode) {
    if (int rc = check_field(f)) return rc;
    if (f->kind != VMB_FIELD_VOXEL) return fail(VMB_INVALID_ARGUMENT, "voxel field backward: not a voxel field");
    const Positions pos{d_points, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0.0};
    if (dtype == VMB_F32)
        return vox_backward(ctx, *f, pos, n, static_cast<const float*>(d_rgb_grads),
                            static_cast<const float*>(d_sigma_grads), d_accum_density, d_accum_color, mode);
    return vox_backward(ctx, *f, pos, n, static_cast<const double*>(d_rgb_grads),
                        static_cast<const double*>(d_sigma_grads), d_accum_density, d_accum_color, mode);
}

int vmb_voxel_field_backward_samples(vmb_ctx* ctx, const vmb_field* f, const vmb_rays* rays,
                                     const uint32_t* d_ray_indices, const double* d_t_starts,
                                     const double* d_t_ends, uint64_t n_samples, double time,
                                     const void* d_rgb_grads, const void* d_sigma_grads, int dtype,
                                     double* d_accum_density, double* d_accum_color, int mode) {
    if (int rc = check_field(f)) return rc;
    if (f->kind != VMB_FIELD_VOXEL) return fail(VMB_INVALID_ARGUMENT, "voxel field backward: not a voxel field");
    const Positions pos = sample_positions(rays, d_ray_indices, d_t_starts, d_t_ends, time);
    if (dtype == VMB_F32)
        return vox_backward(ctx, *f, pos, n_samples, static_cast<const float*>(d_rgb_grads),
                            static_cast<const float*>(d_sigma_grads), d_accum_density, d_accum_color, mode);
    return vox_backward(ctx, *f, pos, n_samples, static_cast<const double*>(d_rgb_grads),
                        static_cast<const double*>(d_sigma_grads), d_accum_density, d_accum_color, mode);
}

int vmb_adam_step(vmb_ctx* ctx, uint64_t n, double* d_params, const double* d_grads, double* d_m, double* d_v,
                  double lr, double beta1, double beta2, double eps, uint64_t step) {
    if (!n) return VMB_OK;
    int rc = reset_error(ctx);
    if (rc) return rc;
    const int blocks = grid_blocks(ctx, n, 256, 8);
    k_adam_check<<<blocks, 256, 0, ctx->stream>>>(d_grads, n, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull)
        return fail(VMB_RUNTIME, "adam: non-finite gradient at index " + std::to_string(err.key));
    const double bias1 = 1.0 - std::pow(beta1, double(step));
    const double bias2 = 1.0 - std::pow(beta2, double(step));
    k_adam<<<blocks, 256, 0, ctx->stream>>>(d_params, d_grads, d_m, d_v, n, lr, beta1, beta2, eps, bias1, bias2);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "adam");
}

}  // extern "C"
