// train.cu — the per-ray pieces of a training step around the hot path
// (tools/voxmarch.cpp cmd_train:460-498): minibatch gather and the photometric
// MSE loss against a white background with its upstream gradients.
#include <cstring>

#include "vm_internal.h"

namespace vmb {
namespace {

constexpr int kLossThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kLossThreads) k_loss_mse_bg(const T* __restrict__ color,
                                                              const T* __restrict__ opacity,
                                                              const T* __restrict__ target, uint64_t n,
                                                              double inv, T* __restrict__ dcol,
                                                              T* __restrict__ dop, T* __restrict__ ddep,
                                                              double* __restrict__ partial) {
    __shared__ double red[kLossThreads];
    double acc = 0.0;
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += uint64_t(gridDim.x) * blockDim.x) {
        const double bg = 1.0 - double(opacity[r]);
        // err = color + Vec3{bg, bg, bg} - target (voxmarch.cpp:481-482)
        const double ex = (double(color[3 * r]) + bg) - double(target[3 * r]);
        const double ey = (double(color[3 * r + 1]) + bg) - double(target[3 * r + 1]);
        const double ez = (double(color[3 * r + 2]) + bg) - double(target[3 * r + 2]);
        acc += (ex * ex + ey * ey + ez * ez) * inv;
        dcol[3 * r] = T(ex * (2.0 * inv));
        dcol[3 * r + 1] = T(ey * (2.0 * inv));
        dcol[3 * r + 2] = T(ez * (2.0 * inv));
        dop[r] = T(-2.0 * inv * (ex + ey + ez));
        ddep[r] = T(0.0);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kLossThreads / 2; s > 0; s >>= 1) {  // fixed-order tree
        if (int(threadIdx.x) < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_sum_partials(const double* __restrict__ partial, int n, double* __restrict__ out) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += partial[i];
        *out = s;
    }
}

template <typename T>
__global__ void k_gather_rays(const T* __restrict__ po, const T* __restrict__ pd, const T* __restrict__ pt,
                              const uint32_t* __restrict__ idx, uint64_t n, T* __restrict__ o, T* __restrict__ d,
                              T* __restrict__ t) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t k = idx[i];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            o[3 * i + a] = po[3 * k + a];
            d[3 * i + a] = pd[3 * k + a];
            if (pt) t[3 * i + a] = pt[3 * k + a];
        }
    }
}

}  // namespace
}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_loss_mse_background(vmb_ctx* ctx, const void* color, const void* opacity, const void* targets, uint64_t n,
                            int dtype, void* dcol, void* dop, void* ddep, double* h_loss) {
    if (!n) {
        if (h_loss) *h_loss = 0.0;
        return VMB_OK;
    }
    const int blocks = grid_blocks(ctx, n, kLossThreads, 4);
    double* partial = static_cast<double*>(scratch(ctx, SCRATCH_MISC, size_t(blocks) * 8));
    if (!partial) return VMB_CUDA;
    const double inv = 1.0 / (3.0 * double(n));
    if (dtype == VMB_F32)
        k_loss_mse_bg<float><<<blocks, kLossThreads, 0, ctx->stream>>>(
            static_cast<const float*>(color), static_cast<const float*>(opacity), static_cast<const float*>(targets),
            n, inv, static_cast<float*>(dcol), static_cast<float*>(dop), static_cast<float*>(ddep), partial);
    else
        k_loss_mse_bg<double><<<blocks, kLossThreads, 0, ctx->stream>>>(
            static_cast<const double*>(color), static_cast<const double*>(opacity),
            static_cast<const double*>(targets), n, inv, static_cast<double*>(dcol), static_cast<double*>(dop),
            static_cast<double*>(ddep), partial);
    k_sum_partials<<<1, 32, 0, ctx->stream>>>(partial, blocks, reinterpret_cast<double*>(ctx->d_u64 + 2));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "loss");
    if (h_loss) {
        e = cudaMemcpyAsync(ctx->h_u64 + 2, ctx->d_u64 + 2, 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "loss");
        std::memcpy(h_loss, ctx->h_u64 + 2, 8);
    }
    return VMB_OK;
}

int vmb_gather_rays(vmb_ctx* ctx, const void* po, const void* pd, const void* pt, const uint32_t* idx, uint64_t n,
                    int dtype, void* o, void* d, void* t) {
    if (!n) return VMB_OK;
    const int blocks = grid_blocks(ctx, n, 256, 8);
    if (dtype == VMB_F32)
        k_gather_rays<float><<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const float*>(po), static_cast<const float*>(pd), static_cast<const float*>(pt), idx, n,
            static_cast<float*>(o), static_cast<float*>(d), static_cast<float*>(t));
    else
        k_gather_rays<double><<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const double*>(po), static_cast<const double*>(pd), static_cast<const double*>(pt), idx,
            n, static_cast<double*>(o), static_cast<double*>(d), static_cast<double*>(t));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "gather rays");
}

}  // extern "C"
