// runtime.cu — context, memory, events, error plumbing, core-type kernels
// (RayBatch validation, pack, validate) and the contraction utilities.
#include <cstdio>
#include <cstring>
#include <string>

#include "vm_internal.h"

namespace vmb {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    g_error = std::string("cuda error in ") + where + ": " + cudaGetErrorString(e);
    return VMB_CUDA;
}

namespace {
__global__ void k_zero_words(uint32_t* __restrict__ p, int n) {
    griddep_wait();
    for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0u;
}
}  // namespace

// A few counters zeroed by a one-warp kernel in the PDL chain (a memset node between
// two kernels would serialise the next kernel's launch behind it).
void zero_words_async(vmb_ctx* ctx, void* p, int n_words) {
    launch_pdl(k_zero_words, dim3(1), dim3(32), 0, ctx->stream, static_cast<uint32_t*>(p), n_words);
}

void* scratch(vmb_ctx* ctx, int slot, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (ctx->scratch_bytes[slot] >= bytes) return ctx->scratch[slot];
    size_t want = bytes + bytes / 4 + 4096;
    if (ctx->scratch[slot]) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(ctx->scratch[slot]);
        ctx->scratch[slot] = nullptr;
        ctx->scratch_bytes[slot] = 0;
    }
    cudaError_t e = cudaMalloc(&ctx->scratch[slot], want);
    if (e != cudaSuccess) {
        cuda_fail(e, "scratch allocation");
        return nullptr;
    }
    ctx->scratch_bytes[slot] = want;
    return ctx->scratch[slot];
}

int reset_error(vmb_ctx* ctx) {
    DevError init{~0ull, -1, 0};
    cudaError_t e = cudaMemcpyAsync(ctx->d_err, &init, sizeof init, cudaMemcpyHostToDevice,
                                    ctx->stream);
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "reset_error");
}

int read_error(vmb_ctx* ctx, DevError* out) {
    cudaError_t e = cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(DevError),
                                    cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "read_error");
    *out = *ctx->h_err;
    return VMB_OK;
}

// ---------------------------------------------------------------- kernels
namespace {

template <typename T>
__global__ void k_rays_validate(const T* __restrict__ o, const T* __restrict__ d, uint64_t n,
                                DevError* err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        D3 a = d3(double(o[3 * i]), double(o[3 * i + 1]), double(o[3 * i + 2]));
        D3 b = d3(double(d[3 * i]), double(d[3 * i + 1]), double(d[3 * i + 2]));
        if (!finite3(a) || !finite3(b)) {
            atomicMin(&err->key, (unsigned long long)(i << 1));
        } else if (fabs(norm(b) - 1.0) > 1e-6) {
            atomicMin(&err->key, (unsigned long long)((i << 1) | 1));
        }
    }
}

__global__ void k_expand_indices(const uint32_t* __restrict__ counts,
                                 const uint32_t* __restrict__ offsets, uint64_t n,
                                 uint32_t* __restrict__ idx) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t o = offsets[r], c = counts[r];
        for (uint32_t k = 0; k < c; ++k) idx[o + k] = uint32_t(r);
    }
}

// validate (core_types.cpp:50-78): each check class reports the smallest failing
// index; the host picks the first class that failed, in the reference's order.
// flags[0]=offset mismatch, [1]=non-positive interval, [2]=per-ray violation key
// (ray << 2 | kind, kind 0 non-monotone, 1 overlapping, 2 partition mismatch).
__global__ void k_validate(const uint32_t* __restrict__ offsets,
                           const uint32_t* __restrict__ counts,
                           const uint32_t* __restrict__ scanned, uint64_t n_rays,
                           const double* __restrict__ ts, const double* __restrict__ te,
                           uint64_t n_samples, const uint32_t* __restrict__ idx,
                           unsigned long long* flags) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (uint64_t r = tid; r < n_rays; r += stride)
        if (offsets[r] != scanned[r]) atomicMin(&flags[0], (unsigned long long)r);
    for (uint64_t s = tid; s < n_samples; s += stride)
        if (!(te[s] > ts[s])) atomicMin(&flags[1], (unsigned long long)s);
    for (uint64_t r = tid; r < n_rays; r += stride) {
        uint64_t b = offsets[r], e = b + counts[r];
        for (uint64_t s = b + 1; s < e; ++s) {
            if (!(ts[s] > ts[s - 1])) { atomicMin(&flags[2], (unsigned long long)((r << 2) | 0)); break; }
            if (ts[s] < te[s - 1]) { atomicMin(&flags[2], (unsigned long long)((r << 2) | 1)); break; }
        }
        for (uint64_t s = b; s < e; ++s)
            if (idx[s] != r) { atomicMin(&flags[2], (unsigned long long)((r << 2) | 2)); break; }
    }
}

__global__ void k_contract(Contract c, const double* __restrict__ x, uint64_t n,
                           double* __restrict__ out, DevError* err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        D3 p = d3(x[3 * i], x[3 * i + 1], x[3 * i + 2]);
        if (!finite3(p)) {
            atomicMin(&err->key, (unsigned long long)i);
            continue;
        }
        D3 g = contract(c, p);
        out[3 * i] = g.x;
        out[3 * i + 1] = g.y;
        out[3 * i + 2] = g.z;
    }
}

__global__ void k_invert(Contract c, const double* __restrict__ g, uint64_t n,
                         double* __restrict__ out, uint8_t* __restrict__ valid) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        D3 w = d3(0.0, 0.0, 0.0);
        bool ok = invert(c, d3(g[3 * i], g[3 * i + 1], g[3 * i + 2]), &w);
        if (!ok) w = d3(0.0, 0.0, 0.0);
        valid[i] = ok;
        out[3 * i] = w.x;
        out[3 * i + 1] = w.y;
        out[3 * i + 2] = w.z;
    }
}

}  // namespace

int check_contraction(const vmb_contraction* c) {
    if (!c) return fail(VMB_INVALID_ARGUMENT, "contraction: null descriptor");
    if (c->kind == VMB_CONTRACT_AABB) {
        if (!(c->box_max[0] > c->box_min[0] && c->box_max[1] > c->box_min[1] &&
              c->box_max[2] > c->box_min[2]))
            return fail(VMB_INVALID_ARGUMENT, "aabb max must be strictly greater than min");
        return VMB_OK;
    }
    if (c->kind == VMB_CONTRACT_SPHERE) {
        if (!(c->radius > 0.0) || !std::isfinite(c->radius) || !std::isfinite(c->center[0]) ||
            !std::isfinite(c->center[1]) || !std::isfinite(c->center[2]))
            return fail(VMB_INVALID_ARGUMENT,
                        "sphere contraction: requires finite center and radius > 0");
        return VMB_OK;
    }
    return fail(VMB_INVALID_ARGUMENT, "contraction: unknown kind");
}

}  // namespace vmb

using namespace vmb;

#define VMB_CUDA_TRY(expr, where)                      \
    do {                                               \
        cudaError_t e_ = (expr);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, where); \
    } while (0)

namespace vmb {
int check_field(const vmb_field* f) {
    if (!f) return fail(VMB_INVALID_ARGUMENT, "field: null");
    const bool boxed = f->kind == VMB_FIELD_UNIFORM_BOX || f->kind == VMB_FIELD_VOXEL;
    if (f->kind == VMB_FIELD_VOXEL && f->vox_resolution < 2)
        return fail(VMB_INVALID_ARGUMENT, "voxel field: resolution must be >= 2 vertices per axis");
    if (boxed && !(f->box_max[0] > f->box_min[0] && f->box_max[1] > f->box_min[1] && f->box_max[2] > f->box_min[2]))
        return fail(VMB_INVALID_ARGUMENT, "aabb max must be strictly greater than min");
    if (f->kind == VMB_FIELD_VOXEL && (!f->vox_density || !f->vox_color))
        return fail(VMB_INVALID_ARGUMENT, "voxel field: parameter arrays required");
    if (f->kind < VMB_FIELD_UNIFORM_BOX || f->kind > VMB_FIELD_VOXEL)
        return fail(VMB_INVALID_ARGUMENT, "field: unknown kind");
    return VMB_OK;
}
}  // namespace vmb

extern "C" {

const char* vmb_last_error(void) { return vmb::g_error.c_str(); }

const char* vmb_version(void) { return "voxmarch_b200 0.1 (sm_100a)"; }

int vmb_device_count(int* n) {
    cudaError_t e = cudaGetDeviceCount(n);
    if (e != cudaSuccess) {
        *n = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return VMB_OK;
}

int vmb_ctx_create(int device, vmb_ctx** out) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(VMB_CUDA, "voxmarch_b200: no CUDA device available (this library has no CPU path)");
    if (device < 0 || device >= n) return fail(VMB_INVALID_ARGUMENT, "voxmarch_b200: bad device index");
    VMB_CUDA_TRY(cudaSetDevice(device), "cudaSetDevice");
    auto* ctx = new vmb_ctx();
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    VMB_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
    ctx->own_stream = true;
    VMB_CUDA_TRY(cudaMalloc(&ctx->d_err, sizeof(DevError)), "cudaMalloc");
    VMB_CUDA_TRY(cudaMallocHost(&ctx->h_err, sizeof(DevError)), "cudaMallocHost");
    VMB_CUDA_TRY(cudaMalloc(&ctx->d_u64, 8 * sizeof(unsigned long long)), "cudaMalloc");
    VMB_CUDA_TRY(cudaMallocHost(&ctx->h_u64, 8 * sizeof(unsigned long long)), "cudaMallocHost");
    for (auto& ev : ctx->events) VMB_CUDA_TRY(cudaEventCreate(&ev), "cudaEventCreate");
    // the async entry points rely on a clean error record from the start
    if (int rc = reset_error(ctx)) return rc;
    VMB_CUDA_TRY(cudaMemsetAsync(ctx->d_u64, 0, 8 * sizeof(unsigned long long), ctx->stream), "cudaMemset");
    VMB_CUDA_TRY(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    *out = ctx;
    return VMB_OK;
}

int vmb_comm_destroy(vmb_ctx* ctx);

int vmb_ctx_destroy(vmb_ctx* ctx) {
    if (!ctx) return VMB_OK;
    cudaSetDevice(ctx->device);
    if (ctx->nccl_comm) vmb_comm_destroy(ctx);
    cudaStreamSynchronize(ctx->stream);
    for (auto& s : ctx->scratch) if (s) cudaFree(s);
    for (auto& ev : ctx->events) if (ev) cudaEventDestroy(ev);
    cudaFree(ctx->d_err);
    cudaFreeHost(ctx->h_err);
    cudaFree(ctx->d_u64);
    cudaFreeHost(ctx->h_u64);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return VMB_OK;
}

static cudaStream_t g_dummy;


int vmb_ctx_set_stream(vmb_ctx* ctx, void* stream) {
    if (ctx->own_stream && stream) {
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        ctx->own_stream = false;
        ctx->stream = static_cast<cudaStream_t>(stream);
    } else if (!stream && !ctx->own_stream) {
        VMB_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "stream");
        ctx->own_stream = true;
    } else if (stream) {
        ctx->stream = static_cast<cudaStream_t>(stream);
    }
    (void)g_dummy;
    return VMB_OK;
}

void* vmb_ctx_stream(vmb_ctx* ctx) { return ctx->stream; }

int vmb_ctx_synchronize(vmb_ctx* ctx) {
    VMB_CUDA_TRY(cudaStreamSynchronize(ctx->stream), "synchronize");
    return VMB_OK;
}

int vmb_malloc(vmb_ctx* ctx, uint64_t bytes, void** out) {
    cudaSetDevice(ctx->device);
    VMB_CUDA_TRY(cudaMalloc(out, bytes ? bytes : 16), "cudaMalloc");
    return VMB_OK;
}

int vmb_free(vmb_ctx* ctx, void* p) {
    if (!p) return VMB_OK;
    cudaStreamSynchronize(ctx->stream);
    VMB_CUDA_TRY(cudaFree(p), "cudaFree");
    return VMB_OK;
}

int vmb_host_alloc(uint64_t bytes, void** out) {
    VMB_CUDA_TRY(cudaMallocHost(out, bytes ? bytes : 16), "cudaMallocHost");
    return VMB_OK;
}

int vmb_host_free(void* p) {
    if (p) VMB_CUDA_TRY(cudaFreeHost(p), "cudaFreeHost");
    return VMB_OK;
}

int vmb_memcpy_h2d(vmb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return VMB_OK;
    VMB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream), "h2d");
    return VMB_OK;
}

int vmb_memcpy_d2h_async(vmb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return VMB_OK;
    VMB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    return VMB_OK;
}

int vmb_memcpy_d2h(vmb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return VMB_OK;
    VMB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    VMB_CUDA_TRY(cudaStreamSynchronize(ctx->stream), "d2h sync");
    return VMB_OK;
}

int vmb_memcpy_d2d(vmb_ctx* ctx, void* dst, const void* src, uint64_t bytes) {
    if (!bytes) return VMB_OK;
    VMB_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream), "d2d");
    return VMB_OK;
}

int vmb_memset(vmb_ctx* ctx, void* dst, int value, uint64_t bytes) {
    if (!bytes) return VMB_OK;
    VMB_CUDA_TRY(cudaMemsetAsync(dst, value, bytes, ctx->stream), "memset");
    return VMB_OK;
}

int vmb_event_record(vmb_ctx* ctx, int slot) {
    if (slot < 0 || slot >= 32) return fail(VMB_INVALID_ARGUMENT, "event slot out of range");
    VMB_CUDA_TRY(cudaEventRecord(ctx->events[slot], ctx->stream), "cudaEventRecord");
    return VMB_OK;
}

int vmb_ctx_wait(vmb_ctx* waiter, vmb_ctx* on, int slot) {
    if (!waiter || !on) return fail(VMB_INVALID_ARGUMENT, "null context");
    if (slot < 0 || slot >= 32) return fail(VMB_INVALID_ARGUMENT, "event slot out of range");
    if (waiter == on || waiter->stream == on->stream) return VMB_OK;
    VMB_CUDA_TRY(cudaEventRecord(on->events[slot], on->stream), "cudaEventRecord");
    VMB_CUDA_TRY(cudaStreamWaitEvent(waiter->stream, on->events[slot], 0), "cudaStreamWaitEvent");
    return VMB_OK;
}

// CUDA graphs of a context's stream: everything enqueued between begin and end
// (kernels, memsets, copies of the async entry points) becomes one graph that
// replays with a single launch — the launch-bound small batches (config 1).
int vmb_graph_begin(vmb_ctx* ctx) {
    VMB_CUDA_TRY(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    return VMB_OK;
}

int vmb_graph_end(vmb_ctx* ctx, void** h_graph) {
    cudaGraph_t g = nullptr;
    VMB_CUDA_TRY(cudaStreamEndCapture(ctx->stream, &g), "cudaStreamEndCapture");
    cudaGraphExec_t x = nullptr;
    cudaError_t e = cudaGraphInstantiate(&x, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
    *h_graph = x;
    return VMB_OK;
}

int vmb_graph_launch(vmb_ctx* ctx, void* graph) {
    VMB_CUDA_TRY(cudaGraphLaunch(static_cast<cudaGraphExec_t>(graph), ctx->stream), "cudaGraphLaunch");
    return VMB_OK;
}

int vmb_graph_destroy(void* graph) {
    if (graph) VMB_CUDA_TRY(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(graph)), "cudaGraphExecDestroy");
    return VMB_OK;
}

int vmb_event_elapsed_ms(vmb_ctx* ctx, int a, int b, float* ms) {
    if (a < 0 || a >= 32 || b < 0 || b >= 32) return fail(VMB_INVALID_ARGUMENT, "event slot out of range");
    VMB_CUDA_TRY(cudaEventSynchronize(ctx->events[b]), "cudaEventSynchronize");
    VMB_CUDA_TRY(cudaEventElapsedTime(ms, ctx->events[a], ctx->events[b]), "cudaEventElapsedTime");
    return VMB_OK;
}

int vmb_shard_range(uint64_t n, int nranks, int rank, uint64_t* begin, uint64_t* end) {
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(VMB_INVALID_ARGUMENT, "shard: rank out of range");
    // parallel.hpp:28-35: chunks = min(workers, n); per = ceil(n / chunks)
    uint64_t chunks = uint64_t(nranks) < n ? uint64_t(nranks) : n;
    if (chunks == 0) {
        *begin = *end = 0;
        return VMB_OK;
    }
    uint64_t per = (n + chunks - 1) / chunks;
    uint64_t b = uint64_t(rank) * per;
    uint64_t e = b + per;
    if (b > n) b = n;
    if (e > n) e = n;
    *begin = b;
    *end = e;
    return VMB_OK;
}

int vmb_rays_validate(vmb_ctx* ctx, const vmb_rays* rays) {
    if (!(rays->near_plane >= 0.0) || !(rays->far_plane > rays->near_plane))
        return fail(VMB_INVALID_ARGUMENT, "ray batch: requires far > near >= 0");
    if (rays->n_rays == 0) return VMB_OK;
    int rc = reset_error(ctx);
    if (rc) return rc;
    int blocks = grid_blocks(ctx, rays->n_rays, 256);
    if (rays->dtype == VMB_F32)
        k_rays_validate<float><<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const float*>(rays->d_origins), static_cast<const float*>(rays->d_directions),
            rays->n_rays, ctx->d_err);
    else
        k_rays_validate<double><<<blocks, 256, 0, ctx->stream>>>(
            static_cast<const double*>(rays->d_origins),
            static_cast<const double*>(rays->d_directions), rays->n_rays, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull) {
        uint64_t i = err.key >> 1;
        return fail(VMB_INVALID_ARGUMENT, std::string(err.key & 1 ? "ray batch: non-unit direction at index "
                                                                  : "ray batch: non-finite ray at index ") +
                                              std::to_string(i));
    }
    return VMB_OK;
}

uint64_t vmb_uniform_step_count(double near_plane, double far_plane, double step) {
    return vmb::uniform_step_count(near_plane, far_plane, step);
}

int vmb_pack(vmb_ctx* ctx, const uint32_t* counts, uint64_t n, uint32_t* offsets,
             uint32_t* ray_indices, uint64_t capacity, uint64_t* total) {
    if (n > 0xffffffffull)
        return fail(VMB_INVALID_ARGUMENT, "pack: ray count exceeds 32-bit index range");
    int rc = scan_counts(ctx, counts, n, offsets, ctx->d_u64);
    if (rc) return rc;
    VMB_CUDA_TRY(cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    VMB_CUDA_TRY(cudaStreamSynchronize(ctx->stream), "pack sync");
    *total = ctx->h_u64[0];
    if (*total > 0xffffffffull)
        return fail(VMB_INVALID_ARGUMENT, "pack: sample count exceeds 32-bit index range");
    if (ray_indices) {
        if (*total > capacity) return fail(VMB_CAPACITY, "pack: ray_indices capacity too small");
        if (n) k_expand_indices<<<grid_blocks(ctx, n, 256), 256, 0, ctx->stream>>>(counts, offsets, n, ray_indices);
        VMB_CUDA_TRY(cudaGetLastError(), "pack expand");
    }
    return VMB_OK;
}

int vmb_validate(vmb_ctx* ctx, const vmb_packed_view* p, const uint32_t* idx, uint64_t n_offsets,
                 uint64_t n_idx, uint64_t n_te, int* result) {
    // length checks (core_types.cpp:51-56) need the counts total
    if (n_offsets != p->n_rays) { *result = 1; return VMB_OK; }
    auto* tmp = static_cast<uint32_t*>(scratch(ctx, SCRATCH_MISC, (p->n_rays + 1) * sizeof(uint32_t) + 64));
    if (!tmp) return VMB_CUDA;
    int rc = scan_counts(ctx, p->d_counts, p->n_rays, tmp, ctx->d_u64);
    if (rc) return rc;
    VMB_CUDA_TRY(cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 8, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    VMB_CUDA_TRY(cudaStreamSynchronize(ctx->stream), "validate sync");
    uint64_t total = ctx->h_u64[0];
    if (total != p->n_samples || total != n_te || total != n_idx) { *result = 1; return VMB_OK; }
    unsigned long long init[3] = {~0ull, ~0ull, ~0ull};
    VMB_CUDA_TRY(cudaMemcpyAsync(ctx->d_u64 + 1, init, sizeof init, cudaMemcpyHostToDevice, ctx->stream), "h2d");
    uint64_t work = p->n_rays > p->n_samples ? p->n_rays : p->n_samples;
    if (work)
        k_validate<<<grid_blocks(ctx, work, 256), 256, 0, ctx->stream>>>(
            p->d_offsets, p->d_counts, tmp, p->n_rays, p->d_t_starts, p->d_t_ends, p->n_samples,
            idx, ctx->d_u64 + 1);
    VMB_CUDA_TRY(cudaMemcpyAsync(ctx->h_u64 + 1, ctx->d_u64 + 1, sizeof init, cudaMemcpyDeviceToHost, ctx->stream), "d2h");
    VMB_CUDA_TRY(cudaStreamSynchronize(ctx->stream), "validate sync");
    const unsigned long long* f = ctx->h_u64 + 1;
    if (f[0] != ~0ull) *result = 2;
    else if (f[1] != ~0ull) *result = 3;
    else if (f[2] != ~0ull) *result = 4 + int(f[2] & 3);
    else *result = 0;
    return VMB_OK;
}

int vmb_contract(vmb_ctx* ctx, const vmb_contraction* c, const double* x, uint64_t n, double* out) {
    int rc = check_contraction(c);
    if (rc) return rc;
    if (!n) return VMB_OK;
    rc = reset_error(ctx);
    if (rc) return rc;
    k_contract<<<grid_blocks(ctx, n, 256), 256, 0, ctx->stream>>>(make_contract(*c), x, n, out, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull) return fail(VMB_INVALID_ARGUMENT, "non-finite coordinate");
    return VMB_OK;
}

int vmb_invert_grid_point(vmb_ctx* ctx, const vmb_contraction* c, const double* g, uint64_t n,
                          double* out, uint8_t* valid) {
    int rc = check_contraction(c);
    if (rc) return rc;
    if (!n) return VMB_OK;
    k_invert<<<grid_blocks(ctx, n, 256), 256, 0, ctx->stream>>>(make_contract(*c), g, n, out, valid);
    VMB_CUDA_TRY(cudaGetLastError(), "invert");
    return VMB_OK;
}

}  // extern "C"
