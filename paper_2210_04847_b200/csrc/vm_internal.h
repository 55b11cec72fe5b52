// vm_internal.h — library-private state and launcher declarations.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>

#include "../../include/vmb200.h"
#include "vm_exact.cuh"

namespace vmb {

// Device-side error record: the FIRST failure in (ray, sample) / (timestamp, cell)
// order wins via atomicMin on a packed 64-bit key, reproducing the reference's
// "first error in sequential order" exception (parallel.hpp:43-46 rethrows the
// lowest chunk's exception). key == UINT64_MAX means "no error".
struct DevError {
    unsigned long long key;
    int kind;
    int pad_;
};

enum ErrKind : int {
    ERR_NONFINITE_SIGMA = 0,   // ray_marching.cpp:124-126
    ERR_NEGATIVE_SIGMA = 1,    // ray_marching.cpp:127-129
    ERR_NONFINITE_COORD = 2,   // contraction.cpp:25 via query()
    ERR_INVALID_DENSITY = 3,   // occupancy_grid.cpp:127-136
};

// key layout for march errors: ray << 32 | low, low = 0 for a non-finite midpoint
// (candidate generation runs before any density check of that ray in the
// reference, ray_marching.cpp:77-116), else (sample + 1) << 2 | kind.
__host__ __device__ inline unsigned long long march_err_key(uint64_t ray, uint64_t sample, int kind) {
    if (kind == ERR_NONFINITE_COORD) return (unsigned long long)(ray << 32);
    uint64_t s = sample >= 0x3ffffffeull ? 0x3ffffffeull : sample;
    return (unsigned long long)((ray << 32) | ((s + 1) << 2) | uint64_t(kind));
}

int check_contraction(const vmb_contraction* c);

}  // namespace vmb

struct vmb_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    vmb::DevError* d_err = nullptr;     // device error record
    vmb::DevError* h_err = nullptr;     // pinned mirror
    unsigned long long* d_u64 = nullptr;  // 8 device scalars (totals, counters)
    unsigned long long* h_u64 = nullptr;  // pinned mirror
    void* scratch[7] = {};          // per-purpose growable device scratch (see scratch(), SCRATCH_SLOTS)
    size_t scratch_bytes[7] = {};
    cudaEvent_t events[32] = {};
    // NCCL (dlopen'ed lazily; see comm.cpp)
    void* nccl_comm = nullptr;
    int nranks = 1;
    int rank = 0;
};

struct vmb_grid {
    int device = 0;
    uint32_t res = 0;
    vmb_contraction con{};
    vmb::Contract k{};
    double thr = 1e-2;
    double ref_step = 0.0;
    uint64_t n_cells = 0;
    uint64_t n_words = 0;          // ceil(n_cells / 32)
    double* cache = nullptr;       // [n_cells] f64 density EMA
    uint32_t* bits = nullptr;      // [n_words] packed, LSB-first, x-fastest == OGRD bytes
    // Coarse, 1-cell-dilated occupancy used by the empty-space-skipping marcher:
    // bit(K) = OR of fine bits over block K expanded by one fine cell per side.
    uint32_t block = 8;
    uint32_t res_c = 0;            // ceil(res / block)
    uint32_t* coarse = nullptr;    // [ceil(res_c^3 / 32)], built on first use after a change
    bool coarse_valid = false;     // (only the fp64 skip walk, walk_skip, reads it)
    uint64_t coarse_words = 0;
    // Chebyshev (L-inf) distance, in cells, from each cell to the nearest occupied
    // cell, capped at kDistCap (0 = occupied). Lets the marcher jump D-1 cells.
    uint8_t* dist = nullptr;       // [n_cells]
    uint8_t* dist_tmp = nullptr;   // [n_cells] scratch of the separable transform
    // Bounding box of the occupied cells, cell units: {min x, y, z, max x+1, y+1, z+1};
    // min > max - 1 on some axis when no cell is occupied. Rebuilt with the distance map.
    uint32_t* bbox = nullptr;      // [6]
    double* probed = nullptr;      // scratch of the sharded / callback update (probed_words doubles)
    uint64_t probed_words = 0;
};

namespace vmb {

// ---------------------------------------------------------------- utilities
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
// Growable device scratch, one buffer per slot so nested users never alias:
// slot 0 = scan tile sums, 1 = march / candidates temporaries, 2 = grid update,
// 3 = validation / misc. Growing synchronizes the stream before freeing.
enum { SCRATCH_SCAN = 0, SCRATCH_MARCH = 1, SCRATCH_GRID = 2, SCRATCH_MISC = 3, SCRATCH_VOXGRAD = 4, SCRATCH_RENDER = 5, SCRATCH_SLAB = 6, SCRATCH_SLOTS = 7 };
static_assert(sizeof(vmb_ctx::scratch) / sizeof(void*) == SCRATCH_SLOTS, "one scratch buffer per slot");
void* scratch(vmb_ctx* ctx, int slot, size_t bytes);
void zero_words_async(vmb_ctx* ctx, void* p, int n_words);  // runtime.cu
// Programmatic dependent launch (PDL): the kernel may be scheduled while the previous
// kernel on the stream drains (its launch latency hidden behind that kernel's tail);
// every kernel launched this way calls griddep_wait() before touching memory.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#ifdef __CUDACC__
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
#endif

inline int grid_blocks(vmb_ctx* ctx, uint64_t work, int threads, int per_sm = 8) {
    uint64_t b = (work + threads - 1) / threads;
    uint64_t cap = uint64_t(ctx->num_sms) * per_sm;
    return int(b < 1 ? 1 : (b > cap ? cap : b));
}
// Host-side field descriptor checks (Aabb ctor math.hpp:50 for box/voxel boxes,
// TrilinearVoxelField ctor fields.cpp:95-101).
int check_field(const vmb_field* f);
int shade_forward_long(vmb_ctx* ctx, const vmb_rays* rays, const vmb_field* f, double time,
                       const vmb_packed_view* p, void* rgb, void* sig, void* color, void* opacity,
                       void* depth, int dtype);  // render.cu; 1 = not applicable
int backward_listed(vmb_ctx* ctx, const vmb_packed_view* p, const void* rgb, const void* sig, const void* dc,
                    const void* dop, const void* ddep, void* g_rgb, void* g_sig, const uint32_t* list,
                    const unsigned int* n_list, int dtype);  // render.cu: k_backward_long over a ray list
int reset_error(vmb_ctx* ctx);
int read_error(vmb_ctx* ctx, DevError* out);  // synchronizes

// ---------------------------------------------------------------- scan (scan.cu)
// Exclusive scan of u32 counts into u32 offsets; device total (u64) at d_total.
int scan_counts(vmb_ctx* ctx, const uint32_t* counts, uint64_t n, uint32_t* offsets,
                unsigned long long* d_total);
uint64_t scan_onepass_tiles(uint64_t n);  // scan.cu: single-pass scan of the march's chunk totals
int scan_counts_onepass(vmb_ctx* ctx, const uint32_t* counts, uint64_t n, uint32_t* offsets,
                        unsigned long long* d_total, unsigned int* ticket, unsigned long long* status);
// Exclusive scan of u8 flags into u32 positions (compaction), device total at d_total.
int scan_flags(vmb_ctx* ctx, const uint8_t* flags, uint64_t n, uint32_t* pos,
               unsigned long long* d_total);

// Stable LSD radix sort of (u32 key, u32 value) pairs by the low end_bit key bits
// (sort.cu); sorted pairs end in one of the two buffers (*k_res / *v_res).
int radix_sort_pairs(vmb_ctx* ctx, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1, uint64_t m,
                     int end_bit, uint32_t** k_res, uint32_t** v_res);

// ---------------------------------------------------------------- grid (grid.cu)
int grid_refresh(vmb_ctx* ctx, vmb_grid* g);      // bits + coarse from cache
int grid_rebuild_coarse(vmb_ctx* ctx, vmb_grid* g);  // distance map + bbox; invalidates coarse
int grid_ensure_coarse(vmb_ctx* ctx, const vmb_grid* g);  // builds the coarse bits if stale (syncs)
#ifndef VMB_DIST_CAP
#define VMB_DIST_CAP 16
#endif
constexpr int kDistCap = VMB_DIST_CAP;

}  // namespace vmb
