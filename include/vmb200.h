/*
 * vmb200.h — C ABI of the B200-native volumetric-rendering hot path
 * (library: paper_2210_04847_b200/lib/libvoxmarch_b200.so, sm_100a).
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (voxmarch, /root/reference/proj) has no plugin registry: its boundary is the
 * public C++ headers in namespace voxmarch. Each entry point below
 * names the reference function it replaces; include/voxmarch/voxmarch.hpp is
 * the C++ facade that restores the reference's exact signatures, value types
 * and exception messages on top of these calls.
 *
 * Conventions
 *  - Plain pointers + sizes only. Pointers named d_* are DEVICE pointers (from
 *    vmb_malloc or any CUDA allocation on the context's device); h_* are host.
 *  - Every call returns a VMB_* status (vmb200_types.h); vmb_last_error()
 *    returns the thread-local message, which for VMB_INVALID_ARGUMENT and
 *    VMB_RUNTIME equals the reference's exception text byte for byte.
 *  - Work is enqueued on the context's CUDA stream. Calls that return a host
 *    value computed on the device (totals, error checks) synchronize that stream.
 *  - Packed samples use the reference layout (core_types.hpp:29-38): offsets,
 *    counts (u32, per ray), t_starts, t_ends (f64, per sample), ray_indices (u32).
 *  - Ray origins/directions are AoS xyz (like std::vector<Vec3>) in f32 or f64
 *    (vmb_rays.dtype); attribute / output arrays are f32 or f64 (dtype args).
 *    All arithmetic is fp64 regardless.
 *  - n_threads of the reference API has no equivalent: results never depend on
 *    the launch configuration (the reference's determinism contract, parallel.hpp:17-19).
 */
#ifndef VMB200_H
#define VMB200_H

#include "vmb200_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vmb_ctx vmb_ctx;   /* device, stream, scratch, error record, optional NCCL comm */
typedef struct vmb_grid vmb_grid; /* device-resident OccupancyGrid */

/* Ray batch on the device; replaces voxmarch::RayBatch (core_types.hpp:15-25). */
typedef struct vmb_rays {
    const void* d_origins;    /* [n_rays][3] */
    const void* d_directions; /* [n_rays][3], unit length */
    int32_t dtype;            /* VMB_F32 | VMB_F64 */
    int32_t pad_;
    uint64_t n_rays;
    double near_plane;
    double far_plane;
} vmb_rays;

/* Caller-owned output of march(); replaces voxmarch::PackedSamples. */
typedef struct vmb_samples {
    uint32_t* d_offsets;      /* [n_rays] */
    uint32_t* d_counts;       /* [n_rays] */
    double* d_t_starts;       /* [capacity] */
    double* d_t_ends;         /* [capacity] */
    uint32_t* d_ray_indices;  /* [capacity] */
    uint64_t capacity;
} vmb_samples;

/* Read-only view of packed samples (input of the rendering calls). */
typedef struct vmb_packed_view {
    const uint32_t* d_offsets;
    const uint32_t* d_counts;
    uint64_t n_rays;
    const double* d_t_starts;
    const double* d_t_ends;
    uint64_t n_samples;
} vmb_packed_view;

/* ------------------------------------------------------------------ runtime */
const char* vmb_last_error(void);
const char* vmb_version(void);
int vmb_device_count(int* h_count);
int vmb_ctx_create(int device, vmb_ctx** out);
int vmb_ctx_destroy(vmb_ctx* ctx);
int vmb_ctx_set_stream(vmb_ctx* ctx, void* cuda_stream); /* NULL restores the owned stream */
void* vmb_ctx_stream(vmb_ctx* ctx);
int vmb_ctx_synchronize(vmb_ctx* ctx);
int vmb_malloc(vmb_ctx* ctx, uint64_t bytes, void** d_out);
int vmb_free(vmb_ctx* ctx, void* d_ptr);
int vmb_host_alloc(uint64_t bytes, void** h_out); /* pinned */
int vmb_host_free(void* h_ptr);
int vmb_memcpy_h2d(vmb_ctx* ctx, void* d_dst, const void* h_src, uint64_t bytes);
int vmb_memcpy_d2h(vmb_ctx* ctx, void* h_dst, const void* d_src, uint64_t bytes);
/* Stream-ordered d2h into pinned memory without waiting: the data is valid after
 * vmb_ctx_synchronize (or an event). vmb_memcpy_d2h waits. */
int vmb_memcpy_d2h_async(vmb_ctx* ctx, void* h_dst, const void* d_src, uint64_t bytes);
int vmb_memcpy_d2d(vmb_ctx* ctx, void* d_dst, const void* d_src, uint64_t bytes);
int vmb_memset(vmb_ctx* ctx, void* d_dst, int value, uint64_t bytes);
/* CUDA events on the context stream (slot 0..31) for device-side timing. */
int vmb_event_record(vmb_ctx* ctx, int slot);
int vmb_event_elapsed_ms(vmb_ctx* ctx, int slot_begin, int slot_end, float* h_ms);
/* Make waiter's stream wait for the work queued so far on `on`'s stream (records
 * on's event `slot`). Lets several contexts on one device pipeline host<->device
 * copies against compute, each context being one CUDA stream. */
int vmb_ctx_wait(vmb_ctx* waiter, vmb_ctx* on, int slot);
/* CUDA graph capture of the context's stream: the calls between begin and end
 * must be asynchronous (the *_async march entry points, render_*, memcpy_*_async)
 * and their scratch already grown by one uncaptured call; end instantiates the
 * graph (an opaque handle), launch replays it on the stream. */
int vmb_graph_begin(vmb_ctx* ctx);
int vmb_graph_end(vmb_ctx* ctx, void** h_graph);
int vmb_graph_launch(vmb_ctx* ctx, void* graph);
int vmb_graph_destroy(void* graph);
/* Host-only helper (no device work): the contiguous shard of n units owned by
 * rank — the static split of parallel_for (parallel.hpp:28-35). */
int vmb_shard_range(uint64_t n, int nranks, int rank, uint64_t* h_begin, uint64_t* h_end);

/* ------------------------------------------------------------------ core types */
/* RayBatch::create validation (core_types.cpp:9-28): finite rays, |d|-1 <= 1e-6,
 * far > near >= 0. Synchronizes; the first offending ray is reported. */
int vmb_rays_validate(vmb_ctx* ctx, const vmb_rays* rays);
/* ------------------------------------------------------------------ cameras
 * validate_camera (scene_camera.cpp:10-23), look_at (:25-44): host-only, exact
 * fp64 as the reference. generate_rays (:46-63): one ray per pixel centre,
 * row-major, unit directions, written on the device into caller buffers of
 * width*height*3 elements (dtype VMB_F32/VMB_F64; directions are computed in
 * fp64 and rounded once). Fills *out_rays (near/far as given) when non-null;
 * the batch satisfies RayBatch::create's checks by construction. */
int vmb_camera_validate(const vmb_camera* camera);
int vmb_camera_look_at(const double eye[3], const double target[3], const double up[3], double focal,
                       int32_t width, int32_t height, vmb_camera* out);
int vmb_generate_rays(vmb_ctx* ctx, const vmb_camera* camera, double near_plane, double far_plane,
                      int dtype, void* d_origins, void* d_directions, vmb_rays* out_rays);
/* Rays of pixels [first_ray, first_ray + n_rays) (row-major) only: a chunk of the
 * image, for pipelined steps. */
int vmb_generate_rays_range(vmb_ctx* ctx, const vmb_camera* camera, double near_plane, double far_plane,
                            int dtype, uint64_t first_ray, uint64_t n_rays, void* d_origins, void* d_directions,
                            vmb_rays* out_rays);

/* ------------------------------------------------------------------ fields
 * query_density / query_rgb_sigma for any field kind (fields.cpp:75-93 and the
 * TrilinearVoxelField versions :142-168), at p - velocity*time: d_points [n][3]
 * f64 -> d_sigmas [n] (+ d_rgbs [n][3] when non-null), f64. Non-finite positions
 * fail with "field: non-finite position at index i" (first i).
 * TrilinearVoxelField::backward (fields.cpp:170-211): accumulates the parameter
 * gradient of the query chain into d_accum_density [R^3] / d_accum_color
 * [R^3][3] (f64, device); gradients d_rgb_grads [n][3] / d_sigma_grads [n] in
 * dtype. The _samples form takes the positions as packed-sample midpoints
 * o + d*(0.5*(t0+t1)) of `rays` (voxmarch.cpp:243-244). mode: VMB_GRAD_*. */
int vmb_field_query(vmb_ctx* ctx, const vmb_field* field, const double* d_points, uint64_t n, double time,
                    double* d_sigmas, double* d_rgbs);
int vmb_voxel_field_backward(vmb_ctx* ctx, const vmb_field* field, const double* d_points, uint64_t n,
                             const void* d_rgb_grads, const void* d_sigma_grads, int dtype,
                             double* d_accum_density, double* d_accum_color, int mode);
int vmb_voxel_field_backward_samples(vmb_ctx* ctx, const vmb_field* field, const vmb_rays* rays,
                                     const uint32_t* d_ray_indices, const double* d_t_starts,
                                     const double* d_t_ends, uint64_t n_samples, double time,
                                     const void* d_rgb_grads, const void* d_sigma_grads, int dtype,
                                     double* d_accum_density, double* d_accum_color, int mode);

/* AdamOptimizer::step (fields.cpp:279-292) on device arrays of n doubles; step =
 * the optimizer's step count t after increment (bias corrections 1 - beta^t).
 * A non-finite gradient fails with "adam: non-finite gradient at index i"
 * (VMB_RUNTIME) before anything is updated. */
int vmb_adam_step(vmb_ctx* ctx, uint64_t n, double* d_params, const double* d_grads, double* d_m, double* d_v,
                  double lr, double beta1, double beta2, double eps, uint64_t step);

/* uniform_step_count (ray_marching.cpp:51-55). Host-only. */
uint64_t vmb_uniform_step_count(double near_plane, double far_plane, double step_size);
/* pack (core_types.cpp:30-48): exclusive scan of counts + ray index expansion.
 * Synchronizes to return the total; d_ray_indices may be NULL (scan only). */
int vmb_pack(vmb_ctx* ctx, const uint32_t* d_counts, uint64_t n_rays, uint32_t* d_offsets,
             uint32_t* d_ray_indices, uint64_t capacity, uint64_t* h_total);
/* validate (core_types.cpp:50-78): 0 = consistent, else 1..6 = length mismatch,
 * offset mismatch, non-positive interval, non-monotone t_starts, overlapping
 * intervals, partition mismatch (first violated invariant in the reference's order). */
int vmb_validate(vmb_ctx* ctx, const vmb_packed_view* packed, const uint32_t* d_ray_indices,
                 uint64_t n_offsets, uint64_t n_ray_indices, uint64_t n_t_ends, int* h_result);

/* ------------------------------------------------------------------ contraction */
/* contract / invert_grid_point (contraction.cpp:24-47) over device point arrays. */
int vmb_contract(vmb_ctx* ctx, const vmb_contraction* c, const double* d_points, uint64_t n,
                 double* d_out);
int vmb_invert_grid_point(vmb_ctx* ctx, const vmb_contraction* c, const double* d_points,
                          uint64_t n, double* d_out, uint8_t* d_valid);

/* ------------------------------------------------------------------ occupancy grid */
/* OccupancyGrid ctor (occupancy_grid.cpp:41-56). */
int vmb_grid_create(vmb_ctx* ctx, uint32_t resolution, const vmb_contraction* c,
                    double alpha_threshold, double reference_step, double initial_density,
                    vmb_grid** out);
int vmb_grid_destroy(vmb_grid* g);
int vmb_grid_clone(vmb_ctx* ctx, const vmb_grid* src, vmb_grid** out);
int vmb_grid_info(const vmb_grid* g, uint32_t* h_resolution, vmb_contraction* h_contraction,
                  double* h_alpha_threshold, double* h_reference_step,
                  double* h_threshold_density);
/* update / update_over_time with a device-evaluable analytic field
 * (occupancy_grid.cpp:91-144; density_batch voxmarch.cpp:211-219; time shift
 * fields.cpp:264-266). With a communicator attached (vmb_comm_init) each rank
 * probes its shard of cells and the probes are combined with ncclAllReduce(max)
 * before the EMA; the resulting grid is bit-identical for any rank count. */
int vmb_grid_update_field(vmb_ctx* ctx, vmb_grid* g, const vmb_field* f,
                          const double* h_timestamps, uint64_t n_timestamps, double ema_decay,
                          int has_seed, uint64_t seed);
/* The probe half of vmb_grid_update_field for cells [cell_begin, cell_end) only
 * (occupancy_grid.cpp:106-140): d_probed (n_cells f64) receives the max density
 * over timestamps for those cells and 0 everywhere else. This is what each rank
 * contributes to the all-reduce(max) of a multi-GPU update; combining the ranks'
 * buffers with max and calling vmb_grid_apply reproduces the single-GPU grid. */
int vmb_grid_probe_field_range(vmb_ctx* ctx, const vmb_grid* g, const vmb_field* f,
                               const double* h_timestamps, uint64_t n_timestamps, int has_seed,
                               uint64_t seed, uint64_t cell_begin, uint64_t cell_end,
                               double* d_probed);
/* Generic host-callback update, step 1: probe points of all invertible cells in
 * cell order (occupancy_grid.cpp:108-119). d_points needs 3*n_cells doubles,
 * d_cells n_cells u32. Synchronizes to return the count. */
int vmb_grid_probe_points(vmb_ctx* ctx, const vmb_grid* g, int has_seed, uint64_t seed,
                          double* d_points, uint32_t* d_cells, uint64_t* h_count);
/* step 2 (per timestamp): validate densities and fold them into the running
 * max (occupancy_grid.cpp:121-140). d_probed (n_cells f64) must start zeroed.
 * Synchronizes; an invalid density yields VMB_RUNTIME with the reference text. */
int vmb_grid_accumulate(vmb_ctx* ctx, const vmb_grid* g, const double* d_densities,
                        const uint32_t* d_cells, uint64_t n, double* d_probed);
/* step 3: cache = max(cache*decay, probed); refresh bits (occupancy_grid.cpp:142-143).
 * With a communicator attached, d_probed is first all-reduced (max) across ranks. */
int vmb_grid_apply(vmb_ctx* ctx, vmb_grid* g, double* d_probed, double ema_decay);
/* seed_occupancy (occupancy_grid.cpp:152-165) from a per-cell mask (u8, cell order). */
int vmb_grid_seed_mask(vmb_ctx* ctx, vmb_grid* g, const uint8_t* d_mask);
/* occupied_fraction numerator (occupancy_grid.cpp:146-150). Synchronizes. */
int vmb_grid_occupied_count(vmb_ctx* ctx, const vmb_grid* g, uint64_t* h_count);
/* query (occupancy_grid.cpp:67-76) for n device points; d_out u8. Synchronizes to
 * report a non-finite point ("non-finite coordinate", contraction.cpp:25). */
int vmb_grid_query(vmb_ctx* ctx, const vmb_grid* g, const double* d_points, uint64_t n,
                   uint8_t* d_out);
/* Host copies of the state: h_bits is the OGRD bit section (ceil(n_cells/8) bytes,
 * LSB-first, x-fastest; occupancy_grid.cpp:197-204) — identical to the device
 * layout, so save/load are plain copies. Either pointer may be NULL. */
int vmb_grid_read(vmb_ctx* ctx, const vmb_grid* g, uint8_t* h_bits, double* h_cache);
int vmb_grid_write(vmb_ctx* ctx, vmb_grid* g, const uint8_t* h_bits, const double* h_cache);
/* The marcher's acceleration structure (not in the reference): per cell the L-inf
 * distance in cells to the nearest occupied cell, capped (*h_cap), u8 [n_cells]. */
int vmb_grid_read_distance(vmb_ctx* ctx, const vmb_grid* g, uint8_t* h_dist, uint32_t* h_cap);
/* The marcher's ray clip box (not in the reference): bounding box of the occupied
 * cells in cell units, h_box = {min x, y, z, max x + 1, y + 1, z + 1}; min >= max on
 * an axis when no cell is occupied. */
int vmb_grid_occupied_bbox(vmb_ctx* ctx, const vmb_grid* g, uint32_t* h_box);
const uint32_t* vmb_grid_device_bits(const vmb_grid* g);
const double* vmb_grid_device_cache(const vmb_grid* g);

/* ------------------------------------------------------------------ ray marching */
/* march() with the density of a device-evaluable analytic field at each midpoint
 * (ray_marching.cpp:57-150 with sigma_fn_for, voxmarch.cpp:221-232). Fused:
 * lattice traversal with empty-space skipping, grid test, inline density,
 * alpha floor, transmittance cut, packing. Output is bit-identical to the
 * reference. Synchronizes to return h_n_samples; if out->capacity is smaller,
 * offsets/counts are still written, no samples are, and VMB_CAPACITY is
 * returned with *h_n_samples set (call again with a larger buffer).
 * h_stats may be NULL (then samples_emitted is not computed). */
int vmb_march_field(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays, const vmb_field* f,
                    const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n_samples,
                    vmb_march_stats* h_stats);
/* vmb_march_field + vmb_shade_field fused: while the kept samples are packed,
 * the field's rgb and sigma at each sample's midpoint (shade_samples,
 * voxmarch.cpp:235-251, with the TimeConditionedField shift at `time`) are
 * written to d_rgbs [capacity][3] / d_sigmas [capacity] in `dtype`. Same capacity
 * protocol as vmb_march_field (the attribute buffers need the same capacity). */
int vmb_march_field_shaded(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                           const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out,
                           void* d_rgbs, void* d_sigmas, int dtype, double time,
                           uint64_t* h_n_samples, vmb_march_stats* h_stats);
/* march + shading + render_forward fused (the forward half of a training step, or
 * inference rendering, with an analytic field): additionally writes the per-ray
 * color [n_rays][3], opacity and depth of render_forward (rendering.cpp:35-65)
 * over the kept samples with the shaded (dtype-rounded) attributes — bit-identical
 * to vmb_march_field_shaded followed by vmb_render_forward, without re-reading the
 * packed samples. */
int vmb_march_render_field(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                           const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out,
                           void* d_rgbs, void* d_sigmas, void* d_color, void* d_opacity,
                           void* d_depth, int dtype, double time, uint64_t* h_n_samples,
                           vmb_march_stats* h_stats);
/* Asynchronous variant for training loops / CUDA graphs: no host round trip.
 * The sample total is written to d_n_samples (u64, device); samples beyond
 * out->capacity are dropped (check d_n_samples afterwards). Errors (negative or
 * non-finite density) are recorded on the device and reported by the next
 * vmb_march_check(). */
int vmb_march_field_async(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                          const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out,
                          uint64_t* d_n_samples);
/* Asynchronous vmb_march_render_field (same contract as vmb_march_field_async);
 * where the fused single pass does not apply (time-shifted fields, growth
 * lattices) it runs the synchronous path and then publishes the total. */
int vmb_march_render_field_async(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays, const vmb_field* f,
                                 const vmb_march_config* cfg, vmb_samples* out, void* d_rgbs, void* d_sigmas,
                                 void* d_color, void* d_opacity, void* d_depth, int dtype, double time,
                                 uint64_t* d_n_samples);
/* The training step in one call: vmb_march_render_field_async's outputs plus
 * render_backward (rendering.cpp:67-112) of them for the upstream gradients
 * d_grad_color [n_rays][3] / d_grad_opacity / d_grad_depth -> d_grad_rgbs
 * [capacity][3] / d_grad_sigmas, computed by the expansion from the samples it has
 * just produced (no re-read). Gradients agree with vmb_render_backward on the same
 * outputs within the rendering tolerance (scans reassociate the T products and
 * suffix sums); packing, shading and the forward are identical. */
int vmb_march_render_backward_field_async(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                                          const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out,
                                          void* d_rgbs, void* d_sigmas, void* d_color, void* d_opacity,
                                          void* d_depth, const void* d_grad_color, const void* d_grad_opacity,
                                          const void* d_grad_depth, void* d_grad_rgbs, void* d_grad_sigmas,
                                          int dtype, double time, uint64_t* d_n);
int vmb_march_check(vmb_ctx* ctx);
/* Generic host-SigmaFn path, step 1: the grid-passing candidate intervals of every
 * ray, capped at max_samples_per_ray (ray_marching.cpp:75-106). Same two-call
 * capacity protocol as vmb_march_field. */
int vmb_march_candidates(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                         const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n);
/* step 2: given one sigma per candidate (d_sigmas, dtype f64), apply the
 * validation, alpha floor and transmittance cut per ray (ray_marching.cpp:118-137)
 * and pack the kept samples. Reports the first invalid density in (ray, sample)
 * order with the reference's message. */
int vmb_march_filter(vmb_ctx* ctx, const vmb_packed_view* candidates, const double* d_sigmas,
                     const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n);
/* march_uniform (ray_marching.cpp:152-168). */
int vmb_march_uniform(vmb_ctx* ctx, const vmb_rays* rays, const vmb_march_config* cfg,
                      vmb_samples* out, uint64_t* h_n);

/* ------------------------------------------------------------------ multi-level grid + cone stepping
 * NerfAcc's cascaded occupancy grid and cone-step sampling (reference non-goals,
 * SPEC.md:215,276). Level 0 is the call's grid (any contraction);
 * levels[0..n_levels) are AABB grids, each strictly containing the one below
 * (vmb_cascade_level_box: level 0's box scaled by 2^l about its center). A point is
 * decided by the FINEST level whose domain contains it, with that level's own
 * OccupancyGrid::query (occupancy_grid.cpp:67-76); each level is updated with the
 * grid API. With n_levels = 0 and cone = 0 the marcher is march() (A13/A14)
 * exactly. cone != 0: the interval starting at t has width
 * dt = min(max(t * cone_angle, step_size), max_step) and t accumulates (t += dt,
 * the growth walk's arithmetic, ray_marching.cpp:88-106); growth > 1 and cone are
 * exclusive. Stacked levels / cone take the accumulated-t walk (count -> scan ->
 * fill), which ends a ray once its midpoint has left the outermost AABB level. */
typedef struct vmb_march_ext {
    const vmb_grid* const* levels; /* levels above level 0, finest first */
    uint32_t n_levels;             /* <= 7 */
    int32_t cone;                  /* 1: cone stepping */
    double cone_angle;
    double max_step;               /* >= step_size */
} vmb_march_ext;
int vmb_cascade_level_box(const vmb_contraction* base, uint32_t level, vmb_contraction* out);
int vmb_cascade_query(vmb_ctx* ctx, const vmb_grid* level0, const vmb_march_ext* ext, const double* d_points,
                      uint64_t n, uint8_t* d_occupied);
int vmb_march_cascade(vmb_ctx* ctx, const vmb_grid* level0, const vmb_march_ext* ext, const vmb_rays* rays,
                      const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n,
                      vmb_march_stats* stats);
/* + analytic shading and render_forward (the vmb_march_render_field outputs). */
int vmb_march_render_cascade(vmb_ctx* ctx, const vmb_grid* level0, const vmb_march_ext* ext,
                             const vmb_rays* rays, const vmb_field* f, const vmb_march_config* cfg,
                             vmb_samples* out, void* d_rgbs, void* d_sigmas, void* d_color, void* d_opacity,
                             void* d_depth, int dtype, double time, uint64_t* h_n, vmb_march_stats* stats);

/* ------------------------------------------------------------------ shading (harness) */
/* shade_samples (voxmarch.cpp:235-251) for an analytic field (+time shift):
 * rgb and sigma at each sample midpoint, written as dtype. */
int vmb_shade_field(vmb_ctx* ctx, const vmb_rays* rays, const vmb_field* f, double time,
                    const uint32_t* d_ray_indices, const double* d_t_starts,
                    const double* d_t_ends, uint64_t n_samples, void* d_rgbs, void* d_sigmas,
                    int dtype);

/* ------------------------------------------------------------------ rendering */
/* Per-sample outputs (transmittance, render_backward) are written only at samples
 * inside some ray's [offset, offset + count): the buffers are caller-owned, so a
 * pack whose rays do not cover [0, n_samples) leaves the other positions as they
 * were. The reference returns zero-initialised vectors (rendering.cpp:22, 78-79);
 * the C++ facade and the Python binding zero the buffers first to match it. */
/* transmittance (rendering.cpp:19-33): exclusive per-ray T, out [n_samples]. */
int vmb_transmittance(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_sigmas,
                      void* d_out, int dtype);
/* render_forward (rendering.cpp:35-65): color [n_rays][3], opacity, depth. */
int vmb_render_forward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_rgbs,
                       const void* d_sigmas, void* d_color, void* d_opacity, void* d_depth,
                       int dtype);
/* render_backward (rendering.cpp:67-112): d_rgbs [n_samples][3], d_sigmas. */
int vmb_render_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_rgbs,
                        const void* d_sigmas, const void* d_color, const void* d_opacity,
                        const void* d_depth, void* d_rgbs_grad, void* d_sigmas_grad,
                        int dtype);
/* render_attribute (rendering.cpp:114-134): out [n_rays][dim]. */
int vmb_render_attribute(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_sigmas,
                         const void* d_values, uint64_t dim, void* d_out, int dtype);

/* ------------------------------------------------------------------ NerfAcc operators
 * Standalone forms of the compositing the reference performs inside render_forward /
 * render_backward (rendering.cpp:47-58, 67-112) — the north_star's
 * render_weight_from_density / render_transmittance_from_alpha (+ backward),
 * accumulate_along_rays and ray_aabb_intersect. Per-sample arrays are [n_samples]
 * (values [n_samples][dim]) in dtype; every output and every upstream-gradient
 * pointer may be NULL (not written / taken as 0). Results agree with the
 * reference's sequential order within rtol 1e-5 (warp-shuffle segmented scans
 * reassociate the products and sums; in practice a few ulps). */
/* alpha = 1 - exp(-sigma (t_end - t_start)), trans = exclusive prod (1 - alpha),
 * weights = trans * alpha (rendering.cpp:47-58 order of operations per sample). */
int vmb_render_weight_from_density(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_sigmas,
                                   void* d_weights, void* d_trans, void* d_alphas, int dtype);
/* d_grad_sigmas from dL/dweights, dL/dtrans, dL/dalphas; with only dL/dweights = v it
 * is render_backward's d_sigma (rendering.cpp:99-108). */
int vmb_render_weight_from_density_backward(vmb_ctx* ctx, const vmb_packed_view* p,
                                            const void* d_sigmas, const void* d_grad_weights,
                                            const void* d_grad_trans, const void* d_grad_alphas,
                                            void* d_grad_sigmas, int dtype);
/* trans = exclusive prod (1 - alpha), weights = trans * alpha (t's unused). */
int vmb_render_weight_from_alpha(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas,
                                 void* d_weights, void* d_trans, int dtype);
int vmb_render_weight_from_alpha_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas,
                                          const void* d_grad_weights, const void* d_grad_trans,
                                          void* d_grad_alphas, int dtype);
int vmb_render_transmittance_from_alpha(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_alphas,
                                        void* d_trans, int dtype);
int vmb_render_transmittance_from_alpha_backward(vmb_ctx* ctx, const vmb_packed_view* p,
                                                 const void* d_alphas, const void* d_grad_trans,
                                                 void* d_grad_alphas, int dtype);
/* out [n_rays][dim] = per-ray sum of weights * values (values NULL: sum of weights);
 * render_attribute (rendering.cpp:114-134) with the weights given. */
int vmb_accumulate_along_rays(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_weights,
                              const void* d_values, uint64_t dim, void* d_out, int dtype);
int vmb_accumulate_along_rays_backward(vmb_ctx* ctx, const vmb_packed_view* p, const void* d_weights,
                                       const void* d_values, uint64_t dim, const void* d_grad_out,
                                       void* d_grad_weights, void* d_grad_values, int dtype);
/* Slab test of every ray against every box [n_aabbs][6] = {min xyz, max xyz}, fp64:
 * t_min = max(near, max_a min(t1, t2)), t_max = min(far, min_a max(t1, t2)) with
 * t = (box - o) / d; hit = t_max > t_min, misses store miss_value. Outputs
 * [n_rays][n_aabbs]; d_hit may be NULL. Nearest reference behaviour: the domain
 * reject of OccupancyGrid::query (occupancy_grid.cpp:69, contraction.cpp:27). */
int vmb_ray_aabb_intersect(vmb_ctx* ctx, const vmb_rays* rays, const double* d_aabbs, uint64_t n_aabbs,
                           double miss_value, double* d_t_min, double* d_t_max, uint8_t* d_hit);

/* ------------------------------------------------------------------ multi-GPU (NCCL) */
/* NCCL is loaded at run time (dlopen "libnccl.so.2") only when these are used. */
int vmb_comm_unique_id(void* h_id128);
int vmb_comm_init(vmb_ctx* ctx, const void* h_id128, int nranks, int rank);
int vmb_comm_destroy(vmb_ctx* ctx);
/* In-place max all-reduce of n f64 (IEEE order == u64 bit order for values >= 0). */
int vmb_comm_allreduce_max_f64(vmb_ctx* ctx, double* d_buf, uint64_t n);
/* In-place sum all-reduce of n f64 (data-parallel parameter gradients). */
int vmb_comm_allreduce_sum_f64(vmb_ctx* ctx, double* d_buf, uint64_t n);
/* In-place all-gather: rank k's block is d_buf[k n, (k + 1) n); the grid update's
 * collective (each rank probes one equal block of cells). */
int vmb_comm_allgather_f64(vmb_ctx* ctx, double* d_buf, uint64_t n_per_rank);

/* ------------------------------------------------------------------ training step helpers
 * (tools/voxmarch.cpp cmd_train, :460-498 — the reference's trainer, outside its
 * library; the B200 framework provides its per-ray pieces on the device.)
 * Photometric MSE against a white background: err = color + (1 - opacity) - target;
 * loss = sum |err|^2 / (3n); d_color = err * 2/(3n); d_opacity = -2/(3n) * sum(err);
 * d_depth = 0. color/opacity/d_* in dtype, targets [n][3] in dtype; *h_loss gets
 * the loss (fp64, fixed-order block reduction). */
int vmb_loss_mse_background(vmb_ctx* ctx, const void* d_color, const void* d_opacity, const void* d_targets,
                            uint64_t n, int dtype, void* d_dcolor, void* d_dopacity, void* d_ddepth,
                            double* h_loss);
/* Minibatch gather: out[i] = pool[idx[i]] for origins, directions (3 x dtype) and
 * targets (3 x dtype) — one kernel. */
int vmb_gather_rays(vmb_ctx* ctx, const void* d_pool_origins, const void* d_pool_dirs,
                    const void* d_pool_targets, const uint32_t* d_idx, uint64_t n, int dtype,
                    void* d_origins, void* d_dirs, void* d_targets);

#ifdef __cplusplus
}
#endif

#endif /* VMB200_H */
