/*
 * vm_oracle.h — C interface of the CPU ORACLE (test infrastructure only).
 *
 * Two libraries implement this interface with identical semantics:
 *   vmr_*  oracle/_ref/libvoxmarch_ref.so  — the reference's own C++ sources
 *          (the .cpp files under /root/reference/proj/src, compiled in place by oracle/Makefile)
 *          wrapped by oracle/ref_capi.cpp;
 *   vmo_*  oracle/_build/libvm_oracle.so   — oracle/vm_oracle.c, a plain-C
 *          restatement of the same algorithms, pinned against vmr_* and the
 *          reference's known-answer tests (tests/test_oracle_*.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load these libraries. The product path (paper_2210_04847_b200/) never
 * links or calls them.
 *
 * All vectors are AoS doubles (x,y,z per element) exactly like std::vector<Vec3>
 * in the reference (proj/include/voxmarch/math.hpp:9-14).
 * Functions return VMB_* status codes (include/vmb200_types.h); the message of
 * the last failure is available from *_last_error() and equals the reference's
 * exception text byte for byte.
 */
#ifndef VM_ORACLE_H
#define VM_ORACLE_H

#include "../include/vmb200_types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Owning result of march()/march_uniform(): PackedSamples (core_types.hpp:29-38)
 * plus MarchStats. Free with *_packed_free. */
typedef struct vmo_packed {
    uint64_t n_rays;
    uint64_t n_samples;
    uint32_t* offsets;
    uint32_t* counts;
    double* t_starts;
    double* t_ends;
    uint32_t* ray_indices;
    uint64_t samples_emitted;
    uint64_t samples_kept;
} vmo_packed;

typedef struct vmo_grid vmo_grid;

/* Host density callback for OccupancyGrid::update_over_time (occupancy_grid.hpp:16-17):
 * fills out[0..n) for points[3*n]; returns the number of values produced
 * (a value != n reproduces the "wrong batch size" error). */
typedef int64_t (*vmo_density_cb)(void* user, const double* points, uint64_t n, double t,
                                  double* out);
/* Host sigma callback for march (ray_marching.hpp:21-24), called once per ray with
 * that ray's emitted candidates; returns the number of sigmas written to out
 * (capacity n + 16). */
typedef int64_t (*vmo_sigma_cb)(void* user, const double* t_starts, const double* t_ends,
                                const uint32_t* ray_indices, uint64_t n, double* out);

#define VMO_DECLARE(P)                                                                          \
    const char* P##_last_error(void);                                                           \
    void P##_packed_free(vmo_packed* p);                                                        \
    uint64_t P##_uniform_step_count(double near_, double far_, double step);                    \
    int P##_pack(const uint32_t* counts, uint64_t n_rays, uint32_t* offsets,                    \
                 uint32_t* ray_indices, uint64_t ray_indices_capacity, uint64_t* total);        \
    int P##_validate(const uint32_t* offsets, uint64_t n_offsets, const uint32_t* counts,       \
                     uint64_t n_counts, const double* t_starts, uint64_t n_ts,                  \
                     const double* t_ends, uint64_t n_te, const uint32_t* ray_indices,          \
                     uint64_t n_idx);                                                           \
    int P##_contract(const vmb_contraction* c, const double* x, uint64_t n, double* out);      \
    int P##_invert_grid_point(const vmb_contraction* c, const double* g, uint64_t n,            \
                              double* out, uint8_t* valid);                                     \
    int P##_grid_create(uint32_t resolution, const vmb_contraction* c, double alpha_threshold,  \
                        double reference_step, double initial_density, vmo_grid** out);         \
    void P##_grid_destroy(vmo_grid* g);                                                         \
    int P##_grid_update_field(vmo_grid* g, const vmb_field* f, const double* timestamps,        \
                              uint64_t n_timestamps, double ema_decay, int has_seed,            \
                              uint64_t seed);                                                   \
    int P##_grid_update_callback(vmo_grid* g, vmo_density_cb cb, void* user,                    \
                                 const double* timestamps, uint64_t n_timestamps,               \
                                 double ema_decay, int has_seed, uint64_t seed);                \
    int P##_grid_seed_mask(vmo_grid* g, const uint8_t* occupied);                               \
    int P##_grid_get(const vmo_grid* g, uint8_t* bits, double* cache);                          \
    int P##_grid_info(const vmo_grid* g, uint32_t* resolution, double* alpha_threshold,         \
                      double* reference_step, double* threshold_density,                        \
                      double* occupied_fraction);                                               \
    int P##_grid_query(const vmo_grid* g, const double* points, uint64_t n, uint8_t* out);      \
    int P##_grid_save(const vmo_grid* g, const char* path);                                     \
    int P##_grid_load(const char* path, vmo_grid** out);                                        \
    int P##_march_field(const double* origins, const double* dirs, uint64_t n_rays,             \
                        double near_, double far_, const vmo_grid* g, const vmb_field* f,       \
                        const vmb_march_config* cfg, int n_threads, vmo_packed** out);          \
    int P##_march_callback(const double* origins, const double* dirs, uint64_t n_rays,          \
                           double near_, double far_, const vmo_grid* g, vmo_sigma_cb cb,       \
                           void* user, const vmb_march_config* cfg, int n_threads,              \
                           vmo_packed** out);                                                   \
    int P##_march_uniform(const double* origins, const double* dirs, uint64_t n_rays,           \
                          double near_, double far_, const vmb_march_config* cfg,               \
                          vmo_packed** out);                                                    \
    int P##_shade(const double* origins, const double* dirs, const uint32_t* ray_indices,       \
                  const double* t_starts, const double* t_ends, uint64_t n_samples,             \
                  const vmb_field* f, double* rgbs, double* sigmas);                            \
    int P##_transmittance(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,     \
                          const double* t_starts, const double* t_ends, uint64_t n_samples,     \
                          const double* sigmas, double* out);                                   \
    int P##_render_forward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,    \
                           const double* t_starts, const double* t_ends, uint64_t n_samples,    \
                           const double* rgbs, const double* sigmas, int n_threads,             \
                           double* color, double* opacity, double* depth);                      \
    int P##_render_backward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,   \
                            const double* t_starts, const double* t_ends, uint64_t n_samples,   \
                            const double* rgbs, const double* sigmas, const double* d_color,    \
                            const double* d_opacity, const double* d_depth, int n_threads,      \
                            double* d_rgbs, double* d_sigmas);                                  \
    int P##_render_attribute(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,  \
                             const double* t_starts, const double* t_ends, uint64_t n_samples,  \
                             const double* sigmas, const double* values, uint64_t n_values,     \
                             uint64_t dim, double* out);                                        \
    int P##_train_step(const double* origins, const double* dirs, uint64_t n_rays,              \
                       double near_, double far_, const vmo_grid* g, const vmb_field* f,        \
                       const vmb_march_config* cfg, const double* d_color,                      \
                       const double* d_opacity, const double* d_depth, int n_threads,           \
                       double* phase_ms, uint64_t* n_samples_out, double* checksum);          \
    int P##_camera_look_at(const double* eye, const double* target, const double* up,           \
                           double focal, int32_t width, int32_t height, vmb_camera* out);       \
    int P##_generate_rays(const vmb_camera* camera, double near_, double far_, double* origins, \
                          double* dirs);                                                        \
    int P##_field_query(const vmb_field* f, const double* points, uint64_t n, double time,      \
                        double* sigmas, double* rgbs);                                          \
    int P##_voxel_field_backward(const vmb_field* f, const double* points, uint64_t n,          \
                                 const double* d_rgbs, const double* d_sigmas,                  \
                                 double* accum_density, double* accum_color);

VMO_DECLARE(vmo)
VMO_DECLARE(vmr)

/* Sharded grid update halves (port only; the reference has no multi-rank update). */
int vmo_grid_probe_range(const vmo_grid* g, const vmb_field* f, const double* timestamps,
                         uint64_t n_timestamps, int has_seed, uint64_t seed, uint64_t c0,
                         uint64_t c1, double* probed);
int vmo_grid_apply(vmo_grid* g, const double* probed, double ema_decay);

/* Multi-level grid + cone stepping (port only; vmb_march_ext semantics, include/vmb200.h):
 * levels above level 0 (finest first), the finest level containing a point decides;
 * cone: dt = min(max(t cone_angle, step), max_step), t accumulated. Walks to `far`. */
int vmo_march_cascade(const double* origins, const double* dirs, uint64_t n_rays, double near_, double far_,
                      const vmo_grid* level0, const vmo_grid* const* levels, uint32_t n_levels, int cone,
                      double cone_angle, double max_step, const vmb_field* f, const vmb_march_config* cfg,
                      vmo_packed** out);
int vmo_cascade_query(const vmo_grid* level0, const vmo_grid* const* levels, uint32_t n_levels,
                      const double* points, uint64_t n, uint8_t* out);

/* NerfAcc operators (port only; the reference performs them only inside
 * render_forward / render_backward, rendering.cpp:47-58, 67-112). Sequential per
 * ray in the reference's order; NULL outputs are skipped, NULL upstream gradients
 * count as 0. The density backward keeps rendering.cpp:99-108's suffix form, so
 * with only grad_weights = value it is render_backward's d_sigma bit for bit. */
int vmo_weight_from_density(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                            const double* t_starts, const double* t_ends, const double* sigmas,
                            double* weights, double* trans, double* alphas);
int vmo_weight_from_density_backward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                                     const double* t_starts, const double* t_ends, const double* sigmas,
                                     const double* g_weights, const double* g_trans,
                                     const double* g_alphas, double* g_sigmas);
int vmo_weight_from_alpha(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                          const double* alphas, double* weights, double* trans);
int vmo_weight_from_alpha_backward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                                   const double* alphas, const double* g_weights, const double* g_trans,
                                   double* g_alphas);
int vmo_accumulate_along_rays(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                              const double* weights, const double* values, uint64_t dim, double* out);
int vmo_accumulate_along_rays_backward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                                       const double* weights, const double* values, uint64_t dim,
                                       const double* g_out, double* g_weights, double* g_values);
int vmo_ray_aabb_intersect(const double* origins, const double* dirs, uint64_t n_rays,
                           const double* aabbs, uint64_t n_aabbs, double near_, double far_,
                           double miss_value, double* t_min, double* t_max, uint8_t* hit);

#ifdef __cplusplus
}
#endif

#endif /* VM_ORACLE_H */
