// ref_capi.cpp — extern "C" shim over the REFERENCE's own C++ API (test infrastructure).
//
// Compiled by oracle/Makefile together with the reference sources where they lie
// (/root/reference/proj/src/{core_types,contraction,occupancy_grid,ray_marching,
// rendering,fields}.cpp) into oracle/_ref/libvoxmarch_ref.so. Nothing here
// re-implements an algorithm: every entry point converts plain arrays into the
// reference's value types, calls the reference function named in its comment,
// and converts the result back. Exceptions become VMB_* codes with the exact
// what() text available from vmr_last_error().
#include <algorithm>
#include <chrono>
#include <memory>
#include <optional>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxmarch/contraction.hpp"
#include "voxmarch/core_types.hpp"
#include "voxmarch/fields.hpp"
#include "voxmarch/occupancy_grid.hpp"
#include "voxmarch/parallel.hpp"
#include "voxmarch/ray_marching.hpp"
#include "voxmarch/rendering.hpp"
#include "vm_oracle.h"

using namespace voxmarch;

struct vmo_grid {
    OccupancyGrid grid;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return VMB_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return VMB_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return VMB_RUNTIME;
    }
}

Vec3 v3(const double* p) { return Vec3{p[0], p[1], p[2]}; }

std::vector<Vec3> vecs(const double* p, uint64_t n) {
    std::vector<Vec3> out(n);
    for (uint64_t i = 0; i < n; ++i) out[i] = v3(p + 3 * i);
    return out;
}

Contraction to_contraction(const vmb_contraction* c) {
    if (c->kind == VMB_CONTRACT_AABB)
        return Contraction::aabb_normalize(Aabb(v3(c->box_min), v3(c->box_max)));
    return Contraction::sphere(v3(c->center), c->radius);
}

AnalyticField to_analytic(const vmb_field* f) {
    if (f->kind == VMB_FIELD_UNIFORM_BOX)
        return UniformBox{Aabb(v3(f->box_min), v3(f->box_max)), f->sigma, v3(f->rgb)};
    if (f->kind == VMB_FIELD_SOLID_SPHERE)
        return SolidSphere{v3(f->center), f->radius, f->sigma, v3(f->rgb)};
    return Checker{f->period, f->sigma, v3(f->rgb), v3(f->rgb_b)};
}

// An analytic field or a TrilinearVoxelField (fields.hpp:55-111) built from the
// descriptor's host arrays; both evaluated by the reference's own code.
struct RefField {
    std::optional<AnalyticField> analytic;
    std::shared_ptr<TrilinearVoxelField> voxel;
    double density(const Vec3& p) const { return voxel ? voxel->density_at(p) : density_at(*analytic, p); }
    std::pair<Vec3, double> rgb_sigma(const Vec3& p, const Vec3& dir) const {
        return voxel ? voxel->rgb_sigma_at(p, dir) : rgb_sigma_at(*analytic, p, dir);
    }
};

std::shared_ptr<TrilinearVoxelField> to_voxel(const vmb_field* f) {
    auto v = std::make_shared<TrilinearVoxelField>(f->vox_resolution, Aabb(v3(f->box_min), v3(f->box_max)));
    v->raw_density().assign(f->vox_density, f->vox_density + v->n_vertices());
    v->raw_color().assign(f->vox_color, f->vox_color + 3 * v->n_vertices());
    return v;
}

RefField to_field(const vmb_field* f) {
    RefField r;
    if (f->kind == VMB_FIELD_VOXEL)
        r.voxel = to_voxel(f);
    else
        r.analytic = to_analytic(f);
    return r;
}

MarchingConfig to_config(const vmb_march_config* c) {
    MarchingConfig m;
    m.step_size = c->step_size;
    m.early_stop_eps = c->early_stop_eps;
    m.alpha_thre = c->alpha_thre;
    m.max_samples_per_ray = c->max_samples_per_ray;
    m.unbounded_step_growth = c->unbounded_step_growth;
    return m;
}

PackedSamples to_packed(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                        const double* ts, const double* te, uint64_t n_samples) {
    PackedSamples p;
    p.offsets.assign(offsets, offsets + n_rays);
    p.counts.assign(counts, counts + n_rays);
    p.t_starts.assign(ts, ts + n_samples);
    p.t_ends.assign(te, te + n_samples);
    p.ray_indices.resize(n_samples);
    for (uint64_t r = 0; r < n_rays; ++r)
        for (uint32_t k = 0; k < counts[r]; ++k)
            if (uint64_t(offsets[r]) + k < n_samples) p.ray_indices[offsets[r] + k] = uint32_t(r);
    return p;
}

template <typename T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
    if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
    return p;
}

vmo_packed* to_result(const PackedSamples& p, const MarchStats& stats) {
    auto* out = static_cast<vmo_packed*>(std::calloc(1, sizeof(vmo_packed)));
    out->n_rays = p.n_rays();
    out->n_samples = p.n_samples();
    out->offsets = dup(p.offsets);
    out->counts = dup(p.counts);
    out->t_starts = dup(p.t_starts);
    out->t_ends = dup(p.t_ends);
    out->ray_indices = dup(p.ray_indices);
    out->samples_emitted = stats.samples_emitted;
    out->samples_kept = stats.samples_kept;
    return out;
}

// sigma_fn_for (tools/voxmarch.cpp:221-232): density of the field at each midpoint.
SigmaFn field_sigma(const RayBatch& rays, const RefField& field) {
    return [&rays, field](std::span<const double> ts, std::span<const double> te,
                          std::span<const uint32_t> idx) {
        std::vector<double> out(ts.size());
        for (size_t s = 0; s < ts.size(); ++s) {
            uint32_t r = idx[s];
            Vec3 p = rays.origins[r] + rays.directions[r] * (0.5 * (ts[s] + te[s]));
            out[s] = field.density(p);
        }
        return out;
    };
}

}  // namespace

extern "C" {

const char* vmr_last_error(void) { return g_err.c_str(); }

void vmr_packed_free(vmo_packed* p) {
    if (!p) return;
    std::free(p->offsets);
    std::free(p->counts);
    std::free(p->t_starts);
    std::free(p->t_ends);
    std::free(p->ray_indices);
    std::free(p);
}

// uniform_step_count — ray_marching.cpp:51-55
uint64_t vmr_uniform_step_count(double near_, double far_, double step) {
    return uniform_step_count(near_, far_, step);
}

// pack — core_types.cpp:30-48
int vmr_pack(const uint32_t* counts, uint64_t n_rays, uint32_t* offsets, uint32_t* ray_indices,
             uint64_t cap, uint64_t* total) {
    return guarded([&] {
        PackResult r = pack(std::span<const uint32_t>(counts, n_rays));
        *total = r.ray_indices.size();
        std::copy(r.offsets.begin(), r.offsets.end(), offsets);
        if (ray_indices && r.ray_indices.size() <= cap)
            std::copy(r.ray_indices.begin(), r.ray_indices.end(), ray_indices);
    });
}

// validate — core_types.cpp:50-78. Returns 0 when consistent, else 1..6 in the
// order: length mismatch, offset mismatch, non-positive interval,
// non-monotone t_starts, overlapping intervals, partition mismatch.
int vmr_validate(const uint32_t* offsets, uint64_t n_offsets, const uint32_t* counts,
                 uint64_t n_counts, const double* ts, uint64_t n_ts, const double* te,
                 uint64_t n_te, const uint32_t* idx, uint64_t n_idx) {
    PackedSamples p;
    p.offsets.assign(offsets, offsets + n_offsets);
    p.counts.assign(counts, counts + n_counts);
    p.t_starts.assign(ts, ts + n_ts);
    p.t_ends.assign(te, te + n_te);
    p.ray_indices.assign(idx, idx + n_idx);
    auto v = validate(p);
    if (!v) return 0;
    static const char* names[] = {"length mismatch",         "offset mismatch",
                                  "non-positive interval",   "non-monotone t_starts",
                                  "overlapping intervals",   "partition mismatch"};
    for (int i = 0; i < 6; ++i)
        if (*v == names[i]) return i + 1;
    return 99;
}

// contract — contraction.cpp:24-30
int vmr_contract(const vmb_contraction* c, const double* x, uint64_t n, double* out) {
    return guarded([&] {
        Contraction con = to_contraction(c);
        for (uint64_t i = 0; i < n; ++i) {
            Vec3 g = contract(con, v3(x + 3 * i));
            out[3 * i] = g.x;
            out[3 * i + 1] = g.y;
            out[3 * i + 2] = g.z;
        }
    });
}

// invert_grid_point — contraction.cpp:37-47
int vmr_invert_grid_point(const vmb_contraction* c, const double* g, uint64_t n, double* out,
                          uint8_t* valid) {
    return guarded([&] {
        Contraction con = to_contraction(c);
        for (uint64_t i = 0; i < n; ++i) {
            auto w = invert_grid_point(con, v3(g + 3 * i));
            valid[i] = w.has_value();
            Vec3 v = w.value_or(Vec3{});
            out[3 * i] = v.x;
            out[3 * i + 1] = v.y;
            out[3 * i + 2] = v.z;
        }
    });
}

// OccupancyGrid ctor — occupancy_grid.cpp:41-56
int vmr_grid_create(uint32_t res, const vmb_contraction* c, double thr, double ref_step,
                    double init, vmo_grid** out) {
    return guarded([&] {
        *out = new vmo_grid{OccupancyGrid(res, to_contraction(c), thr, ref_step, init)};
    });
}

void vmr_grid_destroy(vmo_grid* g) { delete g; }

// update / update_over_time with an analytic field — occupancy_grid.cpp:91-144;
// density batch as in density_batch (voxmarch.cpp:211-219) and TimeConditionedField
// (fields.cpp:264-266).
int vmr_grid_update_field(vmo_grid* g, const vmb_field* f, const double* ts, uint64_t n_ts,
                          double decay, int has_seed, uint64_t seed) {
    return guarded([&] {
        RefField field = to_field(f);
        const Vec3 velocity = v3(f->velocity);
        std::optional<uint64_t> s;
        if (has_seed) s = seed;
        g->grid.update_over_time(
            [&](std::span<const Vec3> pts, double t) {
                std::vector<double> out(pts.size());
                // TimeConditionedField::density_at (fields.cpp:264-266)
                for (size_t i = 0; i < pts.size(); ++i) out[i] = field.density(pts[i] - velocity * t);
                return out;
            },
            std::span<const double>(ts, n_ts), decay, s);
    });
}

int vmr_grid_update_callback(vmo_grid* g, vmo_density_cb cb, void* user, const double* ts,
                             uint64_t n_ts, double decay, int has_seed, uint64_t seed) {
    return guarded([&] {
        std::optional<uint64_t> s;
        if (has_seed) s = seed;
        g->grid.update_over_time(
            [&](std::span<const Vec3> pts, double t) {
                std::vector<double> flat(3 * pts.size());
                for (size_t i = 0; i < pts.size(); ++i) {
                    flat[3 * i] = pts[i].x;
                    flat[3 * i + 1] = pts[i].y;
                    flat[3 * i + 2] = pts[i].z;
                }
                std::vector<double> out(pts.size() + 16);
                int64_t m = cb(user, flat.data(), pts.size(), t, out.data());
                out.resize(m < 0 ? 0 : size_t(m));
                return out;
            },
            std::span<const double>(ts, n_ts), decay, s);
    });
}

// seed_occupancy — occupancy_grid.cpp:152-165; the predicate answers from a
// per-cell mask in the same (iz, iy, ix) visiting order.
int vmr_grid_seed_mask(vmo_grid* g, const uint8_t* occupied) {
    return guarded([&] {
        size_t cursor = 0;
        g->grid.seed_occupancy([&](const Aabb&) { return occupied[cursor++] != 0; });
    });
}

int vmr_grid_get(const vmo_grid* g, uint8_t* bits, double* cache) {
    size_t n = g->grid.n_cells();
    for (size_t c = 0; c < n; ++c) {
        if (bits) bits[c] = g->grid.bit(c) ? 1 : 0;
        if (cache) cache[c] = g->grid.density_cache(c);
    }
    return VMB_OK;
}

int vmr_grid_info(const vmo_grid* g, uint32_t* res, double* thr, double* ref_step,
                  double* thr_density, double* frac) {
    if (res) *res = g->grid.resolution();
    if (thr) *thr = g->grid.alpha_threshold();
    if (ref_step) *ref_step = g->grid.reference_step();
    if (thr_density) *thr_density = g->grid.threshold_density();
    if (frac) *frac = g->grid.occupied_fraction();
    return VMB_OK;
}

// query — occupancy_grid.cpp:67-76
int vmr_grid_query(const vmo_grid* g, const double* pts, uint64_t n, uint8_t* out) {
    return guarded([&] {
        for (uint64_t i = 0; i < n; ++i) out[i] = g->grid.query(v3(pts + 3 * i)) ? 1 : 0;
    });
}

// save_file / load_file — occupancy_grid.cpp:177-249
int vmr_grid_save(const vmo_grid* g, const char* path) {
    return guarded([&] { g->grid.save_file(path); });
}

int vmr_grid_load(const char* path, vmo_grid** out) {
    return guarded([&] { *out = new vmo_grid{OccupancyGrid::load_file(path)}; });
}

// march with the field's density at midpoints — ray_marching.cpp:57-150
int vmr_march_field(const double* o, const double* d, uint64_t n, double near_, double far_,
                    const vmo_grid* g, const vmb_field* f, const vmb_march_config* cfg,
                    int n_threads, vmo_packed** out) {
    return guarded([&] {
        RayBatch rays = RayBatch::create(vecs(o, n), vecs(d, n), near_, far_);
        RefField field = to_field(f);
        MarchStats stats;
        PackedSamples p =
            march(rays, g->grid, field_sigma(rays, field), to_config(cfg), n_threads, &stats);
        *out = to_result(p, stats);
    });
}

int vmr_march_callback(const double* o, const double* d, uint64_t n, double near_, double far_,
                       const vmo_grid* g, vmo_sigma_cb cb, void* user,
                       const vmb_march_config* cfg, int n_threads, vmo_packed** out) {
    return guarded([&] {
        RayBatch rays = RayBatch::create(vecs(o, n), vecs(d, n), near_, far_);
        SigmaFn fn = [&](std::span<const double> ts, std::span<const double> te,
                         std::span<const uint32_t> idx) {
            std::vector<double> res(ts.size() + 16);
            int64_t m = cb(user, ts.data(), te.data(), idx.data(), ts.size(), res.data());
            res.resize(m < 0 ? 0 : size_t(m));
            return res;
        };
        MarchStats stats;
        PackedSamples p = march(rays, g->grid, fn, to_config(cfg), n_threads, &stats);
        *out = to_result(p, stats);
    });
}

// march_uniform — ray_marching.cpp:152-168
int vmr_march_uniform(const double* o, const double* d, uint64_t n, double near_, double far_,
                      const vmb_march_config* cfg, vmo_packed** out) {
    return guarded([&] {
        RayBatch rays = RayBatch::create(vecs(o, n), vecs(d, n), near_, far_);
        PackedSamples p = march_uniform(rays, to_config(cfg));
        MarchStats stats{p.n_samples(), p.n_samples()};
        *out = to_result(p, stats);
    });
}

// shade_samples — voxmarch.cpp:235-251 (rgb_sigma_at at the midpoint)
int vmr_shade(const double* o, const double* d, const uint32_t* idx, const double* ts,
              const double* te, uint64_t n_samples, const vmb_field* f, double* rgbs,
              double* sigmas) {
    return guarded([&] {
        RefField field = to_field(f);
        for (uint64_t s = 0; s < n_samples; ++s) {
            uint32_t r = idx[s];
            Vec3 p = v3(o + 3 * size_t(r)) + v3(d + 3 * size_t(r)) * (0.5 * (ts[s] + te[s]));
            auto [rgb, sigma] = field.rgb_sigma(p, v3(d + 3 * size_t(r)));
            rgbs[3 * s] = rgb.x;
            rgbs[3 * s + 1] = rgb.y;
            rgbs[3 * s + 2] = rgb.z;
            sigmas[s] = sigma;
        }
    });
}

// transmittance — rendering.cpp:19-33
int vmr_transmittance(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                      const double* ts, const double* te, uint64_t n_samples,
                      const double* sigmas, double* out) {
    return guarded([&] {
        PackedSamples p = to_packed(offsets, counts, n_rays, ts, te, n_samples);
        auto t = transmittance(p, std::span<const double>(sigmas, n_samples));
        std::copy(t.begin(), t.end(), out);
    });
}

// render_forward — rendering.cpp:35-65
int vmr_render_forward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                       const double* ts, const double* te, uint64_t n_samples,
                       const double* rgbs, const double* sigmas, int n_threads, double* color,
                       double* opacity, double* depth) {
    return guarded([&] {
        PackedSamples p = to_packed(offsets, counts, n_rays, ts, te, n_samples);
        SampleAttributes a{vecs(rgbs, n_samples),
                           std::vector<double>(sigmas, sigmas + n_samples)};
        RenderOutputs r = render_forward(p, a, n_threads);
        for (uint64_t i = 0; i < n_rays; ++i) {
            color[3 * i] = r.color[i].x;
            color[3 * i + 1] = r.color[i].y;
            color[3 * i + 2] = r.color[i].z;
            opacity[i] = r.opacity[i];
            depth[i] = r.depth[i];
        }
    });
}

// render_backward — rendering.cpp:67-112
int vmr_render_backward(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                        const double* ts, const double* te, uint64_t n_samples,
                        const double* rgbs, const double* sigmas, const double* d_color,
                        const double* d_opacity, const double* d_depth, int n_threads,
                        double* d_rgbs, double* d_sigmas) {
    return guarded([&] {
        PackedSamples p = to_packed(offsets, counts, n_rays, ts, te, n_samples);
        SampleAttributes a{vecs(rgbs, n_samples),
                           std::vector<double>(sigmas, sigmas + n_samples)};
        RenderGradients g = render_backward(
            p, a, vecs(d_color, n_rays), std::span<const double>(d_opacity, n_rays),
            std::span<const double>(d_depth, n_rays), n_threads);
        for (uint64_t s = 0; s < n_samples; ++s) {
            d_rgbs[3 * s] = g.d_rgbs[s].x;
            d_rgbs[3 * s + 1] = g.d_rgbs[s].y;
            d_rgbs[3 * s + 2] = g.d_rgbs[s].z;
            d_sigmas[s] = g.d_sigmas[s];
        }
    });
}

// render_attribute — rendering.cpp:114-134
int vmr_render_attribute(const uint32_t* offsets, const uint32_t* counts, uint64_t n_rays,
                         const double* ts, const double* te, uint64_t n_samples,
                         const double* sigmas, const double* values, uint64_t n_values,
                         uint64_t dim, double* out) {
    return guarded([&] {
        PackedSamples p = to_packed(offsets, counts, n_rays, ts, te, n_samples);
        auto r = render_attribute(p, std::span<const double>(sigmas, n_samples),
                                  std::span<const double>(values, n_values), dim);
        std::copy(r.begin(), r.end(), out);
    });
}

// One benchmark step on the reference's CPU path: march -> shade -> render_forward
// -> render_backward (the cmd_train inner loop, voxmarch.cpp:483-508, with a fixed
// analytic field and caller-supplied upstream gradients). phase_ms[0..3] =
// march, shade, forward, backward wall time (steady_clock, as voxmarch.cpp:31-37).
int vmr_train_step(const double* o, const double* d, uint64_t n, double near_, double far_,
                   const vmo_grid* g, const vmb_field* f, const vmb_march_config* cfg,
                   const double* d_color, const double* d_opacity, const double* d_depth,
                   int n_threads, double* phase_ms, uint64_t* n_samples_out, double* checksum) {
    return guarded([&] {
        using clock = std::chrono::steady_clock;
        auto ms = [](clock::time_point a, clock::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        RayBatch rays = RayBatch::create(vecs(o, n), vecs(d, n), near_, far_);
        RefField field = to_field(f);
        auto t0 = clock::now();
        PackedSamples p = march(rays, g->grid, field_sigma(rays, field), to_config(cfg), n_threads);
        auto t1 = clock::now();
        SampleAttributes a;
        a.rgbs.resize(p.n_samples());
        a.sigmas.resize(p.n_samples());
        parallel_for(p.n_samples(), n_threads, [&](size_t b, size_t e) {
            for (size_t s = b; s < e; ++s) {
                uint32_t r = p.ray_indices[s];
                Vec3 x = rays.origins[r] +
                         rays.directions[r] * (0.5 * (p.t_starts[s] + p.t_ends[s]));
                auto [rgb, sigma] = field.rgb_sigma(x, rays.directions[r]);
                a.rgbs[s] = rgb;
                a.sigmas[s] = sigma;
            }
        });
        auto t2 = clock::now();
        RenderOutputs out = render_forward(p, a, n_threads);
        auto t3 = clock::now();
        RenderGradients gr = render_backward(p, a, vecs(d_color, n),
                                             std::span<const double>(d_opacity, n),
                                             std::span<const double>(d_depth, n), n_threads);
        auto t4 = clock::now();
        phase_ms[0] = ms(t0, t1);
        phase_ms[1] = ms(t1, t2);
        phase_ms[2] = ms(t2, t3);
        phase_ms[3] = ms(t3, t4);
        *n_samples_out = p.n_samples();
        double cs = 0.0;
        for (size_t r = 0; r < n; ++r) cs += out.opacity[r];
        for (size_t s = 0; s < p.n_samples(); ++s) cs += gr.d_sigmas[s];
        *checksum = cs;
    });
}

}  // extern "C"

#include "voxmarch/scene_camera.hpp"

extern "C" {

// Benchmark rays: orbit_camera (tools/voxmarch.cpp:278-286, restated: the CLI
// translation unit needs CLI11) -> look_at + generate_rays from the reference
// (scene_camera.cpp:24-63). origins/dirs hold width*height*3 doubles.
int vmr_orbit_rays(const double* box_min, const double* box_max, double angle, double elevation,
                   int width, int height, double near_, double far_, double* origins,
                   double* dirs) {
    return guarded([&] {
        Aabb domain(v3(box_min), v3(box_max));
        Vec3 center = domain.center();
        double radius = 0.6 * domain.diagonal() / std::sqrt(3.0);
        Vec3 eye = center + Vec3{radius * std::cos(angle) * std::cos(elevation),
                                 radius * std::sin(angle) * std::cos(elevation),
                                 radius * std::sin(elevation)};
        PinholeCamera cam = look_at(eye, center, {0, 0, 1}, 1.1 * width, width, height);
        RayBatch rays = generate_rays(cam, near_, far_);
        for (size_t i = 0; i < rays.n_rays(); ++i) {
            for (int k = 0; k < 3; ++k) {
                origins[3 * i + k] = rays.origins[i][k];
                dirs[3 * i + k] = rays.directions[i][k];
            }
        }
    });
}

}  // extern "C"

extern "C" {

static PinholeCamera to_cam(const vmb_camera* c) {
    PinholeCamera cam;
    for (int i = 0; i < 9; ++i) cam.rotation.m[i] = c->rotation[i];
    cam.position = v3(c->position);
    cam.focal = c->focal;
    cam.width = c->width;
    cam.height = c->height;
    return cam;
}

// look_at / generate_rays (scene_camera.cpp:25-63) of the reference, as is.
int vmr_camera_look_at(const double* eye, const double* target, const double* up, double focal,
                       int32_t width, int32_t height, vmb_camera* out) {
    return guarded([&] {
        PinholeCamera cam = look_at(v3(eye), v3(target), v3(up), focal, width, height);
        for (int i = 0; i < 9; ++i) out->rotation[i] = cam.rotation.m[i];
        for (int k = 0; k < 3; ++k) out->position[k] = cam.position[k];
        out->focal = cam.focal;
        out->width = cam.width;
        out->height = cam.height;
    });
}

int vmr_generate_rays(const vmb_camera* c, double near_, double far_, double* origins, double* dirs) {
    return guarded([&] {
        RayBatch rays = generate_rays(to_cam(c), near_, far_);
        for (size_t i = 0; i < rays.n_rays(); ++i)
            for (int k = 0; k < 3; ++k) {
                origins[3 * i + k] = rays.origins[i][k];
                dirs[3 * i + k] = rays.directions[i][k];
            }
    });
}

}  // extern "C"

extern "C" {

// query_density / query_rgb_sigma (fields.cpp:75-93, :142-168) at p - velocity*t.
int vmr_field_query(const vmb_field* f, const double* pts, uint64_t n, double t, double* sig, double* rgb) {
    return guarded([&] {
        RefField field = to_field(f);
        std::vector<Vec3> p = vecs(pts, n);
        for (auto& x : p) x = x - v3(f->velocity) * t;
        if (field.voxel) {
            if (rgb) {
                std::vector<Vec3> rgbs;
                std::vector<double> sigmas;
                field.voxel->query_rgb_sigma(p, {}, rgbs, sigmas);
                for (size_t i = 0; i < n; ++i) {
                    sig[i] = sigmas[i];
                    for (int k = 0; k < 3; ++k) rgb[3 * i + k] = rgbs[i][k];
                }
            } else {
                std::vector<double> d = field.voxel->query_density(p);
                std::copy(d.begin(), d.end(), sig);
            }
        } else {
            if (rgb) {
                std::vector<Vec3> rgbs;
                std::vector<double> sigmas;
                query_rgb_sigma(*field.analytic, p, {}, rgbs, sigmas);
                for (size_t i = 0; i < n; ++i) {
                    sig[i] = sigmas[i];
                    for (int k = 0; k < 3; ++k) rgb[3 * i + k] = rgbs[i][k];
                }
            } else {
                std::vector<double> d = query_density(*field.analytic, p);
                std::copy(d.begin(), d.end(), sig);
            }
        }
    });
}

// TrilinearVoxelField::backward (fields.cpp:170-211), accumulating into the
// caller's arrays.
int vmr_voxel_field_backward(const vmb_field* f, const double* pts, uint64_t n, const double* d_rgbs,
                             const double* d_sigmas, double* acc_d, double* acc_c) {
    return guarded([&] {
        auto v = to_voxel(f);
        TrilinearVoxelField::ParamGradients g;
        g.d_raw_density.assign(acc_d, acc_d + v->n_vertices());
        g.d_raw_color.assign(acc_c, acc_c + 3 * v->n_vertices());
        v->backward(vecs(pts, n), vecs(d_rgbs, n), std::span<const double>(d_sigmas, n), g);
        std::copy(g.d_raw_density.begin(), g.d_raw_density.end(), acc_d);
        std::copy(g.d_raw_color.begin(), g.d_raw_color.end(), acc_c);
    });
}

}  // extern "C"
