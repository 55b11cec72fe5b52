// facade.cpp — namespace voxmarch on top of the C ABI (include/vmb200.h).
//
// Every hot-path computation (packing, grid update/query, marching, rendering)
// runs in the CUDA kernels of libvoxmarch_b200.so. This file converts the
// reference's value types to device buffers and back, calls the user's host
// callbacks (SigmaFn / DensityBatchFn) exactly where the reference does, and
// rethrows C-ABI failures as the reference's exception types and messages.
// Single-point utilities (contract, invert_grid_point, density_at) evaluate the
// same __host__ __device__ expressions (csrc/vm_exact.cuh) the kernels use.
#include <cstring>
#include <istream>
#include <mutex>
#include <ostream>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iterator>

#include "vm_exact.cuh"
#include "vmb200.h"
#include "voxmarch/voxmarch.hpp"

namespace voxmarch {
namespace {

std::recursive_mutex g_mu;  // one device context shared by all facade calls

void check(int rc) {
    if (rc == VMB_OK) return;
    std::string msg = vmb_last_error();
    if (rc == VMB_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

vmb_ctx* ctx() {
    static vmb_ctx* c = nullptr;
    if (!c) check(vmb_ctx_create(0, &c));
    return c;
}

// Owning device allocation.
struct Dev {
    void* p = nullptr;
    size_t bytes = 0;
    Dev() = default;
    explicit Dev(size_t n) : bytes(n) { check(vmb_malloc(ctx(), n ? n : 16, &p)); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; }
    Dev& operator=(Dev&& o) noexcept {
        if (this != &o) {
            if (p) vmb_free(ctx(), p);
            p = o.p;
            bytes = o.bytes;
            o.p = nullptr;
        }
        return *this;
    }
    ~Dev() {
        if (p) vmb_free(ctx(), p);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

template <typename T>
Dev upload(const T* data, size_t n) {
    Dev d(n * sizeof(T));
    if (n) check(vmb_memcpy_h2d(ctx(), d.p, data, n * sizeof(T)));
    return d;
}
template <typename T>
Dev upload(const std::vector<T>& v) { return upload(v.data(), v.size()); }

template <typename T>
std::vector<T> download(const Dev& d, size_t n) {
    std::vector<T> out(n);
    if (n) check(vmb_memcpy_d2h(ctx(), out.data(), d.p, n * sizeof(T)));
    return out;
}

vmb_contraction to_c(const Contraction& c) {
    vmb_contraction o{};
    o.kind = c.kind == Contraction::Kind::AabbNormalize ? VMB_CONTRACT_AABB : VMB_CONTRACT_SPHERE;
    for (int a = 0; a < 3; ++a) {
        o.box_min[a] = c.box.min[a];
        o.box_max[a] = c.box.max[a];
        o.center[a] = c.center[a];
    }
    o.radius = c.radius;
    return o;
}

vmb_field to_f(const AnalyticField& f) {
    vmb_field o{};
    if (auto* b = std::get_if<UniformBox>(&f)) {
        o.kind = VMB_FIELD_UNIFORM_BOX;
        for (int a = 0; a < 3; ++a) {
            o.box_min[a] = b->box.min[a];
            o.box_max[a] = b->box.max[a];
            o.rgb[a] = b->rgb[a];
        }
        o.sigma = b->sigma;
    } else if (auto* s = std::get_if<SolidSphere>(&f)) {
        o.kind = VMB_FIELD_SOLID_SPHERE;
        for (int a = 0; a < 3; ++a) {
            o.center[a] = s->center[a];
            o.rgb[a] = s->rgb[a];
        }
        o.radius = s->radius;
        o.sigma = s->sigma;
    } else {
        const auto& c = std::get<Checker>(f);
        o.kind = VMB_FIELD_CHECKER;
        o.period = c.period;
        o.sigma = c.sigma;
        for (int a = 0; a < 3; ++a) {
            o.rgb[a] = c.rgb_a[a];
            o.rgb_b[a] = c.rgb_b[a];
        }
    }
    return o;
}

vmb_march_config to_m(const MarchingConfig& c) {
    vmb_march_config o{};
    o.step_size = c.step_size;
    o.early_stop_eps = c.early_stop_eps;
    o.alpha_thre = c.alpha_thre;
    o.max_samples_per_ray = c.max_samples_per_ray;
    o.unbounded_step_growth = c.unbounded_step_growth;
    return o;
}

vmb::D3 d3v(const Vec3& v) { return vmb::d3(v.x, v.y, v.z); }
Vec3 v3d(const vmb::D3& v) { return Vec3{v.x, v.y, v.z}; }

// Device copy of a ray batch (Vec3 is three packed doubles: AoS f64).
struct DevRays {
    Dev o, d;
    vmb_rays r{};
    explicit DevRays(const RayBatch& rays)
        : o(upload(reinterpret_cast<const double*>(rays.origins.data()), 3 * rays.n_rays())),
          d(upload(reinterpret_cast<const double*>(rays.directions.data()), 3 * rays.n_rays())) {
        r.d_origins = o.p;
        r.d_directions = d.p;
        r.dtype = VMB_F64;
        r.n_rays = rays.n_rays();
        r.near_plane = rays.near;
        r.far_plane = rays.far;
    }
};

// Device packed samples with the capacity protocol of vmb_march_*.
struct DevPacked {
    Dev off, cnt, ts, te, idx;
    size_t n_rays = 0, n_samples = 0, cap = 0;
    DevPacked(size_t rays, size_t capacity)
        : off(rays * 4), cnt(rays * 4), ts(capacity * 8), te(capacity * 8), idx(capacity * 4),
          n_rays(rays), cap(capacity) {}
    vmb_samples samples() const {
        return vmb_samples{off.as<uint32_t>(), cnt.as<uint32_t>(), ts.as<double>(), te.as<double>(),
                           idx.as<uint32_t>(), cap};
    }
    vmb_packed_view view() const {
        return vmb_packed_view{off.as<uint32_t>(), cnt.as<uint32_t>(), n_rays, ts.as<double>(),
                               te.as<double>(), n_samples};
    }
    PackedSamples to_host() const {
        PackedSamples p;
        p.offsets = download<uint32_t>(off, n_rays);
        p.counts = download<uint32_t>(cnt, n_rays);
        p.t_starts = download<double>(ts, n_samples);
        p.t_ends = download<double>(te, n_samples);
        p.ray_indices = download<uint32_t>(idx, n_samples);
        return p;
    }
};

// Runs a vmb_march_* call, retrying once with the exact capacity it reports.
template <typename F>
DevPacked run_packed(size_t n_rays, size_t guess, F&& call) {
    DevPacked out(n_rays, guess ? guess : 1);
    uint64_t n = 0;
    vmb_samples s = out.samples();
    int rc = call(&s, &n);
    if (rc == VMB_CAPACITY) {
        out = DevPacked(n_rays, n);
        s = out.samples();
        rc = call(&s, &n);
    }
    check(rc);
    out.n_samples = n;
    return out;
}

// Device copy of host PackedSamples (input of the rendering calls).
struct DevView {
    Dev off, cnt, ts, te;
    vmb_packed_view v{};
    explicit DevView(const PackedSamples& p)
        : off(upload(p.offsets)), cnt(upload(p.counts)), ts(upload(p.t_starts)), te(upload(p.t_ends)) {
        v = vmb_packed_view{off.as<uint32_t>(), cnt.as<uint32_t>(), p.counts.size(), ts.as<double>(),
                            te.as<double>(), p.t_starts.size()};
    }
};

const double* flat(const std::vector<Vec3>& v) { return reinterpret_cast<const double*>(v.data()); }

}  // namespace

// ================================================================== core types
RayBatch RayBatch::create(std::vector<Vec3> origins, std::vector<Vec3> directions, double near,
                          double far) {
    if (origins.size() != directions.size())
        throw std::invalid_argument("ray batch: origins/directions size mismatch");
    RayBatch b;
    b.origins = std::move(origins);
    b.directions = std::move(directions);
    b.near = near;
    b.far = far;
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevRays dr(b);  // core_types.cpp:9-28 checks run in a device kernel
    check(vmb_rays_validate(ctx(), &dr.r));
    return b;
}

PackResult pack(std::span<const uint32_t> counts) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    uint64_t total = 0;
    for (uint32_t c : counts) total += c;  // capacity only; the device computes the result
    if (total > 0xffffffffull)
        throw std::invalid_argument("pack: sample count exceeds 32-bit index range");
    Dev dc = upload(counts.data(), counts.size());
    Dev doff(counts.size() * 4), didx(total * 4);
    uint64_t n = 0;
    check(vmb_pack(ctx(), dc.as<uint32_t>(), counts.size(), doff.as<uint32_t>(), didx.as<uint32_t>(),
                   total, &n));
    return PackResult{download<uint32_t>(doff, counts.size()), download<uint32_t>(didx, n)};
}

std::optional<std::string> validate(const PackedSamples& p) {
    static const char* names[] = {nullptr,
                                  "length mismatch",
                                  "offset mismatch",
                                  "non-positive interval",
                                  "non-monotone t_starts",
                                  "overlapping intervals",
                                  "partition mismatch"};
    if (p.offsets.size() != p.counts.size()) return std::string(names[1]);
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    Dev off = upload(p.offsets), cnt = upload(p.counts), ts = upload(p.t_starts),
        te = upload(p.t_ends), idx = upload(p.ray_indices);
    vmb_packed_view v{off.as<uint32_t>(), cnt.as<uint32_t>(), p.counts.size(), ts.as<double>(),
                      te.as<double>(), p.t_starts.size()};
    int res = 0;
    check(vmb_validate(ctx(), &v, idx.as<uint32_t>(), p.offsets.size(), p.ray_indices.size(),
                       p.t_ends.size(), &res));
    if (!res) return std::nullopt;
    return std::string(names[res]);
}

// ================================================================== contraction
Contraction Contraction::sphere(const Vec3& center, double radius) {
    if (!(radius > 0.0) || !std::isfinite(radius) || !is_finite(center))
        throw std::invalid_argument("sphere contraction: requires finite center and radius > 0");
    Contraction c;
    c.kind = Kind::SphereContract;
    c.center = center;
    c.radius = radius;
    return c;
}

Vec3 contract_to_ball(const Vec3& u) {
    double r = norm(u);
    if (r <= 1.0) return u;
    return u * ((2.0 - 1.0 / r) / r);
}

Vec3 contract(const Contraction& c, const Vec3& x) {
    if (!is_finite(x)) throw std::invalid_argument("non-finite coordinate");
    return v3d(vmb::contract(vmb::make_contract(to_c(c)), d3v(x)));
}

bool is_inside_domain(const Contraction& c, const Vec3& x) {
    Vec3 g = contract(c, x);
    return g.x >= 0.0 && g.x <= 1.0 && g.y >= 0.0 && g.y <= 1.0 && g.z >= 0.0 && g.z <= 1.0;
}

std::optional<Vec3> invert_grid_point(const Contraction& c, const Vec3& g) {
    vmb::D3 w;
    if (!vmb::invert(vmb::make_contract(to_c(c)), d3v(g), &w)) return std::nullopt;
    return v3d(w);
}

// ================================================================== analytic fields
double density_at(const AnalyticField& field, const Vec3& p) {
    return vmb::field_density(to_f(field), d3v(p));
}

std::pair<Vec3, double> rgb_sigma_at(const AnalyticField& field, const Vec3& p, const Vec3&) {
    vmb::D3 rgb;
    double s = vmb::field_rgb_sigma(to_f(field), d3v(p), &rgb);
    return {v3d(rgb), s};
}

namespace {
// Batch field query on the device (vmb_field_query); rgbs == nullptr: density only.
void device_query(const vmb_field& f, std::span<const Vec3> positions, std::vector<double>& sigmas,
                  std::vector<Vec3>* rgbs) {
    const size_t n = positions.size();
    sigmas.resize(n);
    if (rgbs) rgbs->resize(n);
    if (!n) {
        check(vmb_field_query(ctx(), &f, nullptr, 0, 0.0, nullptr, nullptr));  // descriptor checks
        return;
    }
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    Dev dp = upload(reinterpret_cast<const double*>(positions.data()), 3 * n);
    Dev ds(n * 8), dc(rgbs ? n * 24 : 0);
    check(vmb_field_query(ctx(), &f, dp.as<double>(), n, 0.0, ds.as<double>(), rgbs ? dc.as<double>() : nullptr));
    check(vmb_memcpy_d2h(ctx(), sigmas.data(), ds.p, n * 8));
    if (rgbs) check(vmb_memcpy_d2h(ctx(), rgbs->data(), dc.p, n * 24));
}
}  // namespace

std::vector<double> query_density(const AnalyticField& field, std::span<const Vec3> positions) {
    std::vector<double> out;
    device_query(to_f(field), positions, out, nullptr);
    return out;
}

void query_rgb_sigma(const AnalyticField& field, std::span<const Vec3> positions, std::span<const Vec3>,
                     std::vector<Vec3>& rgbs, std::vector<double>& sigmas) {
    device_query(to_f(field), positions, sigmas, &rgbs);
}

// ================================================================== occupancy grid
OccupancyGrid::OccupancyGrid(uint32_t resolution, const Contraction& contraction,
                             double alpha_threshold, double reference_step, double initial_density)
    : resolution_(resolution), contraction_(contraction), alpha_threshold_(alpha_threshold) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    vmb_contraction c = to_c(contraction);
    check(vmb_grid_create(ctx(), resolution, &c, alpha_threshold, reference_step, initial_density,
                          &handle_));
    check(vmb_grid_info(handle_, nullptr, nullptr, nullptr, &reference_step_, nullptr));
}

OccupancyGrid::OccupancyGrid(const OccupancyGrid& o)
    : resolution_(o.resolution_), contraction_(o.contraction_),
      alpha_threshold_(o.alpha_threshold_), reference_step_(o.reference_step_) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    check(vmb_grid_clone(ctx(), o.handle_, &handle_));
}

OccupancyGrid::OccupancyGrid(OccupancyGrid&& o) noexcept
    : resolution_(o.resolution_), contraction_(o.contraction_),
      alpha_threshold_(o.alpha_threshold_), reference_step_(o.reference_step_), handle_(o.handle_) {
    o.handle_ = nullptr;
}

OccupancyGrid& OccupancyGrid::operator=(const OccupancyGrid& o) {
    if (this != &o) *this = OccupancyGrid(o);
    return *this;
}

OccupancyGrid& OccupancyGrid::operator=(OccupancyGrid&& o) noexcept {
    if (this != &o) {
        if (handle_) vmb_grid_destroy(handle_);
        resolution_ = o.resolution_;
        contraction_ = o.contraction_;
        alpha_threshold_ = o.alpha_threshold_;
        reference_step_ = o.reference_step_;
        handle_ = o.handle_;
        o.handle_ = nullptr;
        mirror_valid_ = false;
    }
    return *this;
}

OccupancyGrid::~OccupancyGrid() {
    if (handle_) vmb_grid_destroy(handle_);
}

bool OccupancyGrid::query(const Vec3& x) const {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    Dev p = upload(&x.x, 3);
    Dev out(1);
    check(vmb_grid_query(ctx(), handle_, p.as<double>(), 1, out.as<uint8_t>()));
    return download<uint8_t>(out, 1)[0] != 0;
}

void OccupancyGrid::update(const DensityBatchFn& density_fn, double ema_decay,
                           std::optional<uint64_t> jitter_seed) {
    double t0 = 0.0;
    update_over_time([&](std::span<const Vec3> pts, double) { return density_fn(pts); },
                     std::span<const double>(&t0, 1), ema_decay, jitter_seed);
}

void OccupancyGrid::update_over_time(const TimeDensityBatchFn& density_fn,
                                     std::span<const double> timestamps, double ema_decay,
                                     std::optional<uint64_t> jitter_seed) {
    if (timestamps.empty())
        throw std::invalid_argument("occupancy grid: timestamps must be non-empty");
    if (!(ema_decay >= 0.0 && ema_decay <= 1.0))
        throw std::invalid_argument("occupancy grid: ema_decay must be in [0,1]");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    const size_t n = n_cells();
    Dev pts(n * 24), cells(n * 4), probed(n * 8);
    uint64_t m = 0;
    check(vmb_grid_probe_points(ctx(), handle_, jitter_seed.has_value(), jitter_seed.value_or(0),
                                pts.as<double>(), cells.as<uint32_t>(), &m));
    std::vector<Vec3> host_pts(m);
    if (m) check(vmb_memcpy_d2h(ctx(), host_pts.data(), pts.p, m * 24));
    check(vmb_memset(ctx(), probed.p, 0, n * 8));
    Dev dens(m * 8);
    for (double t : timestamps) {  // occupancy_grid.cpp:121-140
        std::vector<double> d = density_fn(std::span<const Vec3>(host_pts), t);
        if (d.size() != m)
            throw std::runtime_error("occupancy grid: density_fn returned wrong batch size");
        if (m) check(vmb_memcpy_h2d(ctx(), dens.p, d.data(), m * 8));
        check(vmb_grid_accumulate(ctx(), handle_, dens.as<double>(), cells.as<uint32_t>(), m,
                                  probed.as<double>()));
    }
    check(vmb_grid_apply(ctx(), handle_, probed.as<double>(), ema_decay));
    invalidate();
}

void OccupancyGrid::update(const AnalyticField& field, double ema_decay,
                           std::optional<uint64_t> jitter_seed) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    vmb_field f = to_f(field);
    double t0 = 0.0;
    check(vmb_grid_update_field(ctx(), handle_, &f, &t0, 1, ema_decay, jitter_seed.has_value(),
                                jitter_seed.value_or(0)));
    invalidate();
}

double OccupancyGrid::occupied_fraction() const {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    uint64_t c = 0;
    check(vmb_grid_occupied_count(ctx(), handle_, &c));
    return double(c) / double(n_cells());
}

double OccupancyGrid::threshold_density() const {
    return -std::log1p(-alpha_threshold_) / reference_step_;  // occupancy_grid.cpp:63-65
}

std::optional<Aabb> OccupancyGrid::cell_world_box(uint32_t ix, uint32_t iy, uint32_t iz) const {
    Vec3 lo{double(ix) / resolution_, double(iy) / resolution_, double(iz) / resolution_};
    Vec3 hi{double(ix + 1) / resolution_, double(iy + 1) / resolution_, double(iz + 1) / resolution_};
    auto wlo = invert_grid_point(contraction_, lo);
    auto whi = invert_grid_point(contraction_, hi);
    if (!wlo || !whi) return std::nullopt;
    if (contraction_.kind == Contraction::Kind::AabbNormalize) return Aabb(*wlo, *whi);
    return Aabb(min(*wlo, *whi), max(*wlo, *whi));
}

void OccupancyGrid::seed_occupancy(const std::function<bool(const Aabb&)>& occupied) {
    if (contraction_.kind != Contraction::Kind::AabbNormalize)
        throw std::invalid_argument("seed_occupancy: supported for AabbNormalize grids only");
    std::vector<uint8_t> mask(n_cells());
    for (uint32_t iz = 0; iz < resolution_; ++iz)  // the predicate is user host code
        for (uint32_t iy = 0; iy < resolution_; ++iy)
            for (uint32_t ix = 0; ix < resolution_; ++ix)
                mask[cell_index(ix, iy, iz)] = occupied(*cell_world_box(ix, iy, iz)) ? 1 : 0;
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    Dev d = upload(mask);
    check(vmb_grid_seed_mask(ctx(), handle_, d.as<uint8_t>()));
    invalidate();
}

void OccupancyGrid::sync_mirror() const {
    if (mirror_valid_) return;
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    std::vector<uint8_t> packed((n_cells() + 7) / 8);
    cache_mirror_.resize(n_cells());
    check(vmb_grid_read(ctx(), handle_, packed.data(), cache_mirror_.data()));
    bits_mirror_.resize(n_cells());
    for (size_t c = 0; c < n_cells(); ++c) bits_mirror_[c] = (packed[c >> 3] >> (c & 7)) & 1u;
    mirror_valid_ = true;
}

bool OccupancyGrid::bit(size_t cell) const {
    sync_mirror();
    return bits_mirror_[cell] != 0;
}

double OccupancyGrid::density_cache(size_t cell) const {
    sync_mirror();
    return cache_mirror_[cell];
}

// OGRD v1 (occupancy_grid.cpp:177-236; proj/README.md:116-121). The bit section is
// byte-identical to the device bitfield, so it is copied, not repacked.
namespace {
template <typename T>
void put(std::ostream& out, const T& v) { out.write(reinterpret_cast<const char*>(&v), sizeof(T)); }
template <typename T>
T get(std::istream& in) {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw std::runtime_error("occupancy grid: truncated stream");
    return v;
}
}  // namespace

void OccupancyGrid::save(std::ostream& out) const {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    out.write("OGRD", 4);
    put(out, uint32_t(1));
    put(out, resolution_);
    put(out, uint8_t(contraction_.kind));
    if (contraction_.kind == Contraction::Kind::AabbNormalize) {
        for (int i = 0; i < 3; ++i) put(out, contraction_.box.min[i]);
        for (int i = 0; i < 3; ++i) put(out, contraction_.box.max[i]);
    } else {
        for (int i = 0; i < 3; ++i) put(out, contraction_.center[i]);
        put(out, contraction_.radius);
    }
    put(out, alpha_threshold_);
    put(out, reference_step_);
    std::vector<uint8_t> packed((n_cells() + 7) / 8);
    std::vector<double> cache(n_cells());
    check(vmb_grid_read(ctx(), handle_, packed.data(), cache.data()));
    std::vector<float> c32(cache.begin(), cache.end());
    out.write(reinterpret_cast<const char*>(c32.data()), std::streamsize(c32.size() * 4));
    out.write(reinterpret_cast<const char*>(packed.data()), std::streamsize(packed.size()));
    if (!out) throw std::runtime_error("occupancy grid: write failed");
}

OccupancyGrid OccupancyGrid::load(std::istream& in) {
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, "OGRD", 4) != 0) throw std::runtime_error("occupancy grid: bad magic");
    if (get<uint32_t>(in) != 1) throw std::runtime_error("occupancy grid: unsupported version");
    uint32_t res = get<uint32_t>(in);
    uint8_t tag = get<uint8_t>(in);
    Contraction c;
    if (tag == 0) {
        Vec3 lo, hi;
        for (int i = 0; i < 3; ++i) lo[i] = get<double>(in);
        for (int i = 0; i < 3; ++i) hi[i] = get<double>(in);
        c = Contraction::aabb_normalize(Aabb(lo, hi));
    } else if (tag == 1) {
        Vec3 ctr;
        for (int i = 0; i < 3; ++i) ctr[i] = get<double>(in);
        double r = get<double>(in);
        c = Contraction::sphere(ctr, r);
    } else {
        throw std::runtime_error("occupancy grid: unknown contraction tag");
    }
    double thr = get<double>(in);
    double ref = get<double>(in);
    OccupancyGrid g(res, c, thr, ref);
    size_t n = g.n_cells();
    std::vector<float> c32(n);
    in.read(reinterpret_cast<char*>(c32.data()), std::streamsize(n * 4));
    std::vector<uint8_t> packed((n + 7) / 8);
    in.read(reinterpret_cast<char*>(packed.data()), std::streamsize(packed.size()));
    if (!in) throw std::runtime_error("occupancy grid: truncated stream");
    std::vector<double> cache(c32.begin(), c32.end());
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    check(vmb_grid_write(ctx(), g.handle_, packed.data(), cache.data()));
    return g;
}

void OccupancyGrid::save_file(const std::string& path) const {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("occupancy grid: cannot open " + path);
    save(out);
}

OccupancyGrid OccupancyGrid::load_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("occupancy grid: cannot open " + path);
    return load(in);
}

// ================================================================== marching
size_t uniform_step_count(double near, double far, double step_size) {
    return size_t(vmb_uniform_step_count(near, far, step_size));
}

PackedSamples march(const RayBatch& rays, const OccupancyGrid& grid, const AnalyticField& field,
                    const MarchingConfig& config, int, MarchStats* stats) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevRays dr(rays);
    vmb_field f = to_f(field);
    vmb_march_config cfg = to_m(config);
    vmb_march_stats st{};
    DevPacked out = run_packed(rays.n_rays(), 8 * rays.n_rays() + 1024, [&](vmb_samples* s, uint64_t* n) {
        return vmb_march_field(ctx(), grid.device_handle(), &dr.r, &f, &cfg, s, n, stats ? &st : nullptr);
    });
    if (stats) {
        stats->samples_emitted = st.samples_emitted;
        stats->samples_kept = st.samples_kept;
    }
    return out.to_host();
}

PackedSamples march(const RayBatch& rays, const OccupancyGrid& grid, const SigmaFn& sigma_fn,
                    const MarchingConfig& config, int, MarchStats* stats) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevRays dr(rays);
    vmb_march_config cfg = to_m(config);
    // 1. grid-passing candidates of every ray (ray_marching.cpp:75-106), on device
    DevPacked cand = run_packed(rays.n_rays(), 32 * rays.n_rays() + 1024, [&](vmb_samples* s, uint64_t* n) {
        return vmb_march_candidates(ctx(), grid.device_handle(), &dr.r, &cfg, s, n);
    });
    PackedSamples hc = cand.to_host();
    // 2. one SigmaFn call per ray on its candidates (ray_marching.cpp:108-116)
    std::vector<double> sig(hc.n_samples());
    auto filter = [&](size_t n_rays_done) {
        Dev ds = upload(sig);
        vmb_packed_view v = cand.view();
        v.n_rays = n_rays_done;
        return run_packed(n_rays_done, hc.n_samples() + 1, [&](vmb_samples* s, uint64_t* n) {
            return vmb_march_filter(ctx(), &v, ds.as<double>(), &cfg, s, n);
        });
    };
    for (size_t r = 0; r < hc.n_rays(); ++r) {
        size_t b = hc.offsets[r], c = hc.counts[r];
        if (c == 0) continue;
        std::vector<uint32_t> idx(c, uint32_t(r));
        std::vector<double> s = sigma_fn(std::span<const double>(hc.t_starts.data() + b, c),
                                         std::span<const double>(hc.t_ends.data() + b, c), idx);
        if (s.size() != c) {
            filter(r);  // a density error of an earlier ray is reported first
            throw std::runtime_error("marching: sigma_fn returned " + std::to_string(s.size()) +
                                     " values for " + std::to_string(c) + " samples");
        }
        std::copy(s.begin(), s.end(), sig.begin() + b);
    }
    // 3. validation, alpha floor, transmittance cut, packing (ray_marching.cpp:118-149), on device
    DevPacked out = filter(hc.n_rays());
    if (stats) {
        stats->samples_emitted = hc.n_samples();
        stats->samples_kept = out.n_samples;
    }
    return out.to_host();
}

PackedSamples march_uniform(const RayBatch& rays, const MarchingConfig& config) {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevRays dr(rays);
    vmb_march_config cfg = to_m(config);
    size_t guess = rays.n_rays() * uniform_step_count(rays.near, rays.far, config.step_size) + 1;
    return run_packed(rays.n_rays(), guess, [&](vmb_samples* s, uint64_t* n) {
               return vmb_march_uniform(ctx(), &dr.r, &cfg, s, n);
           }).to_host();
}

// ================================================================== rendering
std::vector<double> transmittance(const PackedSamples& packed, std::span<const double> sigmas) {
    if (sigmas.size() != packed.n_samples())
        throw std::invalid_argument("rendering: sigma length mismatch");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevView dv(packed);
    Dev ds = upload(sigmas.data(), sigmas.size()), out(packed.n_samples() * 8);
    // the reference returns a zero-initialised vector (rendering.cpp:22); the kernel
    // writes only samples inside some ray's range
    check(vmb_memset(ctx(), out.p, 0, packed.n_samples() * 8));
    check(vmb_transmittance(ctx(), &dv.v, ds.p, out.p, VMB_F64));
    return download<double>(out, packed.n_samples());
}

RenderOutputs render_forward(const PackedSamples& packed, const SampleAttributes& attrs, int) {
    if (attrs.rgbs.size() != packed.n_samples() || attrs.sigmas.size() != packed.n_samples())
        throw std::invalid_argument("rendering: attribute length mismatch");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    const size_t n = packed.n_rays();
    DevView dv(packed);
    Dev rgb = upload(flat(attrs.rgbs), 3 * attrs.rgbs.size()), sig = upload(attrs.sigmas);
    Dev col(n * 24), op(n * 8), dep(n * 8);
    check(vmb_render_forward(ctx(), &dv.v, rgb.p, sig.p, col.p, op.p, dep.p, VMB_F64));
    RenderOutputs o;
    o.color.resize(n);
    if (n) check(vmb_memcpy_d2h(ctx(), o.color.data(), col.p, n * 24));
    o.opacity = download<double>(op, n);
    o.depth = download<double>(dep, n);
    return o;
}

RenderGradients render_backward(const PackedSamples& packed, const SampleAttributes& attrs,
                                std::span<const Vec3> d_color, std::span<const double> d_opacity,
                                std::span<const double> d_depth, int) {
    if (attrs.rgbs.size() != packed.n_samples() || attrs.sigmas.size() != packed.n_samples())
        throw std::invalid_argument("rendering: attribute length mismatch");
    if (d_color.size() != packed.n_rays() || d_opacity.size() != packed.n_rays() ||
        d_depth.size() != packed.n_rays())
        throw std::invalid_argument("rendering: upstream gradient length mismatch");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    const size_t s = packed.n_samples();
    DevView dv(packed);
    Dev rgb = upload(flat(attrs.rgbs), 3 * s), sig = upload(attrs.sigmas);
    Dev dc = upload(reinterpret_cast<const double*>(d_color.data()), 3 * d_color.size());
    Dev dop = upload(d_opacity.data(), d_opacity.size()), ddep = upload(d_depth.data(), d_depth.size());
    Dev g_rgb(s * 24), g_sig(s * 8);
    // rendering.cpp:78-79 zero-fills; samples outside every ray stay 0
    check(vmb_memset(ctx(), g_rgb.p, 0, s * 24));
    check(vmb_memset(ctx(), g_sig.p, 0, s * 8));
    check(vmb_render_backward(ctx(), &dv.v, rgb.p, sig.p, dc.p, dop.p, ddep.p, g_rgb.p, g_sig.p,
                              VMB_F64));
    RenderGradients g;
    g.d_rgbs.resize(s);
    if (s) check(vmb_memcpy_d2h(ctx(), g.d_rgbs.data(), g_rgb.p, s * 24));
    g.d_sigmas = download<double>(g_sig, s);
    return g;
}

std::vector<double> render_attribute(const PackedSamples& packed, std::span<const double> sigmas,
                                     std::span<const double> values, size_t dim) {
    if (sigmas.size() != packed.n_samples())
        throw std::invalid_argument("rendering: sigma length mismatch");
    if (dim == 0 || values.size() != packed.n_samples() * dim)
        throw std::invalid_argument("rendering: value length mismatch");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevView dv(packed);
    Dev ds = upload(sigmas.data(), sigmas.size()), dvals = upload(values.data(), values.size());
    Dev out(packed.n_rays() * dim * 8);
    check(vmb_render_attribute(ctx(), &dv.v, ds.p, dvals.p, dim, out.p, VMB_F64));
    return download<double>(out, packed.n_rays() * dim);
}

// ================================================================== TrilinearVoxelField
// fields.cpp:95-262. Host vectors hold the parameters (value semantics); batch
// queries and the backward upload them and run on the device.
namespace {
vmb_field voxel_desc(uint32_t res, const Aabb& box, const double* dens, const double* col) {
    vmb_field f{};
    f.kind = VMB_FIELD_VOXEL;
    for (int a = 0; a < 3; ++a) {
        f.box_min[a] = box.min[a];
        f.box_max[a] = box.max[a];
    }
    f.vox_resolution = res;
    f.vox_density = dens;
    f.vox_color = col;
    return f;
}

struct DevVoxel {  // the parameters on the device + the descriptor pointing at them
    Dev d, c;
    vmb_field f;
    explicit DevVoxel(const TrilinearVoxelField& v)
        : d(upload(v.raw_density())), c(upload(v.raw_color())),
          f(voxel_desc(v.resolution(), v.box(), d.as<double>(), c.as<double>())) {}
};

constexpr char kVxfdMagic[4] = {'V', 'X', 'F', 'D'};
constexpr uint32_t kVxfdVersion = 1;

template <typename T>
T vget(std::istream& in) {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw std::runtime_error("voxel field: truncated stream");
    return v;
}
}  // namespace

TrilinearVoxelField::TrilinearVoxelField(uint32_t resolution, const Aabb& box)
    : resolution_(resolution), box_(box) {
    if (resolution < 2) throw std::invalid_argument("voxel field: resolution must be >= 2 vertices per axis");
    size_t n = size_t(resolution) * resolution * resolution;
    raw_density_.assign(n, 0.0);
    raw_color_.assign(3 * n, 0.0);
}

// Single-point queries evaluate the kernels' own __host__ __device__ stencil.
double TrilinearVoxelField::density_at(const Vec3& p) const {
    return vmb::field_density(voxel_desc(resolution_, box_, raw_density_.data(), raw_color_.data()), d3v(p));
}

std::pair<Vec3, double> TrilinearVoxelField::rgb_sigma_at(const Vec3& p, const Vec3&) const {
    vmb::D3 rgb;
    double s = vmb::field_rgb_sigma(voxel_desc(resolution_, box_, raw_density_.data(), raw_color_.data()),
                                    d3v(p), &rgb);
    return {v3d(rgb), s};
}

std::vector<double> TrilinearVoxelField::query_density(std::span<const Vec3> positions) const {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevVoxel dv(*this);
    std::vector<double> out;
    device_query(dv.f, positions, out, nullptr);
    return out;
}

void TrilinearVoxelField::query_rgb_sigma(std::span<const Vec3> positions, std::span<const Vec3>,
                                          std::vector<Vec3>& rgbs, std::vector<double>& sigmas) const {
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevVoxel dv(*this);
    device_query(dv.f, positions, sigmas, &rgbs);
}

TrilinearVoxelField::ParamGradients TrilinearVoxelField::zero_gradients() const {
    ParamGradients g;
    g.d_raw_density.assign(raw_density_.size(), 0.0);
    g.d_raw_color.assign(raw_color_.size(), 0.0);
    return g;
}

void TrilinearVoxelField::backward(std::span<const Vec3> positions, std::span<const Vec3> d_rgbs,
                                   std::span<const double> d_sigmas, ParamGradients& accum) const {
    if (d_rgbs.size() != positions.size() || d_sigmas.size() != positions.size())
        throw std::invalid_argument("voxel field: gradient length mismatch");
    if (accum.d_raw_density.size() != raw_density_.size() || accum.d_raw_color.size() != raw_color_.size())
        throw std::invalid_argument("voxel field: gradient buffer size mismatch");
    const size_t n = positions.size();
    if (!n) return;
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    DevVoxel dv(*this);
    Dev dp = upload(reinterpret_cast<const double*>(positions.data()), 3 * n);
    Dev dr = upload(reinterpret_cast<const double*>(d_rgbs.data()), 3 * n);
    Dev ds = upload(d_sigmas.data(), n);
    Dev ad = upload(accum.d_raw_density), ac = upload(accum.d_raw_color);
    check(vmb_voxel_field_backward(ctx(), &dv.f, dp.as<double>(), n, dr.p, ds.p, VMB_F64, ad.as<double>(),
                                   ac.as<double>(), VMB_GRAD_DETERMINISTIC));
    check(vmb_memcpy_d2h(ctx(), accum.d_raw_density.data(), ad.p, ad.bytes));
    check(vmb_memcpy_d2h(ctx(), accum.d_raw_color.data(), ac.p, ac.bytes));
}

void TrilinearVoxelField::save(std::ostream& out) const {  // fields.cpp:224-233
    out.write(kVxfdMagic, 4);
    put(out, kVxfdVersion);
    put(out, resolution_);
    for (int i = 0; i < 3; ++i) put(out, box_.min[i]);
    for (int i = 0; i < 3; ++i) put(out, box_.max[i]);
    for (double d : raw_density_) put(out, float(d));
    for (double d : raw_color_) put(out, float(d));
    if (!out) throw std::runtime_error("voxel field: write failed");
}

TrilinearVoxelField TrilinearVoxelField::load(std::istream& in) {  // fields.cpp:235-250
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, kVxfdMagic, 4) != 0) throw std::runtime_error("voxel field: bad magic");
    if (vget<uint32_t>(in) != kVxfdVersion) throw std::runtime_error("voxel field: unsupported version");
    uint32_t resolution = vget<uint32_t>(in);
    Vec3 lo, hi;
    for (int i = 0; i < 3; ++i) lo[i] = vget<double>(in);
    for (int i = 0; i < 3; ++i) hi[i] = vget<double>(in);
    TrilinearVoxelField field(resolution, Aabb(lo, hi));
    for (double& d : field.raw_density_) d = vget<float>(in);
    for (double& d : field.raw_color_) d = vget<float>(in);
    return field;
}

void TrilinearVoxelField::save_file(const std::string& path) const {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("voxel field: cannot open " + path);
    save(out);
}

TrilinearVoxelField TrilinearVoxelField::load_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("voxel field: cannot open " + path);
    return load(in);
}

// fields.cpp:264-271
double TimeConditionedField::density_at(const Vec3& p, double t) const {
    return voxmarch::density_at(base, p - velocity * t);
}
std::pair<Vec3, double> TimeConditionedField::rgb_sigma_at(const Vec3& p, const Vec3& dir, double t) const {
    return voxmarch::rgb_sigma_at(base, p - velocity * t, dir);
}

// ================================================================== AdamOptimizer (fields.cpp:273-292)
AdamOptimizer::AdamOptimizer(size_t n_params, double lr, double beta1, double beta2, double eps)
    : lr_(lr), beta1_(beta1), beta2_(beta2), eps_(eps), m_(n_params, 0.0), v_(n_params, 0.0) {}

void AdamOptimizer::step(std::span<double> params, std::span<const double> grads) {
    if (params.size() != m_.size() || grads.size() != m_.size())
        throw std::invalid_argument("adam: parameter/gradient size mismatch");
    const size_t n = params.size();
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    Dev dp = upload(params.data(), n), dg = upload(grads.data(), n), dm = upload(m_), dv = upload(v_);
    check(vmb_adam_step(ctx(), n, dp.as<double>(), dg.as<double>(), dm.as<double>(), dv.as<double>(), lr_, beta1_,
                        beta2_, eps_, t_ + 1));
    ++t_;  // only after the gradients passed the finiteness check, as the reference
    if (n) {
        check(vmb_memcpy_d2h(ctx(), params.data(), dp.p, n * 8));
        check(vmb_memcpy_d2h(ctx(), m_.data(), dm.p, n * 8));
        check(vmb_memcpy_d2h(ctx(), v_.data(), dv.p, n * 8));
    }
}

// ================================================================== cameras (scene_camera.cpp)
namespace {
vmb_camera to_cam(const PinholeCamera& c) {
    vmb_camera o{};
    for (int i = 0; i < 9; ++i) o.rotation[i] = c.rotation.m[i];
    for (int a = 0; a < 3; ++a) o.position[a] = c.position[a];
    o.focal = c.focal;
    o.width = c.width;
    o.height = c.height;
    return o;
}
PinholeCamera from_cam(const vmb_camera& c) {
    PinholeCamera o;
    for (int i = 0; i < 9; ++i) o.rotation.m[i] = c.rotation[i];
    for (int a = 0; a < 3; ++a) o.position[a] = c.position[a];
    o.focal = c.focal;
    o.width = c.width;
    o.height = c.height;
    return o;
}
}  // namespace

void validate_camera(const PinholeCamera& camera) {
    vmb_camera c = to_cam(camera);
    check(vmb_camera_validate(&c));
}

PinholeCamera look_at(const Vec3& eye, const Vec3& target, const Vec3& up, double focal, int width, int height) {
    const double e[3] = {eye.x, eye.y, eye.z}, t[3] = {target.x, target.y, target.z}, u[3] = {up.x, up.y, up.z};
    vmb_camera c{};
    check(vmb_camera_look_at(e, t, u, focal, width, height, &c));
    return from_cam(c);
}

RayBatch generate_rays(const PinholeCamera& camera, double near, double far) {
    vmb_camera c = to_cam(camera);
    check(vmb_camera_validate(&c));
    const size_t n = size_t(camera.width) * size_t(camera.height);
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    Dev o(n * 24), d(n * 24);
    vmb_rays r{};
    check(vmb_generate_rays(ctx(), &c, near, far, VMB_F64, o.p, d.p, &r));
    RayBatch b;
    b.origins.resize(n);
    b.directions.resize(n);
    if (n) {
        check(vmb_memcpy_d2h(ctx(), b.origins.data(), o.p, n * 24));
        check(vmb_memcpy_d2h(ctx(), b.directions.data(), d.p, n * 24));
    }
    b.near = near;
    b.far = far;
    return b;
}

// {"focal": f, "width": w, "height": h, "pose": [12 numbers, row-major 3x4]}
// (scene_camera.cpp:66-99). A small reader for exactly this schema.
namespace {
const char* skip_ws(const char* p) {
    while (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t') ++p;
    return p;
}
double json_number(const std::string& text, const std::string& key) {
    size_t k = text.find("\"" + key + "\"");
    if (k == std::string::npos) throw std::runtime_error("camera: missing key " + key);
    const char* p = skip_ws(text.c_str() + k + key.size() + 2);
    if (*p != ':') throw std::runtime_error("camera: malformed json");
    char* end = nullptr;
    double v = std::strtod(skip_ws(p + 1), &end);
    if (end == skip_ws(p + 1)) throw std::runtime_error("camera: malformed json");
    return v;
}
std::vector<double> json_array(const std::string& text, const std::string& key) {
    size_t k = text.find("\"" + key + "\"");
    if (k == std::string::npos) throw std::runtime_error("camera: missing key " + key);
    const char* p = skip_ws(text.c_str() + k + key.size() + 2);
    if (*p != ':') throw std::runtime_error("camera: malformed json");
    p = skip_ws(p + 1);
    if (*p != '[') throw std::runtime_error("camera: malformed json");
    std::vector<double> out;
    p = skip_ws(p + 1);
    while (*p && *p != ']') {
        char* end = nullptr;
        out.push_back(std::strtod(p, &end));
        if (end == p) throw std::runtime_error("camera: malformed json");
        p = skip_ws(end);
        if (*p == ',') p = skip_ws(p + 1);
    }
    return out;
}
}  // namespace

PinholeCamera load_camera_json(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("camera: cannot open " + path);
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    PinholeCamera camera;
    camera.focal = json_number(text, "focal");
    camera.width = int(json_number(text, "width"));
    camera.height = int(json_number(text, "height"));
    std::vector<double> pose = json_array(text, "pose");
    if (pose.size() != 12) throw std::runtime_error("camera: pose must have 12 numbers");
    for (int row = 0; row < 3; ++row) {
        for (int col = 0; col < 3; ++col) camera.rotation.m[3 * row + col] = pose[4 * row + col];
        camera.position[row] = pose[4 * row + 3];
    }
    validate_camera(camera);
    return camera;
}

void save_camera_json(const PinholeCamera& camera, const std::string& path) {
    validate_camera(camera);
    std::ofstream out(path);
    if (!out) throw std::runtime_error("camera: cannot open " + path);
    char buf[64];
    auto num = [&](double v) {
        std::snprintf(buf, sizeof buf, "%.17g", v);
        return std::string(buf);
    };
    out << "{\n  \"focal\": " << num(camera.focal) << ",\n  \"height\": " << camera.height << ",\n  \"pose\": [";
    for (int row = 0; row < 3; ++row)
        for (int col = 0; col < 4; ++col) {
            double v = col < 3 ? camera.rotation.m[3 * row + col] : camera.position[row];
            out << (row || col ? ",\n    " : "\n    ") << num(v);
        }
    out << "\n  ],\n  \"width\": " << camera.width << "\n}\n";
}

}  // namespace voxmarch
