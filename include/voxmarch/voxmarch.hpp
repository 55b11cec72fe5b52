// voxmarch.hpp — C++ drop-in facade for the reference's hot-path API, executed on
// B200 by libvoxmarch_b200.so (through the C ABI in include/vmb200.h).
//
// A program written against the reference headers (namespace voxmarch in
// /root/reference/proj/include/voxmarch/*.hpp) compiles unchanged against this
// include directory (the per-module headers next to this file forward here) and
// links with -lvoxmarch_cpp. Signatures, value semantics, defaults and the text of
// every exception follow the reference; the cited lines are the declarations this
// file stands in for. Differences, all additive:
//   * march(rays, grid, const AnalyticField&, ...) and
//     OccupancyGrid::update(const AnalyticField&, ...) evaluate an analytic field
//     inside the CUDA kernels (no host callback round trip);
//   * n_threads is accepted and ignored (results never depend on it, as in the
//     reference, parallel.hpp:17-19);
//   * the library has no CPU path: without a CUDA device the first call throws
//     std::runtime_error("voxmarch_b200: no CUDA device available ...").
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

struct vmb_grid;

namespace voxmarch {

// ------------------------------------------------------------------ math.hpp:9-86
struct Vec3 {
    double x = 0.0, y = 0.0, z = 0.0;
    double& operator[](int i) { return (&x)[i]; }
    const double& operator[](int i) const { return (&x)[i]; }
};

inline Vec3 operator+(const Vec3& a, const Vec3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline Vec3 operator-(const Vec3& a, const Vec3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline Vec3 operator*(const Vec3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline Vec3 operator*(double s, const Vec3& a) { return a * s; }
inline Vec3 operator*(const Vec3& a, const Vec3& b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
inline Vec3 operator/(const Vec3& a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline Vec3 operator/(const Vec3& a, const Vec3& b) { return {a.x / b.x, a.y / b.y, a.z / b.z}; }
inline Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
inline Vec3& operator+=(Vec3& a, const Vec3& b) { return a = a + b; }
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }
inline Vec3 normalize(const Vec3& a) { return a / norm(a); }
inline bool is_finite(const Vec3& a) {
    return std::isfinite(a.x) && std::isfinite(a.y) && std::isfinite(a.z);
}
inline Vec3 min(const Vec3& a, const Vec3& b) {
    return {a.x < b.x ? a.x : b.x, a.y < b.y ? a.y : b.y, a.z < b.z ? a.z : b.z};
}
inline Vec3 max(const Vec3& a, const Vec3& b) {
    return {a.x < b.x ? b.x : a.x, a.y < b.y ? b.y : a.y, a.z < b.z ? b.z : a.z};
}

struct Aabb {
    Vec3 min{0.0, 0.0, 0.0};
    Vec3 max{1.0, 1.0, 1.0};
    Aabb() = default;
    Aabb(const Vec3& lo, const Vec3& hi) : min(lo), max(hi) {
        if (!(hi.x > lo.x && hi.y > lo.y && hi.z > lo.z))
            throw std::invalid_argument("aabb max must be strictly greater than min");
    }
    Vec3 center() const { return (min + max) * 0.5; }
    Vec3 size() const { return max - min; }
    double diagonal() const { return norm(max - min); }
    bool contains(const Vec3& p) const {
        return p.x >= min.x && p.x <= max.x && p.y >= min.y && p.y <= max.y && p.z >= min.z &&
               p.z <= max.z;
    }
};

struct Mat3 {
    double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    static Mat3 identity() { return Mat3{}; }
    static Mat3 from_columns(const Vec3& c0, const Vec3& c1, const Vec3& c2) {
        Mat3 r;
        r.m[0] = c0.x, r.m[1] = c1.x, r.m[2] = c2.x;
        r.m[3] = c0.y, r.m[4] = c1.y, r.m[5] = c2.y;
        r.m[6] = c0.z, r.m[7] = c1.z, r.m[8] = c2.z;
        return r;
    }
    Vec3 col(int i) const { return {m[i], m[3 + i], m[6 + i]}; }
    Vec3 row(int i) const { return {m[3 * i], m[3 * i + 1], m[3 * i + 2]}; }
};
inline Vec3 operator*(const Mat3& a, const Vec3& v) {
    return {dot(a.row(0), v), dot(a.row(1), v), dot(a.row(2), v)};
}
inline Mat3 transpose(const Mat3& a) { return Mat3::from_columns(a.row(0), a.row(1), a.row(2)); }
inline double determinant(const Mat3& a) { return dot(a.col(0), cross(a.col(1), a.col(2))); }

// ------------------------------------------------------------------ rng.hpp:10-51
inline uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
inline uint64_t mix_seed(uint64_t a, uint64_t b) {
    uint64_t s = a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2));
    return splitmix64(s);
}
inline double unit_double(uint64_t bits) { return double(bits >> 11) * 0x1.0p-53; }

class Rng {
public:
    explicit Rng(uint64_t seed = 0) : state_(seed) { splitmix64(state_); }
    uint64_t next_u64() { return splitmix64(state_); }
    double uniform() { return unit_double(next_u64()); }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    Vec3 uniform_vec3() {
        double a = uniform(), b = uniform(), c = uniform();
        return {a, b, c};
    }
    uint64_t uniform_below(uint64_t n) {
        if (n == 0) return 0;
        uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t v = next_u64();
        while (v >= limit) v = next_u64();
        return v % n;
    }

private:
    uint64_t state_;
};

// ------------------------------------------------------------------ core_types.hpp:15-57
struct RayBatch {
    std::vector<Vec3> origins;
    std::vector<Vec3> directions;
    double near = 0.0;
    double far = 1.0;
    static RayBatch create(std::vector<Vec3> origins, std::vector<Vec3> directions, double near,
                           double far);
    size_t n_rays() const { return origins.size(); }
};

struct PackedSamples {
    std::vector<uint32_t> offsets;
    std::vector<uint32_t> counts;
    std::vector<double> t_starts;
    std::vector<double> t_ends;
    std::vector<uint32_t> ray_indices;
    size_t n_rays() const { return counts.size(); }
    size_t n_samples() const { return t_starts.size(); }
};

struct RenderOutputs {
    std::vector<Vec3> color;
    std::vector<double> opacity;
    std::vector<double> depth;
};

struct PackResult {
    std::vector<uint32_t> offsets;
    std::vector<uint32_t> ray_indices;
};

PackResult pack(std::span<const uint32_t> counts);
std::optional<std::string> validate(const PackedSamples& packed);

// ------------------------------------------------------------------ contraction.hpp:14-45
struct Contraction {
    enum class Kind : uint8_t { AabbNormalize = 0, SphereContract = 1 };
    Kind kind = Kind::AabbNormalize;
    Aabb box;
    Vec3 center{0.0, 0.0, 0.0};
    double radius = 1.0;
    static Contraction aabb_normalize(const Aabb& box) {
        Contraction c;
        c.kind = Kind::AabbNormalize;
        c.box = box;
        return c;
    }
    static Contraction sphere(const Vec3& center, double radius);
};

Vec3 contract_to_ball(const Vec3& u);
Vec3 contract(const Contraction& c, const Vec3& x);
bool is_inside_domain(const Contraction& c, const Vec3& x);
std::optional<Vec3> invert_grid_point(const Contraction& c, const Vec3& g);

// ------------------------------------------------------------------ fields.hpp:17-48 (analytic)
struct UniformBox {
    Aabb box;
    double sigma = 1.0;
    Vec3 rgb{1.0, 1.0, 1.0};
};
struct SolidSphere {
    Vec3 center{0.5, 0.5, 0.5};
    double radius = 0.2;
    double sigma = 1.0;
    Vec3 rgb{1.0, 1.0, 1.0};
};
struct Checker {
    double period = 0.125;
    double sigma = 1.0;
    Vec3 rgb_a{1.0, 1.0, 1.0};
    Vec3 rgb_b{0.0, 0.0, 0.0};
};
using AnalyticField = std::variant<UniformBox, SolidSphere, Checker>;

double density_at(const AnalyticField& field, const Vec3& p);
std::pair<Vec3, double> rgb_sigma_at(const AnalyticField& field, const Vec3& p, const Vec3& dir);
std::vector<double> query_density(const AnalyticField& field, std::span<const Vec3> positions);
void query_rgb_sigma(const AnalyticField& field, std::span<const Vec3> positions,
                     std::span<const Vec3> directions, std::vector<Vec3>& rgbs,
                     std::vector<double>& sigmas);

inline double softplus(double x) {  // fields.hpp:47-50
    return x > 0.0 ? x + std::log1p(std::exp(-x)) : std::log1p(std::exp(x));
}
inline double sigmoid(double x) {  // fields.hpp:51-54
    if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
    double e = std::exp(x);
    return e / (1.0 + e);
}

// fields.hpp:56-111. Parameters live in these host vectors (the reference's value
// semantics: raw_density()/raw_color() are mutable references); batch queries and
// backward upload them and run on the device (vmb_field_query,
// vmb_voxel_field_backward in the reference's sample-order fold).
class TrilinearVoxelField {
public:
    TrilinearVoxelField(uint32_t resolution, const Aabb& box);

    double density_at(const Vec3& p) const;
    std::pair<Vec3, double> rgb_sigma_at(const Vec3& p, const Vec3& dir) const;
    std::vector<double> query_density(std::span<const Vec3> positions) const;
    void query_rgb_sigma(std::span<const Vec3> positions, std::span<const Vec3> directions,
                         std::vector<Vec3>& rgbs, std::vector<double>& sigmas) const;

    struct ParamGradients {
        std::vector<double> d_raw_density;  // resolution^3
        std::vector<double> d_raw_color;    // 3 * resolution^3
    };
    ParamGradients zero_gradients() const;
    void backward(std::span<const Vec3> positions, std::span<const Vec3> d_rgbs,
                  std::span<const double> d_sigmas, ParamGradients& accum) const;

    std::vector<double>& raw_density() { return raw_density_; }
    const std::vector<double>& raw_density() const { return raw_density_; }
    std::vector<double>& raw_color() { return raw_color_; }
    const std::vector<double>& raw_color() const { return raw_color_; }

    uint32_t resolution() const { return resolution_; }
    const Aabb& box() const { return box_; }
    size_t n_vertices() const { return raw_density_.size(); }
    size_t vertex_index(uint32_t ix, uint32_t iy, uint32_t iz) const {
        return size_t(ix) + size_t(resolution_) * (size_t(iy) + size_t(resolution_) * iz);
    }

    void save(std::ostream& out) const;
    void save_file(const std::string& path) const;
    static TrilinearVoxelField load(std::istream& in);
    static TrilinearVoxelField load_file(const std::string& path);

private:
    uint32_t resolution_ = 0;
    Aabb box_;
    std::vector<double> raw_density_;
    std::vector<double> raw_color_;
};

// fields.hpp:113-121
struct TimeConditionedField {
    AnalyticField base;
    Vec3 velocity{0.0, 0.0, 0.0};

    double density_at(const Vec3& p, double t) const;
    std::pair<Vec3, double> rgb_sigma_at(const Vec3& p, const Vec3& dir, double t) const;
};

// fields.hpp:123-142; the update runs on the device (vmb_adam_step).
class AdamOptimizer {
public:
    explicit AdamOptimizer(size_t n_params, double lr = 1e-2, double beta1 = 0.9,
                           double beta2 = 0.999, double eps = 1e-8);

    void step(std::span<double> params, std::span<const double> grads);

    double learning_rate() const { return lr_; }
    void set_learning_rate(double lr) { lr_ = lr; }

private:
    double lr_, beta1_, beta2_, eps_;
    uint64_t t_ = 0;
    std::vector<double> m_, v_;
};

// ------------------------------------------------------------------ scene_camera.hpp:10-38
struct PinholeCamera {
    Mat3 rotation;
    Vec3 position;
    double focal = 1.0;  // pixels
    int width = 0;
    int height = 0;
};

void validate_camera(const PinholeCamera& camera);
PinholeCamera look_at(const Vec3& eye, const Vec3& target, const Vec3& up, double focal,
                      int width, int height);
// one ray per pixel centre, generated on the device (vmb_generate_rays)
RayBatch generate_rays(const PinholeCamera& camera, double near, double far);
PinholeCamera load_camera_json(const std::string& path);
void save_camera_json(const PinholeCamera& camera, const std::string& path);

// ------------------------------------------------------------------ occupancy_grid.hpp:16-89
using DensityBatchFn = std::function<std::vector<double>(std::span<const Vec3>)>;
using TimeDensityBatchFn = std::function<std::vector<double>(std::span<const Vec3>, double)>;

class OccupancyGrid {
public:
    OccupancyGrid(uint32_t resolution, const Contraction& contraction,
                  double alpha_threshold = 1e-2, double reference_step = 0.0,
                  double initial_density = 0.0);
    OccupancyGrid(const OccupancyGrid& other);
    OccupancyGrid(OccupancyGrid&& other) noexcept;
    OccupancyGrid& operator=(const OccupancyGrid& other);
    OccupancyGrid& operator=(OccupancyGrid&& other) noexcept;
    ~OccupancyGrid();

    bool query(const Vec3& x) const;
    void update(const DensityBatchFn& density_fn, double ema_decay,
                std::optional<uint64_t> jitter_seed = std::nullopt);
    void update_over_time(const TimeDensityBatchFn& density_fn, std::span<const double> timestamps,
                          double ema_decay, std::optional<uint64_t> jitter_seed = std::nullopt);
    // device fast path: the analytic field is evaluated inside the probe kernel
    void update(const AnalyticField& field, double ema_decay,
                std::optional<uint64_t> jitter_seed = std::nullopt);
    double occupied_fraction() const;
    double threshold_density() const;
    void seed_occupancy(const std::function<bool(const Aabb&)>& occupied);

    void save(std::ostream& out) const;
    void save_file(const std::string& path) const;
    static OccupancyGrid load(std::istream& in);
    static OccupancyGrid load_file(const std::string& path);

    uint32_t resolution() const { return resolution_; }
    const Contraction& contraction() const { return contraction_; }
    double alpha_threshold() const { return alpha_threshold_; }
    double reference_step() const { return reference_step_; }
    size_t n_cells() const { return size_t(resolution_) * resolution_ * resolution_; }
    bool bit(size_t cell) const;
    double density_cache(size_t cell) const;
    size_t cell_index(uint32_t ix, uint32_t iy, uint32_t iz) const {
        return size_t(ix) + size_t(resolution_) * (size_t(iy) + size_t(resolution_) * iz);
    }
    std::optional<Aabb> cell_world_box(uint32_t ix, uint32_t iy, uint32_t iz) const;

    vmb_grid* device_handle() const { return handle_; }

private:
    OccupancyGrid() = default;
    void invalidate() { mirror_valid_ = false; }
    void sync_mirror() const;

    uint32_t resolution_ = 0;
    Contraction contraction_;
    double alpha_threshold_ = 1e-2;
    double reference_step_ = 0.0;
    vmb_grid* handle_ = nullptr;
    // host mirror of the device state for the element accessors (lazily refreshed)
    mutable bool mirror_valid_ = false;
    mutable std::vector<uint8_t> bits_mirror_;
    mutable std::vector<double> cache_mirror_;
};

// ------------------------------------------------------------------ ray_marching.hpp:11-49
struct MarchingConfig {
    double step_size = 1.6914558667664816e-3;
    double early_stop_eps = 1e-4;
    double alpha_thre = 1e-2;
    uint32_t max_samples_per_ray = 2048;
    double unbounded_step_growth = 1.0;
};

inline double default_step_size(const Aabb& box) { return box.diagonal() / 1024.0; }

using SigmaFn = std::function<std::vector<double>(std::span<const double>, std::span<const double>,
                                                  std::span<const uint32_t>)>;

struct MarchStats {
    size_t samples_emitted = 0;
    size_t samples_kept = 0;
};

PackedSamples march(const RayBatch& rays, const OccupancyGrid& grid, const SigmaFn& sigma_fn,
                    const MarchingConfig& config, int n_threads = 1, MarchStats* stats = nullptr);
// fused device path: density of an analytic field at each candidate midpoint
PackedSamples march(const RayBatch& rays, const OccupancyGrid& grid, const AnalyticField& field,
                    const MarchingConfig& config, int n_threads = 1, MarchStats* stats = nullptr);
PackedSamples march_uniform(const RayBatch& rays, const MarchingConfig& config);
size_t uniform_step_count(double near, double far, double step_size);

// ------------------------------------------------------------------ rendering.hpp:10-45
struct SampleAttributes {
    std::vector<Vec3> rgbs;
    std::vector<double> sigmas;
};

struct RenderGradients {
    std::vector<Vec3> d_rgbs;
    std::vector<double> d_sigmas;
};

std::vector<double> transmittance(const PackedSamples& packed, std::span<const double> sigmas);
RenderOutputs render_forward(const PackedSamples& packed, const SampleAttributes& attrs,
                             int n_threads = 1);
RenderGradients render_backward(const PackedSamples& packed, const SampleAttributes& attrs,
                                std::span<const Vec3> d_color, std::span<const double> d_opacity,
                                std::span<const double> d_depth, int n_threads = 1);
std::vector<double> render_attribute(const PackedSamples& packed, std::span<const double> sigmas,
                                     std::span<const double> values, size_t dim);

}  // namespace voxmarch
