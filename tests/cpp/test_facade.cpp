// test_facade.cpp — the reference's hot-path test intents (proj/tests/unit/
// test_{core_types,occupancy_grid,ray_marching,rendering}.cpp) exercised through
// the C++ drop-in facade, i.e. on the B200 kernels. Written for this repo; each
// case names the reference test whose property it checks.
#include <cmath>
#include <sstream>

#include "mini_check.hpp"
#include "voxmarch/core_types.hpp"
#include "voxmarch/occupancy_grid.hpp"
#include "voxmarch/ray_marching.hpp"
#include "voxmarch/rendering.hpp"
#include "voxmarch/rng.hpp"

using namespace voxmarch;

namespace {

const Contraction kUnit = Contraction::aabb_normalize(Aabb({0, 0, 0}, {1, 1, 1}));

RayBatch x_ray(double near = 0.2, double far = 1.0) {
    return RayBatch::create({{0.0, 0.5, 0.5}}, {{1.0, 0.0, 0.0}}, near, far);
}

SigmaFn density_sigma(const RayBatch& rays, std::function<double(const Vec3&)> f) {
    return [&rays, f](std::span<const double> ts, std::span<const double> te,
                      std::span<const uint32_t> idx) {
        std::vector<double> out(ts.size());
        for (size_t s = 0; s < ts.size(); ++s)
            out[s] = f(rays.origins[idx[s]] + rays.directions[idx[s]] * (0.5 * (ts[s] + te[s])));
        return out;
    };
}

struct Instance {
    PackedSamples p;
    SampleAttributes a;
};

Instance random_instance(Rng& rng, size_t max_rays = 8, size_t max_per = 16) {
    std::vector<uint32_t> counts(rng.uniform_below(max_rays + 1));
    for (auto& c : counts) c = uint32_t(rng.uniform_below(max_per + 1));
    PackResult pr = pack(counts);
    Instance in;
    in.p.offsets = pr.offsets;
    in.p.counts = counts;
    in.p.ray_indices = pr.ray_indices;
    for (size_t r = 0; r < counts.size(); ++r) {
        double t = rng.uniform(0.0, 0.5);
        for (uint32_t k = 0; k < counts[r]; ++k) {
            double w = rng.uniform(0.01, 0.2);
            in.p.t_starts.push_back(t);
            in.p.t_ends.push_back(t + w);
            t += w;
        }
    }
    for (size_t s = 0; s < in.p.n_samples(); ++s) {
        in.a.rgbs.push_back({rng.uniform(), rng.uniform(), rng.uniform()});
        in.a.sigmas.push_back(rng.uniform(0.0, 8.0));
    }
    return in;
}

}  // namespace

// ------------------------------------------------------------ core types
TEST("pack: worked examples and 32-bit overflow (test_core_types.cpp:32-50)") {
    PackResult r = pack(std::vector<uint32_t>{2, 0, 3});
    CHECK((r.offsets == std::vector<uint32_t>{0, 2, 2}));
    CHECK((r.ray_indices == std::vector<uint32_t>{0, 0, 2, 2, 2}));
    CHECK(pack(std::vector<uint32_t>{}).offsets.empty());
    CHECK((pack(std::vector<uint32_t>{5}).ray_indices == std::vector<uint32_t>(5, 0)));
    CHECK_THROWS_MSG(pack(std::vector<uint32_t>{0x80000000u, 0x80000001u}), std::invalid_argument,
                     "pack: sample count exceeds 32-bit index range");
}

TEST("validate: first violated invariant (test_core_types.cpp:85-129)") {
    PackedSamples p;
    p.counts = {2, 0, 3};
    p.offsets = {0, 2, 2};
    p.ray_indices = {0, 0, 2, 2, 2};
    p.t_starts = {0.1, 0.3, 0.0, 0.2, 0.5};
    p.t_ends = {0.2, 0.4, 0.1, 0.3, 0.6};
    CHECK(!validate(p).has_value());
    auto q = p;
    q.offsets = {0, 1, 2};
    CHECK(validate(q) == std::optional<std::string>("offset mismatch"));
    q = p;
    q.t_ends[3] = 0.2;
    CHECK(validate(q) == std::optional<std::string>("non-positive interval"));
    q = p;
    q.t_starts[3] = 0.0;  // equal to its predecessor: intervals stay positive
    CHECK(validate(q) == std::optional<std::string>("non-monotone t_starts"));
    q = p;
    q.t_ends[3] = 0.55;
    CHECK(validate(q) == std::optional<std::string>("overlapping intervals"));
    q = p;
    q.ray_indices[3] = 1;
    CHECK(validate(q) == std::optional<std::string>("partition mismatch"));
    q = p;
    q.t_ends.pop_back();
    CHECK(validate(q) == std::optional<std::string>("length mismatch"));
}

TEST("RayBatch::create validation messages (core_types.cpp:9-28)") {
    CHECK_THROWS_MSG(RayBatch::create({{0, 0, 0}}, {{1, 1, 0}}, 0.2, 1.0), std::invalid_argument,
                     "ray batch: non-unit direction at index 0");
    CHECK_THROWS_MSG(RayBatch::create({{0, 0, NAN}}, {{1, 0, 0}}, 0.2, 1.0), std::invalid_argument,
                     "ray batch: non-finite ray at index 0");
    CHECK_THROWS_MSG(RayBatch::create({}, {}, 1.0, 0.5), std::invalid_argument,
                     "ray batch: requires far > near >= 0");
}

// ------------------------------------------------------------ marching
TEST("march_uniform emits the arithmetic lattice (test_ray_marching.cpp:34-59)") {
    MarchingConfig c;
    c.step_size = 0.1;
    PackedSamples p = march_uniform(x_ray(), c);
    CHECK(p.n_samples() == 8);
    for (size_t i = 0; i < p.n_samples(); ++i) {
        CHECK_NEAR(p.t_starts[i], 0.2 + 0.1 * double(i), 1e-12);
        CHECK_NEAR(p.t_ends[i], 0.3 + 0.1 * double(i), 1e-12);
    }
    CHECK(!validate(p).has_value());
    PackedSamples one = march_uniform(x_ray(0.2, 0.25), c);
    CHECK(one.n_samples() == 1 && std::fabs(one.t_ends[0] - 0.25) < 1e-12);
    PackedSamples none = march_uniform(RayBatch::create({}, {}, 0.2, 1.0), c);
    CHECK(none.n_rays() == 0 && none.n_samples() == 0);
}

TEST("empty grid emits nothing (test_ray_marching.cpp:61-72)") {
    OccupancyGrid g(16, kUnit);
    RayBatch rays = x_ray();
    MarchingConfig c;
    c.step_size = 0.05;
    MarchStats st;
    PackedSamples p = march(rays, g, density_sigma(rays, [](const Vec3&) { return 1.0; }), c, 1, &st);
    CHECK(p.n_samples() == 0 && p.counts == std::vector<uint32_t>{0} && st.samples_emitted == 0);
}

TEST("alpha floor drops thin samples (test_ray_marching.cpp:74-93)") {
    OccupancyGrid g(16, kUnit, 1e-2, 0.0, 1e6);
    RayBatch rays = x_ray();
    MarchingConfig c;
    c.step_size = 0.1;
    auto fn = density_sigma(rays, [](const Vec3&) { return 0.1; });
    MarchStats st;
    CHECK(march(rays, g, fn, c, 1, &st).n_samples() == 0);
    CHECK(st.samples_emitted == 8);
    c.alpha_thre = 0.0;
    CHECK(march(rays, g, fn, c).n_samples() == 8);
    // the same through the fused device path with an analytic field
    c.alpha_thre = 1e-2;
    UniformBox box{Aabb({-1, -1, -1}, {2, 2, 2}), 0.1, {1, 1, 1}};
    CHECK(march(rays, g, AnalyticField(box), c, 1, &st).n_samples() == 0);
    CHECK(st.samples_emitted == 8);
}

TEST("opaque wall stops the ray (test_ray_marching.cpp:95-117)") {
    OccupancyGrid g(64, kUnit);
    g.seed_occupancy([](const Aabb& cell) { return cell.max.x > 0.4 && cell.min.x < 0.5; });
    RayBatch rays = x_ray();
    MarchingConfig c;
    c.step_size = 0.01;
    c.alpha_thre = 0.0;
    auto wall = [](const Vec3& p) { return (p.x >= 0.4 && p.x <= 0.5) ? 1000.0 : 0.0; };
    PackedSamples p = march(rays, g, density_sigma(rays, wall), c);
    CHECK(p.n_samples() >= 1 && p.n_samples() <= 10);
    double tau = 0.0;
    for (size_t s = 0; s < p.n_samples(); ++s)
        tau += wall({0.5 * (p.t_starts[s] + p.t_ends[s]), 0.5, 0.5}) * (p.t_ends[s] - p.t_starts[s]);
    CHECK(std::exp(-tau) < 1e-4);
}

TEST("early termination removes only the sub-threshold tail (test_ray_marching.cpp:119-147)") {
    Rng rng(77);
    for (int trial = 0; trial < 30; ++trial) {
        OccupancyGrid g(16, kUnit, 1e-2, 0.0, 1e6);
        RayBatch rays = x_ray();
        MarchingConfig c;
        c.step_size = 0.02;
        c.alpha_thre = 0.0;
        c.early_stop_eps = 1e-3;
        double scale = rng.uniform(0.0, 60.0);
        auto dens = [scale](const Vec3& p) { return scale * (0.5 + 0.5 * std::sin(20 * p.x)); };
        PackedSamples p = march(rays, g, density_sigma(rays, dens), c);
        CHECK(!validate(p).has_value());
        double prod = 1.0, last = 0.0;
        for (size_t s = 0; s < p.n_samples(); ++s) {
            last = 1.0 - std::exp(-dens({0.5 * (p.t_starts[s] + p.t_ends[s]), 0.5, 0.5}) *
                                  (p.t_ends[s] - p.t_starts[s]));
            if (s + 1 < p.n_samples()) CHECK(prod * (1.0 - last) >= c.early_stop_eps);
            prod *= 1.0 - last;
        }
        if (p.n_samples()) CHECK(prod >= c.early_stop_eps * (1.0 - last));
    }
}

TEST("density callback errors (test_ray_marching.cpp:201-221)") {
    OccupancyGrid g(8, kUnit, 1e-2, 0.0, 1e6);
    RayBatch rays = x_ray();
    MarchingConfig c;
    c.step_size = 0.1;
    SigmaFn wrong = [](std::span<const double> ts, std::span<const double>, std::span<const uint32_t>) {
        return std::vector<double>(ts.size() + 1, 1.0);
    };
    CHECK_THROWS_MSG(march(rays, g, wrong, c), std::runtime_error,
                     "marching: sigma_fn returned 9 values for 8 samples");
    SigmaFn nan_last = [](std::span<const double> ts, std::span<const double>, std::span<const uint32_t>) {
        std::vector<double> v(ts.size(), 1.0);
        v.back() = std::nan("");
        return v;
    };
    CHECK_THROWS_MSG(march(rays, g, nan_last, c), std::runtime_error,
                     "marching: non-finite density at ray 0 sample 7");
    CHECK_THROWS_MSG(march(rays, g, AnalyticField(UniformBox{Aabb({-1, -1, -1}, {2, 2, 2}), -1.0, {}}), c),
                     std::runtime_error, "marching: negative density at ray 0 sample 0");
    c.step_size = 0.0;
    CHECK_THROWS_MSG(march(rays, g, wrong, c), std::invalid_argument, "marching: step_size must be > 0");
}

TEST("step growth outside the unit ball (test_ray_marching.cpp:223-245)") {
    OccupancyGrid g(32, Contraction::sphere({0, 0, 0}, 0.5), 1e-2, 0.0, 1e6);
    RayBatch rays = RayBatch::create({{0, 0, 0}}, {{1, 0, 0}}, 0.01, 100.0);
    MarchingConfig fixed;
    fixed.step_size = 0.02;
    fixed.alpha_thre = 0.0;
    fixed.max_samples_per_ray = 256;
    MarchingConfig growing = fixed;
    growing.unbounded_step_growth = 1.05;
    auto fn = density_sigma(rays, [](const Vec3&) { return 0.01; });
    PackedSamples a = march(rays, g, fn, fixed), b = march(rays, g, fn, growing);
    CHECK(a.n_samples() == 256);
    CHECK(b.n_samples() < a.n_samples());
    CHECK(std::fabs(b.t_ends.back() - 100.0) < 1e-9);
    for (size_t s = 1; s + 1 < b.n_samples(); ++s)
        CHECK(b.t_ends[s] - b.t_starts[s] >= b.t_ends[s - 1] - b.t_starts[s - 1] - 1e-12);
}

TEST("conservative pruning matches uniform rendering (test_ray_marching.cpp:247-293)") {
    OccupancyGrid g(32, kUnit);
    Vec3 ctr{0.5, 0.5, 0.5};
    double rad = 0.22;
    g.seed_occupancy([&](const Aabb& cell) { return norm(max(cell.min, min(ctr, cell.max)) - ctr) <= rad; });
    Rng rng(7);
    std::vector<Vec3> o, d;
    for (int r = 0; r < 32; ++r) {
        o.push_back({rng.uniform(0.3, 0.7), rng.uniform(0.3, 0.7), -0.1});
        d.push_back(normalize(Vec3{rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 1.0}));
    }
    RayBatch rays = RayBatch::create(o, d, 0.1, 1.3);
    MarchingConfig c;
    c.step_size = 0.01;
    c.alpha_thre = 0.0;
    c.early_stop_eps = 0.0;
    AnalyticField field = SolidSphere{ctr, rad, 40.0, {0.9, 0.4, 0.1}};
    auto shade = [&](const PackedSamples& p) {
        SampleAttributes a;
        for (size_t s = 0; s < p.n_samples(); ++s) {
            uint32_t r = p.ray_indices[s];
            auto [rgb, sig] = rgb_sigma_at(field, rays.origins[r] + rays.directions[r] * (0.5 * (p.t_starts[s] + p.t_ends[s])), {});
            a.rgbs.push_back(rgb);
            a.sigmas.push_back(sig);
        }
        return render_forward(p, a);
    };
    RenderOutputs pruned = shade(march(rays, g, field, c));
    RenderOutputs via_cb = shade(march(rays, g, density_sigma(rays, [&](const Vec3& p) { return density_at(field, p); }), c));
    RenderOutputs uni = shade(march_uniform(rays, c));
    for (size_t r = 0; r < rays.n_rays(); ++r) {
        CHECK(norm(pruned.color[r] - uni.color[r]) < 1e-5);
        CHECK(std::fabs(pruned.opacity[r] - uni.opacity[r]) < 1e-5);
        CHECK(pruned.opacity[r] == via_cb.opacity[r]);  // fused == callback path, bit for bit
    }
}

// ------------------------------------------------------------ rendering
TEST("transmittance and closed forms (test_rendering.cpp:73-155)") {
    PackedSamples p;
    p.offsets = {0};
    p.counts = {2};
    p.t_starts = {0.0, 1.0};
    p.t_ends = {1.0, 2.0};
    p.ray_indices = {0, 0};
    auto T = transmittance(p, std::vector<double>{std::log(2.0), 3.0});
    CHECK(T[0] == 1.0 && std::fabs(T[1] - 0.5) < 1e-12);
    SampleAttributes a{{{1, 0, 0}, {0, 1, 0}}, {std::log(2.0), std::log(2.0)}};
    RenderOutputs o = render_forward(p, a);
    CHECK(std::fabs(o.color[0].x - 0.5) < 1e-12 && std::fabs(o.color[0].y - 0.25) < 1e-12);
    CHECK(o.color[0].z == 0.0 && std::fabs(o.opacity[0] - 0.75) < 1e-12);
    CHECK_THROWS_TYPE(transmittance(p, std::vector<double>{1.0}), std::invalid_argument);
    PackedSamples empty;
    empty.offsets = {0, 0};
    empty.counts = {0, 0};
    CHECK((render_forward(empty, SampleAttributes{}).opacity == std::vector<double>{0.0, 0.0}));
}

TEST("forward matches a brute-force recomputation (test_rendering.cpp:157-191)") {
    Rng rng(101);
    for (int trial = 0; trial < 100; ++trial) {
        Instance in = random_instance(rng);
        RenderOutputs o = render_forward(in.p, in.a);
        for (size_t r = 0; r < in.p.n_rays(); ++r) {
            Vec3 col{};
            double op = 0.0, dep = 0.0;
            for (size_t i = in.p.offsets[r]; i < in.p.offsets[r] + in.p.counts[r]; ++i) {
                double tau = 0.0;
                for (size_t j = in.p.offsets[r]; j < i; ++j)
                    tau += in.a.sigmas[j] * (in.p.t_ends[j] - in.p.t_starts[j]);
                double w = std::exp(-tau) * (1.0 - std::exp(-in.a.sigmas[i] * (in.p.t_ends[i] - in.p.t_starts[i])));
                col += in.a.rgbs[i] * w;
                op += w;
                dep += w * 0.5 * (in.p.t_starts[i] + in.p.t_ends[i]);
            }
            for (int k = 0; k < 3; ++k) CHECK(mini::near_rel(o.color[r][k], col[k], 1e-6, 1e-10));
            CHECK(mini::near_rel(o.opacity[r], op, 1e-6, 1e-10));
            CHECK(mini::near_rel(o.depth[r], dep, 1e-6, 1e-10));
            CHECK(o.opacity[r] <= 1.0 + 1e-12);
        }
    }
}

TEST("backward matches central finite differences (test_rendering.cpp:253-293)") {
    Rng rng(113);
    const double h = 1e-4;
    for (int trial = 0; trial < 20; ++trial) {
        Instance in = random_instance(rng, 4, 8);
        size_t n = in.p.n_rays();
        std::vector<Vec3> dc(n);
        std::vector<double> dop(n), ddep(n);
        for (size_t r = 0; r < n; ++r) {
            dc[r] = {rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1)};
            dop[r] = rng.uniform(-1, 1);
            ddep[r] = rng.uniform(-1, 1);
        }
        auto loss = [&](const SampleAttributes& a) {
            RenderOutputs o = render_forward(in.p, a);
            double L = 0.0;
            for (size_t r = 0; r < n; ++r) L += dot(dc[r], o.color[r]) + dop[r] * o.opacity[r] + ddep[r] * o.depth[r];
            return L;
        };
        RenderGradients g = render_backward(in.p, in.a, dc, dop, ddep);
        for (size_t s = 0; s < in.p.n_samples(); ++s) {
            SampleAttributes plus = in.a, minus = in.a;
            plus.sigmas[s] += h;
            minus.sigmas[s] -= h;
            CHECK(mini::near_rel(g.d_sigmas[s], (loss(plus) - loss(minus)) / (2 * h), 1e-5, 1e-8));
        }
    }
}

TEST("render_attribute reproduces opacity and depth (test_rendering.cpp:313-348)") {
    Rng rng(131);
    for (int trial = 0; trial < 30; ++trial) {
        Instance in = random_instance(rng);
        RenderOutputs o = render_forward(in.p, in.a);
        std::vector<double> ones(in.p.n_samples(), 1.0), mids(in.p.n_samples());
        for (size_t s = 0; s < mids.size(); ++s) mids[s] = 0.5 * (in.p.t_starts[s] + in.p.t_ends[s]);
        auto op = render_attribute(in.p, in.a.sigmas, ones, 1);
        auto dep = render_attribute(in.p, in.a.sigmas, mids, 1);
        for (size_t r = 0; r < in.p.n_rays(); ++r) {
            CHECK(mini::near_rel(op[r], o.opacity[r], 1e-12, 1e-15));
            CHECK(mini::near_rel(dep[r], o.depth[r], 1e-12, 1e-15));
        }
    }
    PackedSamples p;
    p.offsets = {0};
    p.counts = {1};
    p.t_starts = {0.0};
    p.t_ends = {0.1};
    p.ray_indices = {0};
    CHECK_THROWS_TYPE(render_attribute(p, std::vector<double>{1.0}, std::vector<double>{1.0, 2.0}, 3),
                      std::invalid_argument);
}

// ------------------------------------------------------------ occupancy grid
TEST("query on fresh and saturated grids (test_occupancy_grid.cpp:32-43)") {
    OccupancyGrid empty(8, kUnit);
    CHECK(!empty.query({0.5, 0.5, 0.5}));
    OccupancyGrid full(8, kUnit, 1e-2, 0.0, 1e6);
    CHECK(full.query({0.5, 0.5, 0.5}) && full.query({0, 0, 0}) && full.query({1, 1, 1}));
    CHECK(!full.query({5, 5, 5}));
    CHECK_THROWS_MSG(full.query({std::nan(""), 0, 0}), std::invalid_argument, "non-finite coordinate");
}

TEST("update: zero, saturating and ball fraction (test_occupancy_grid.cpp:45-66)") {
    OccupancyGrid g(16, kUnit, 1e-2, 0.0, 1e6);
    g.update([](std::span<const Vec3> p) { return std::vector<double>(p.size(), 0.0); }, 0.0);
    CHECK(g.occupied_fraction() == 0.0);
    double sig = 4.0 * g.threshold_density();
    g.update([sig](std::span<const Vec3> p) { return std::vector<double>(p.size(), sig); }, 0.95);
    CHECK(g.occupied_fraction() == 1.0);
    const double ball = 4.0 * M_PI * 0.027 / 3.0;
    OccupancyGrid b(64, kUnit);
    AnalyticField f = SolidSphere{{0.5, 0.5, 0.5}, 0.3, 50.0, {1, 1, 1}};
    for (int i = 0; i < 16; ++i) b.update(f, 0.95, mix_seed(99, uint64_t(i)));
    CHECK(b.occupied_fraction() > 0.8 * ball && b.occupied_fraction() < 1.2 * ball);
}

TEST("center probes are exact on cellwise fields (test_occupancy_grid.cpp:68-84)") {
    OccupancyGrid g(32, kUnit);
    auto fn = [](std::span<const Vec3> p) {
        std::vector<double> out(p.size());
        for (size_t i = 0; i < p.size(); ++i) out[i] = norm(p[i] - Vec3{0.4, 0.6, 0.5}) <= 0.25 ? 30.0 : 0.0;
        return out;
    };
    g.update(fn, 0.0);
    uint32_t R = g.resolution();
    for (uint32_t iz = 0; iz < R; ++iz)
        for (uint32_t iy = 0; iy < R; ++iy)
            for (uint32_t ix = 0; ix < R; ++ix) {
                Vec3 c{(ix + 0.5) / R, (iy + 0.5) / R, (iz + 0.5) / R};
                double s = fn(std::span<const Vec3>(&c, 1))[0];
                CHECK(g.bit(g.cell_index(ix, iy, iz)) == ((1.0 - std::exp(-s * g.reference_step())) > g.alpha_threshold()));
            }
}

TEST("invalid densities name the first offending cell (test_occupancy_grid.cpp:185-194)") {
    OccupancyGrid g(4, kUnit);
    auto bad = [](std::span<const Vec3> p) {
        std::vector<double> out(p.size(), 1.0);
        if (p.size() > 5) out[5] = -2.0;
        return out;
    };
    CHECK_THROWS_MSG(g.update(bad, 0.95), std::runtime_error, "occupancy grid: invalid density at cell (1,1,0)");
    CHECK_THROWS_TYPE(g.update_over_time([](std::span<const Vec3> p, double) { return std::vector<double>(p.size()); },
                                         std::span<const double>(), 0.95),
                      std::invalid_argument);
}

TEST("OGRD round trip is byte identical (test_occupancy_grid.cpp:196-220)") {
    OccupancyGrid g(16, Contraction::sphere({0.5, 0.5, 0.5}, 0.75), 2e-2, 0.001);
    g.update(AnalyticField(SolidSphere{{0.5, 0.5, 0.5}, 0.4, 60.0, {1, 1, 1}}), 0.95, 1234);
    std::stringstream a;
    g.save(a);
    OccupancyGrid l = OccupancyGrid::load(a);
    CHECK(l.resolution() == g.resolution() && l.reference_step() == g.reference_step());
    for (size_t c = 0; c < g.n_cells(); ++c) {
        CHECK(l.bit(c) == g.bit(c));
        CHECK(l.density_cache(c) == double(float(g.density_cache(c))));
    }
    std::stringstream b, c2;
    l.save(b);
    g.save(c2);
    CHECK(b.str() == c2.str());
    OccupancyGrid copy = g;  // value semantics: deep copy of the device grid
    copy.update([](std::span<const Vec3> p) { return std::vector<double>(p.size(), 0.0); }, 0.0);
    CHECK(copy.occupied_fraction() == 0.0 && g.occupied_fraction() > 0.0);
}

int main() { return mini::run_all(); }
