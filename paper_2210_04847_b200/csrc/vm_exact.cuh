// vm_exact.cuh — exact-arithmetic building blocks of the hot path, shared by every
// kernel (and by the host launch code, hence __host__ __device__).
//
// Bit-exactness contract: each expression below performs the
// same IEEE-754 double operations, in the same order, as the reference C++
// (cited per function). The library is compiled with --fmad=false, so no
// multiply-add is ever contracted into an FMA; division and sqrt are the
// correctly-rounded IEEE operations on both sides. The only non-identical
// primitive is exp() (CUDA: <= 1 ulp; glibc: < 1 ulp), which can only move a
// threshold decision when a value sits within ~1 ulp of the threshold.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/vmb200_types.h"

#ifdef __CUDACC__
#define VM_HD __host__ __device__ __forceinline__
#else
#define VM_HD inline
#endif

namespace vmb {

#ifndef __CUDACC__
using std::floor;
using std::isfinite;
using std::sqrt;
#endif

struct D3 {
    double x, y, z;
};

VM_HD D3 d3(double x, double y, double z) { return D3{x, y, z}; }
VM_HD D3 operator+(D3 a, D3 b) { return D3{a.x + b.x, a.y + b.y, a.z + b.z}; }
VM_HD D3 operator-(D3 a, D3 b) { return D3{a.x - b.x, a.y - b.y, a.z - b.z}; }
VM_HD D3 operator*(D3 a, double s) { return D3{a.x * s, a.y * s, a.z * s}; }
VM_HD double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }  // math.hpp:27
VM_HD double norm(D3 a) { return sqrt(dot(a, a)); }                          // math.hpp:31
VM_HD double min_ref(double a, double b) { return (b < a) ? b : a; }         // std::min
VM_HD double max_ref(double a, double b) { return (a < b) ? b : a; }         // std::max
VM_HD bool finite3(D3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

// ----------------------------------------------------------------- contraction
// Device-resident copy of a vmb_contraction with the derived per-axis constants.
struct Contract {
    int kind;
    D3 lo, size;        // AabbNormalize: box.min, box.max - box.min (contraction.cpp:27)
    D3 inv_size;        // 1/size, used ONLY when the axis size is a power of two
    int pow2[3];        // size_k == 2^e exactly -> x/size == x*inv_size bit for bit
    D3 center;          // SphereContract
    double radius;
    int rpow2;          // radius == 2^e exactly -> x/radius == x*inv_radius bit for bit
    double inv_radius;
};

inline Contract make_contract(const vmb_contraction& c) {
    Contract k{};
    k.kind = c.kind;
    k.lo = d3(c.box_min[0], c.box_min[1], c.box_min[2]);
    k.size = d3(c.box_max[0] - c.box_min[0], c.box_max[1] - c.box_min[1],
                c.box_max[2] - c.box_min[2]);
    const double s[3] = {k.size.x, k.size.y, k.size.z};
    double inv[3];
    for (int a = 0; a < 3; ++a) {
        int e = 0;
        double m = frexp(s[a], &e);  // s = m * 2^e, m in [0.5, 1)
        k.pow2[a] = (m == 0.5) && s[a] > 0.0;
        inv[a] = k.pow2[a] ? ldexp(1.0, 1 - e) : 0.0;
    }
    k.inv_size = d3(inv[0], inv[1], inv[2]);
    k.center = d3(c.center[0], c.center[1], c.center[2]);
    k.radius = c.radius;
    {
        int e = 0;
        const double m = frexp(c.radius, &e);
        k.rpow2 = (m == 0.5) && c.radius > 0.0 && e > -1000 && e < 1000;
        k.inv_radius = k.rpow2 ? ldexp(1.0, 1 - e) : 0.0;
    }
    return k;
}

// (x - lo) / size per axis (contraction.cpp:27). Dividing by a power of two and
// multiplying by its exact reciprocal round the same real number, so both
// branches are bit-identical; the multiply avoids the ~10x costlier DP divide.
VM_HD double aabb_axis(double x, double lo, double size, double inv, int pow2) {
    double v = x - lo;
    return pow2 ? v * inv : v / size;
}

// contract() — contraction.cpp:18-30 (caller guarantees a finite point)
VM_HD D3 contract(const Contract& c, D3 x) {
    if (c.kind == VMB_CONTRACT_AABB)
        return d3(aabb_axis(x.x, c.lo.x, c.size.x, c.inv_size.x, c.pow2[0]),
                  aabb_axis(x.y, c.lo.y, c.size.y, c.inv_size.y, c.pow2[1]),
                  aabb_axis(x.z, c.lo.z, c.size.z, c.inv_size.z, c.pow2[2]));
    // (x - center) / radius (contraction.cpp:19); a power-of-two radius divides
    // by multiplying with its exact reciprocal (same real number, same rounding)
    D3 u = c.rpow2 ? d3((x.x - c.center.x) * c.inv_radius, (x.y - c.center.y) * c.inv_radius,
                        (x.z - c.center.z) * c.inv_radius)
                   : d3((x.x - c.center.x) / c.radius, (x.y - c.center.y) / c.radius,
                        (x.z - c.center.z) / c.radius);
    double r = norm(u);
    if (!(r <= 1.0)) u = u * ((2.0 - 1.0 / r) / r);  // contract_to_ball (:18-22)
    return d3((u.x + 2.0) / 4.0, (u.y + 2.0) / 4.0, (u.z + 2.0) / 4.0);
}

// invert_grid_point() — contraction.cpp:37-47; returns false for "nullopt".
VM_HD bool invert(const Contract& c, D3 g, D3* out) {
    if (c.kind == VMB_CONTRACT_AABB) {
        *out = d3(c.lo.x + g.x * c.size.x, c.lo.y + g.y * c.size.y, c.lo.z + g.z * c.size.z);
        return true;
    }
    D3 ball = d3(g.x * 4.0 - 2.0, g.y * 4.0 - 2.0, g.z * 4.0 - 2.0);
    double r = norm(ball);
    if (r <= 1.0) {
        *out = c.center + ball * c.radius;
        return true;
    }
    if (r >= 2.0) return false;
    double world_r = 1.0 / (2.0 - r);
    *out = c.center + ball * (world_r / r * c.radius);
    return true;
}

// Cell lookup of query() — occupancy_grid.cpp:67-76. Returns the linear cell
// index, or -1 when the contracted point leaves [0,1]^3.
VM_HD int64_t cell_of_point(const Contract& c, uint32_t res, D3 x) {
    D3 g = contract(c, x);
    if (g.x < 0.0 || g.x > 1.0 || g.y < 0.0 || g.y > 1.0 || g.z < 0.0 || g.z > 1.0) return -1;
    const double R = double(res);
    uint32_t last = res - 1;
    uint32_t ix = uint32_t(g.x * R), iy = uint32_t(g.y * R), iz = uint32_t(g.z * R);
    ix = ix > last ? last : ix;
    iy = iy > last ? last : iy;
    iz = iz > last ? last : iz;
    return int64_t(ix) + int64_t(res) * (int64_t(iy) + int64_t(res) * int64_t(iz));
}

// ----------------------------------------------------------------- fields
// Analytic fields — fields.cpp:39-73 (+ TimeConditionedField shift, :264-271).
VM_HD bool box_contains(const vmb_field& f, D3 p) {  // math.hpp:57-60
    return p.x >= f.box_min[0] && p.x <= f.box_max[0] && p.y >= f.box_min[1] &&
           p.y <= f.box_max[1] && p.z >= f.box_min[2] && p.z <= f.box_max[2];
}

// TrilinearVoxelField (fields.hpp:47-54 activations; fields.cpp:105-168 stencil).
VM_HD double vox_softplus(double x) { return x > 0.0 ? x + log1p(exp(-x)) : log1p(exp(x)); }
VM_HD double vox_sigmoid(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    double e = exp(x);
    return e / (1.0 + e);
}

// 1/x when x is a normal power of two (exact: x / y == x * (1/y) bit for bit), else 0
VM_HD double pow2_recip(double x) {
#ifdef __CUDA_ARCH__
    const unsigned long long b = __double_as_longlong(x);
#else
    unsigned long long b;
    memcpy(&b, &x, 8);
#endif
    const unsigned long long e = (b >> 52) & 0x7ffull;
    if ((b & 0x800fffffffffffffull) != 0 || e == 0 || e >= 2046) return 0.0;
    const unsigned long long r = (2046ull - e) << 52;
#ifdef __CUDA_ARCH__
    return __longlong_as_double(r);
#else
    double y;
    memcpy(&y, &r, 8);
    return y;
#endif
}

// stencil_at: cell (lower corner vertex) and fractional offsets; false outside
// the box (Aabb::contains, inclusive).
VM_HD bool vox_stencil(const vmb_field& f, D3 p, uint32_t c[3], double fr[3]) {
    if (!box_contains(f, p)) return false;
    const double r1 = double(f.vox_resolution - 1);
    const uint32_t last_cell = f.vox_resolution - 2;
    const double pk[3] = {p.x, p.y, p.z};
    for (int a = 0; a < 3; ++a) {
        // Vec3 rel = (p - min) / box.size() * double(R - 1); a power-of-two size
        // divides exactly by multiplying with its (exact) reciprocal
        const double size = f.box_max[a] - f.box_min[a];
        const double inv = pow2_recip(size);
        const double q = inv != 0.0 ? (pk[a] - f.box_min[a]) * inv : (pk[a] - f.box_min[a]) / size;
        const double rel = q * r1;
        const double fl = floor(rel);
        uint32_t ca = 0;
        if (!(fl < 0.0)) {
            ca = uint32_t(fl);
            ca = ca > last_cell ? last_cell : ca;
        }
        c[a] = ca;
        fr[a] = rel - double(ca);
    }
    return true;
}

// vertex k (dz outer, dy, dx inner) of cell c and its weight wx[dx]*wy[dy]*wz[dz]
VM_HD uint64_t vox_vertex(const vmb_field& f, const uint32_t c[3], int k) {
    const uint64_t R = f.vox_resolution;
    return uint64_t(c[0] + (k & 1)) + R * (uint64_t(c[1] + ((k >> 1) & 1)) + R * uint64_t(c[2] + (k >> 2)));
}
VM_HD double vox_weight(const double fr[3], int k) {
    const double wx = (k & 1) ? fr[0] : 1.0 - fr[0];
    const double wy = ((k >> 1) & 1) ? fr[1] : 1.0 - fr[1];
    const double wz = (k >> 2) ? fr[2] : 1.0 - fr[2];
    return wx * wy * wz;
}

// interpolated raw density (and raw rgb when rgb != nullptr), in stencil order
VM_HD bool vox_raw(const vmb_field& f, D3 p, double* raw_d, D3* raw_c) {
    uint32_t c[3];
    double fr[3];
    if (!vox_stencil(f, p, c, fr)) return false;
    double d = 0.0, r = 0.0, g = 0.0, b = 0.0;
    for (int k = 0; k < 8; ++k) {
        const double w = vox_weight(fr, k);
        const uint64_t v = vox_vertex(f, c, k);
        d += w * f.vox_density[v];
        if (raw_c) {
            r += w * f.vox_color[3 * v];
            g += w * f.vox_color[3 * v + 1];
            b += w * f.vox_color[3 * v + 2];
        }
    }
    *raw_d = d;
    if (raw_c) *raw_c = D3{r, g, b};
    return true;
}

// Field evaluation. Kernels are instantiated with VOX = true only when the field
// is a stored voxel field, so the analytic instantiations never carry the
// stencil's registers; field_density / field_rgb_sigma dispatch at run time.
template <bool VOX>
VM_HD double field_density_t(const vmb_field& f, D3 p);
template <bool VOX>
VM_HD double field_rgb_sigma_t(const vmb_field& f, D3 p, D3* rgb);

// The reference's SolidSphere test compares norm(p - c) = sqrt(d2) with the
// radius. sqrt is correctly rounded and monotone, so when d2 is more than a
// relative 1e-12 away from r^2 the comparison of d2 with r^2 decides it the same
// way; only the thin shell in between takes the sqrt. Returns +1 outside
// (norm > r), -1 inside (norm < r), 0 undecided.
VM_HD int sphere_side(const vmb_field& f, double d2) {
    const double r2 = f.radius * f.radius;
    if (!(r2 > 1e-200 && r2 < 1e200)) return 0;
    if (d2 > r2 * (1.0 + 1e-12)) return 1;
    if (d2 < r2 * (1.0 - 1e-12)) return -1;
    return 0;
}

VM_HD bool sphere_outside(const vmb_field& f, D3 p) {  // norm(p - c) > radius (fields.cpp:45,60)
    const D3 q = p - d3(f.center[0], f.center[1], f.center[2]);
    const double d2 = dot(q, q);  // norm(q) == sqrt(dot(q, q)), math.hpp:30
    const int side = sphere_side(f, d2);
    return side != 0 ? side > 0 : sqrt(d2) > f.radius;
}

VM_HD double field_density_analytic(const vmb_field& f, D3 p) {
    if (f.kind == VMB_FIELD_UNIFORM_BOX) return box_contains(f, p) ? f.sigma : 0.0;
    if (f.kind == VMB_FIELD_SOLID_SPHERE) {  // norm <= r; NaN midpoints never reach here
        const D3 q = p - d3(f.center[0], f.center[1], f.center[2]);
        const double d2 = dot(q, q);
        const int side = sphere_side(f, d2);
        return (side != 0 ? side < 0 : sqrt(d2) <= f.radius) ? f.sigma : 0.0;
    }
    return f.sigma;
}

VM_HD double field_rgb_sigma_analytic(const vmb_field& f, D3 p, D3* rgb) {
    if (f.kind == VMB_FIELD_UNIFORM_BOX || f.kind == VMB_FIELD_SOLID_SPHERE) {
        bool in = f.kind == VMB_FIELD_UNIFORM_BOX
                      ? box_contains(f, p)
                      : !sphere_outside(f, p);
        if (!in) {
            *rgb = d3(0.0, 0.0, 0.0);
            return 0.0;
        }
        *rgb = d3(f.rgb[0], f.rgb[1], f.rgb[2]);
        return f.sigma;
    }
    long long parity = (long long)floor(p.x / f.period) + (long long)floor(p.y / f.period) +
                       (long long)floor(p.z / f.period);
    *rgb = ((parity % 2 + 2) % 2 == 0) ? d3(f.rgb[0], f.rgb[1], f.rgb[2])
                                       : d3(f.rgb_b[0], f.rgb_b[1], f.rgb_b[2]);
    return f.sigma;
}

template <bool VOX>
VM_HD double field_density_t(const vmb_field& f, D3 p) {
    if (VOX && f.kind == VMB_FIELD_VOXEL) {
        double raw;
        return vox_raw(f, p, &raw, nullptr) ? vox_softplus(raw) : 0.0;
    }
    return field_density_analytic(f, p);
}

template <bool VOX>
VM_HD double field_rgb_sigma_t(const vmb_field& f, D3 p, D3* rgb) {
    if (VOX && f.kind == VMB_FIELD_VOXEL) {
        double raw_d;
        D3 raw_c;
        if (!vox_raw(f, p, &raw_d, &raw_c)) {
            *rgb = d3(0.0, 0.0, 0.0);
            return 0.0;
        }
        *rgb = d3(vox_sigmoid(raw_c.x), vox_sigmoid(raw_c.y), vox_sigmoid(raw_c.z));
        return vox_softplus(raw_d);
    }
    return field_rgb_sigma_analytic(f, p, rgb);
}

VM_HD double field_density(const vmb_field& f, D3 p) { return field_density_t<true>(f, p); }
VM_HD double field_rgb_sigma(const vmb_field& f, D3 p, D3* rgb) { return field_rgb_sigma_t<true>(f, p, rgb); }

VM_HD D3 time_shift(const vmb_field& f, D3 p, double t) {  // p - velocity * t
    return p - d3(f.velocity[0], f.velocity[1], f.velocity[2]) * t;
}

// ----------------------------------------------------------------- rng
// splitmix64 / mix_seed / unit_double — rng.hpp:10-24
VM_HD uint64_t splitmix64(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
VM_HD uint64_t mix_seed(uint64_t a, uint64_t b) {
    uint64_t s = a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2));
    return splitmix64(s);
}
VM_HD double unit_double(uint64_t bits) { return double(bits >> 11) * 0x1.0p-53; }

// probe_grid_point — occupancy_grid.cpp:78-89
VM_HD D3 probe_point(uint64_t cell, uint32_t res, bool has_seed, uint64_t seed) {
    uint32_t ix = uint32_t(cell % res);
    uint32_t iy = uint32_t((cell / res) % res);
    uint32_t iz = uint32_t(cell / (uint64_t(res) * res));
    double ox = 0.5, oy = 0.5, oz = 0.5;
    if (has_seed) {
        uint64_t st = mix_seed(seed, cell);
        splitmix64(st);  // Rng ctor discards one draw (rng.hpp:30)
        ox = unit_double(splitmix64(st));
        oy = unit_double(splitmix64(st));
        oz = unit_double(splitmix64(st));
    }
    const double R = double(res);
    return d3((double(ix) + ox) / R, (double(iy) + oy) / R, (double(iz) + oz) / R);
}

// ----------------------------------------------------------------- lattice
// uniform_step_count — ray_marching.cpp:51-55
VM_HD uint64_t uniform_step_count(double near_, double far_, double step) {
    if (!(far_ > near_)) return 0;
    double q = (far_ - near_) / step;
    return uint64_t(ceil(q * (1.0 - 1e-12)));
}

}  // namespace vmb
