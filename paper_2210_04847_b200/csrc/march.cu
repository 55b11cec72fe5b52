// march.cu — occupancy-grid ray marching + sample packing (ray_marching.cpp:57-168).
//
// One thread per ray. For each ray the kernel walks the reference's candidate
// lattice (t0 = near + i*step, t1 = min(near + (i+1)*step, far), midpoint query)
// but only EVALUATES the lattice steps that can possibly be occupied:
//
//   * a coarse DDA (Amanatides-Woo, fp64) walks the 8^3-cell blocks of the grid
//     along the ray, clipped to the domain [0,R]^3 (ray_aabb_intersect);
//   * blocks whose 1-cell-DILATED coarse bit is 0 are skipped wholesale: a point
//     whose ideal position lies in such a block computes (with <= 1e-15 rounding
//     error) to a cell inside the block's halo, all of whose bits are 0, so the
//     reference would reject it too;
//   * every step whose interval [t0,t1] meets an occupied block's t-range (plus
//     one step of slack each side) is evaluated with the reference's exact fp64
//     arithmetic (vm_exact.cuh), in increasing order.
//
// The emitted candidate sequence is therefore identical to the reference's
// per-step scan ("a DDA fast path is permitted but must be
// output-identical"). The density of the analytic field is evaluated inline at
// the same midpoint (sigma_fn_for, voxmarch.cpp:221-232), followed by the alpha
// floor and the transmittance cut (ray_marching.cpp:118-137) — so a ray stops as
// soon as T < eps instead of generating all candidates first.
//
// Packing is count -> CUB-free scan -> fill (the two passes re-walk the same
// rays; both passes together read rays twice, write 8 B/ray + 20 B/sample).
#include <string>
#include <type_traits>

#include "vm_internal.h"
#include "vm_scan.cuh"
#include "vm_bulk.cuh"

namespace vmb {

int check_contraction(const vmb_contraction* c);

namespace {

// BUFFER_FWD = BUFFER + the render_forward compositing of each kept sample, done
// in filter_sample as the sample is kept (vmb_march_render_field).
enum Mode { COUNT = 0, FILL = 1, BUFFER = 2, BUFFER_FWD = 3 };
#ifndef VMB_WALK_THREADS
#define VMB_WALK_THREADS 128
#endif
constexpr int kAccStride = VMB_WALK_THREADS;  // = the walk kernel's block size
// k_march_walk's per-thread shared-memory slots, at namespace scope so every access
// is indexed by threadIdx.x (two generic pointers held in the Sink cost registers and
// spills under the 64-register cap): the six fused-forward accumulators (k = Tf, r,
// g, b, opacity, depth) and the ray's twelve fp32 constants (A, B, o, d; RSMM).
__shared__ double walk_acc[6][kAccStride];
__shared__ float walk_rc[12][kAccStride];
#define WACC(k) walk_acc[k][threadIdx.x]
#define WRC(k) walk_rc[k][threadIdx.x]
// bit 2 of a mode: the kernel evaluates a stored voxel field (field_density_t<true>)
constexpr int VOXM = 4;
__host__ __device__ constexpr int mbase(int m) { return m & 3; }
__host__ __device__ constexpr bool mvox(int m) { return (m & VOXM) != 0; }
// bit 3: k_march_walk holds the constant-density alpha table (P.atab_n entries) in
// its dynamic shared memory, walk_dyn_smem
constexpr int ATABM = 8;
__host__ __device__ constexpr bool matab(int m) { return (m & ATABM) != 0; }
// bit 4: walk_fast keeps the ray's fp32 constants (A, B, o, d) in the caller's
// shared-memory slot Sink::rc, read back where used, instead of leaving the register
// allocator to rematerialize them from the fp64 ray in every loop iteration
constexpr int RSMM = 16;
__host__ __device__ constexpr bool mrsm(int m) { return (m & RSMM) != 0; }
// bit 5: vmb_march_cascade's accumulated-t walk (stacked levels / cone stepping),
// in its own k_march instantiations so the other walks keep their register budget
constexpr int EXTM = 32;
__host__ __device__ constexpr bool mext(int m) { return (m & EXTM) != 0; }
// bit 7 (FILL, k_march): the slab pass of a long-ray walk (k_march's comment)
constexpr int SLABM = 128;
__host__ __device__ constexpr bool mslab(int m) { return (m & SLABM) != 0; }
// bit 6 (BUFFER_FWD): each kept sample's rgb/sigma, rounded to the attribute dtype,
// also go to the walk's scratch beside its lattice index, so the expansion copies
// them instead of evaluating a non-constant field a second time (Sink::attr)
constexpr int ATTRM = 64;
__host__ __device__ constexpr bool mattr(int m) { return (m & ATTRM) != 0; }
extern __shared__ double walk_dyn_smem[];

constexpr int kMaxLevels = 8;  // vmb_march_ext: level 0 + up to 7 nested levels

struct MarchParams {
    Contract k;
    uint32_t res;
    const uint32_t* bits;
    const uint32_t* coarse;
    const vmb_grid* grid;  // for grid_ensure_coarse (walk_skip)
    const uint8_t* dist;  // capped L-inf distance to the nearest occupied cell
    const uint32_t* bbox; // occupied cells' bounding box {min xyz, max+1 xyz} (vmb_grid::bbox)
    uint32_t block, res_c;
    double scale[3];      // R / size_k: world -> fine-cell units (approximate, DDA only)
    double near_, far_, step;
    uint64_t n_steps;     // lattice length after the host-side !(t1 > t0) check
    bool skip;            // DDA empty-space skipping allowed (AABB, bounded lattice)
    bool grows;           // SphereContract && growth > 1 (ray_marching.cpp:60-61)
    double growth;
    D3 ball_c;
    double ball_r;
    // filtered growth test: |q|^2 outside [r2_lo, r2_hi] decides norm(q) > r
    // without the sqrt (r^2 (1 -+ 2^-40): far beyond the roundings of r^2 and
    // of the correctly rounded sqrt); ball_filter = false when r^2 is not a
    // well-scaled normal number
    bool ball_filter;
    double ball_r2_lo, ball_r2_hi;
    double eps, thr;
    uint32_t max_cand;
    bool fast;            // fp32 DDA + filtered fp32 cell test (walk_fast)
    bool f32_safe;        // max(|near|, |far|) < 1e250: every f32 ray passes ray_safe
    bool sphere_fast;     // SolidSphere field: filtered fp32 density decision
    uint32_t atab_n;      // k_march_walk: alpha + midpoint table length (n_steps, sphere_fast only) or 0
    bool tab_same32;      // the SolidSphere sigma is exact in fp32 (attribute dtype f32: same alpha, same T)
    float sph_c[3], sph_r, sph_r2, sph_cmax;
    double sph_sig32, sph_rgb32[3];  // SolidSphere sigma / rgb rounded through fp32 (fused forward)
    float step_f, m0_f, inv_step_f, near_f, far_f, Mf;
    bool full;            // walk to the end (stats / candidate mode), ignore the T cut
    bool filter;          // apply inline density + alpha floor + T cut
    vmb_field f;
    // Multi-level grid (NerfAcc cascades, vmb_march_cascade): levels 1..n_lv are AABB
    // grids nested around level 0 (k / res / bits above); a point is decided by the
    // FINEST level whose domain contains it (level 0 first: with n_lv = 0 this is
    // OccupancyGrid::query exactly, occupancy_grid.cpp:67-76).
    uint32_t n_lv;
    Contract lv_k[kMaxLevels - 1];
    uint32_t lv_res[kMaxLevels - 1];
    const uint32_t* lv_bits[kMaxLevels - 1];
    // accumulated-t walk (walk_growth) for cascades / cone stepping, not only growth
    bool accum;
    // cone stepping: dt = min(max(t cone_angle, step), max_step) at each interval's t
    bool cone;
    double cone_angle, max_step;
    // the outermost level is an AABB: a midpoint outside it on an axis the ray does
    // not come back along ends the walk (every later midpoint is outside every level)
    bool exit_box;
    // empty-space skipping of walk_ext (every level an AABB grid, no growth): per
    // level (0 = the base grid) its box origin and cells per world unit, the box of
    // the level below in this level's cell units, and its distance map
    bool ext_skip;
    struct {
        double lo[3], scale[3];
        float in_lo[3], in_hi[3];
    } xs[kMaxLevels];
    const uint8_t* lv_dist[kMaxLevels - 1];
};

template <typename T>
__device__ __forceinline__ D3 load3(const T* p, uint64_t i) {
    return d3(double(p[3 * i]), double(p[3 * i + 1]), double(p[3 * i + 2]));
}

__device__ __forceinline__ bool fine_bit(const uint32_t* bits, int64_t c) {
    return (__ldg(bits + (uint64_t(c) >> 5)) >> (uint64_t(c) & 31)) & 1u;
}

// Per-ray consumer of candidate intervals: alpha floor + transmittance cut and
// output (count or fill). Returns false when the ray is finished.
constexpr int kStgStride = 128;  // k_march's block size

struct Sink {
    uint64_t ray;
    uint32_t n_cand = 0;   // candidates seen (emitted)
    uint32_t n_kept = 0;
    double T = 1.0;
    bool filtering = true; // false after the T cut (stats walk continues)
    // FILL
    double* ts = nullptr;
    double* te = nullptr;
    uint32_t* idx = nullptr;
    uint64_t base = 0;
    uint64_t cap = 0;
    // FILL staging (k_march): a lane's samples are collected per aligned group of 4
    // output slots in shared memory (stg[k * kStgStride], k = slot & 3: t0 at +0,
    // t1 at +4 * kStgStride) and a complete group goes out as 16-byte vector stores;
    // per-sample scalar stores from 32 lanes at 32 unrelated addresses were the
    // two-pass fill's bound (partial-sector writes: 1.6x the algorithmic DRAM bytes).
    double* stg = nullptr;
    bool vec = false;  // ts/te/idx 16-byte aligned

    __device__ __forceinline__ void put(double t0, double t1) {
        const uint64_t o = base + n_kept;
        if (o >= cap) return;
        if (!stg) {
            ts[o] = t0;
            te[o] = t1;
            idx[o] = uint32_t(ray);
            return;
        }
        const int k = int(o & 3);
        stg[k * kStgStride] = t0;
        stg[(4 + k) * kStgStride] = t1;
        if (k == 3) flush_group(o - 3 >= base ? o - 3 : base, o + 1);
    }
    // slots [lo, hi) of one aligned group of 4, all < cap
    __device__ __forceinline__ void flush_group(uint64_t lo, uint64_t hi) {
        if (vec && hi - lo == 4) {
            const double2 a0 = make_double2(stg[0], stg[kStgStride]);
            const double2 a1 = make_double2(stg[2 * kStgStride], stg[3 * kStgStride]);
            const double2 b0 = make_double2(stg[4 * kStgStride], stg[5 * kStgStride]);
            const double2 b1 = make_double2(stg[6 * kStgStride], stg[7 * kStgStride]);
            reinterpret_cast<double2*>(ts + lo)[0] = a0;
            reinterpret_cast<double2*>(ts + lo)[1] = a1;
            reinterpret_cast<double2*>(te + lo)[0] = b0;
            reinterpret_cast<double2*>(te + lo)[1] = b1;
            const uint32_t r = uint32_t(ray);
            *reinterpret_cast<uint4*>(idx + lo) = make_uint4(r, r, r, r);
            return;
        }
        for (uint64_t q = lo; q < hi; ++q) {
            const int k = int(q & 3);
            ts[q] = stg[k * kStgStride];
            te[q] = stg[(4 + k) * kStgStride];
            idx[q] = uint32_t(ray);
        }
    }
    // after the walk: the incomplete last group
    __device__ __forceinline__ void flush_tail() {
        if (!stg) return;
        uint64_t e = base + n_kept;
        if (e > cap) e = cap;
        if (e <= base || (e & 3) == 0) return;
        const uint64_t g = e & ~uint64_t(3);
        flush_group(g > base ? g : base, e);
    }
    // BUFFER (fused single-pass kernel): kept lattice indices go to shared memory
    uint32_t* buf = nullptr;
    uint32_t buf_stride = 0;
    uint32_t buf_cap = 0;
    // BUFFER_FWD: rendering.cpp:47-58 accumulators (Tf follows the attribute-dtype
    // sigma, T the march's fp64 sigma; they differ only if sigma is not exact in it)
    // The six accumulators live in shared memory (acc[k * kAccStride], k = Tf, r, g,
    // b, opacity, depth): they are touched only per kept sample, and keeping them
    // out of registers leaves the walk loop its 64 registers.
    bool at32 = false;
    void* attr = nullptr;  // ATTRM: float4 / double4 rows beside buf (same stride)

    // One kept sample, with exactly k_shade + k_forward's expressions (FwdAcc):
    // sigma/rgb are rounded to the attribute dtype; alpha is reused when the
    // rounding is exact (same expression, same operands).
    __device__ __forceinline__ void composite(double sigma, D3 c, double t0, double t1, double alpha) {
        if (at32)
            composite_rounded(sigma, double(float(sigma)), d3(double(float(c.x)), double(float(c.y)), double(float(c.z))),
                              t0, t1, alpha);
        else
            composite_rounded(sigma, sigma, c, t0, t1, alpha);
    }
    // sg / c already rounded to the attribute dtype (constant-field fast path)
    __device__ __forceinline__ void composite_rounded(double sigma, double sg, D3 c, double t0, double t1,
                                                      double alpha) {
        const double a = sg == sigma ? alpha : 1.0 - exp(-sg * (t1 - t0));
        const double Tf = WACC(0);
        const double w = Tf * a;
        WACC(1) = WACC(1) + c.x * w;
        WACC(2) = WACC(2) + c.y * w;
        WACC(3) = WACC(3) + c.z * w;
        WACC(4) += w;
        WACC(5) += w * 0.5 * (t0 + t1);
        WACC(0) = Tf * (1.0 - a);
    }
};

template <int MODE>
__device__ __forceinline__ bool filter_sample(const MarchParams& P, Sink& s, uint64_t i, uint32_t ci,
                                              double t0, double t1, double sigma, DevError* err,
                                              D3 rgb = D3{0.0, 0.0, 0.0}, bool rounded = false,
                                              double sg_r = 0.0, double alpha_pre = -1.0);

// Handles one grid-passing candidate. Mirrors ray_marching.cpp:78,111-137.
template <int MODE>
__device__ __forceinline__ bool on_candidate(const MarchParams& P, Sink& s, uint64_t i, double t0,
                                             double t1, D3 p, DevError* err) {
    if (s.n_cand >= P.max_cand) return false;  // candidate cap (:78 / :91)
    uint32_t ci = s.n_cand++;
    if (!P.filter) {  // candidate mode: keep every grid-passing interval
        if (mbase(MODE) == FILL) {
            s.put(t0, t1);
        }
        if (mbase(MODE) >= BUFFER && s.n_kept < s.buf_cap) s.buf[s.n_kept * s.buf_stride] = uint32_t(i);
        s.n_kept++;
        return true;
    }
    if (!s.filtering) return true;  // after the cut only the emitted count matters
    if (mbase(MODE) == BUFFER_FWD) {  // field_rgb_sigma's sigma == field_density's for finite p
        D3 c;
        const double sg = field_rgb_sigma_t<mvox(MODE)>(P.f, p, &c);
        return filter_sample<MODE>(P, s, i, ci, t0, t1, sg, err, c);
    }
    return filter_sample<MODE>(P, s, i, ci, t0, t1, field_density_t<mvox(MODE)>(P.f, p), err);
}

// Density validation, alpha floor and transmittance cut of candidate ci with
// density sigma (ray_marching.cpp:122-137).
template <int MODE>
__device__ __forceinline__ bool filter_sample(const MarchParams& P, Sink& s, uint64_t i, uint32_t ci,
                                              double t0, double t1, double sigma, DevError* err,
                                              D3 rgb, bool rounded, double sg_r, double alpha_pre) {
    if (!isfinite(sigma) || sigma < 0.0) {
        int kind = !isfinite(sigma) ? ERR_NONFINITE_SIGMA : ERR_NEGATIVE_SIGMA;
        atomicMin(&err->key, march_err_key(s.ray, ci, kind));
        s.filtering = false;
        return false;
    }
    // sigma == 0: alpha = 1 - exp(-0 * delta) = 0 exactly, never above a floor >= 0
    if (sigma == 0.0 && P.thr >= 0.0) return true;
    // alpha_pre: the same expression evaluated ahead (constant-density table)
    const double alpha = alpha_pre >= 0.0 ? alpha_pre : 1.0 - exp(-sigma * (t1 - t0));
    if (alpha <= P.thr) return true;
    if (mbase(MODE) == FILL) {
        s.put(t0, t1);
    }
    if (mbase(MODE) >= BUFFER && s.n_kept < s.buf_cap) s.buf[s.n_kept * s.buf_stride] = uint32_t(i);
    if (mbase(MODE) == BUFFER_FWD) {
        if (rounded)
            s.composite_rounded(sigma, sg_r, rgb, t0, t1, alpha);
        else
            s.composite(sigma, rgb, t0, t1, alpha);
        if (mattr(MODE) && s.n_kept < s.buf_cap) {  // k_shade's AT(rgb), AT(sigma) of this sample
            if (s.at32)
                static_cast<float4*>(s.attr)[s.n_kept * s.buf_stride] =
                    make_float4(float(rgb.x), float(rgb.y), float(rgb.z), float(sigma));
            else
                static_cast<double4*>(s.attr)[s.n_kept * s.buf_stride] = make_double4(rgb.x, rgb.y, rgb.z, sigma);
        }
    }
    s.n_kept++;
    s.T *= 1.0 - alpha;
    if (s.T < P.eps) {
        s.filtering = false;
        return P.full;  // continue only to count emitted candidates
    }
    return true;
}

// Exact evaluation of lattice step i (ray_marching.cpp:79-86). Returns false on a
// non-finite midpoint (query() throws "non-finite coordinate").
template <int MODE>
__device__ __forceinline__ bool eval_step(const MarchParams& P, Sink& s, D3 o, D3 d, uint64_t i,
                                          DevError* err, bool* alive) {
    double t0 = P.near_ + double(i) * P.step;
    double t1 = min_ref(P.near_ + double(i + 1) * P.step, P.far_);
    double m = 0.5 * (t0 + t1);
    D3 p = o + d * m;
    if (!finite3(p)) {
        atomicMin(&err->key, march_err_key(s.ray, 0, ERR_NONFINITE_COORD));
        *alive = false;
        return false;
    }
    int64_t c = cell_of_point(P.k, P.res, p);
    if (c >= 0 && fine_bit(P.bits, c)) {
        if (!on_candidate<MODE>(P, s, i, t0, t1, p, err)) {
            *alive = false;
            return false;
        }
    }
    return true;
}

__device__ __forceinline__ bool coarse_bit(const MarchParams& P, int cx, int cy, int cz) {
    uint32_t kc = uint32_t(cx) + P.res_c * (uint32_t(cy) + P.res_c * uint32_t(cz));
    return (__ldg(P.coarse + (kc >> 5)) >> (kc & 31)) & 1u;
}

// Bounded lattice with empty-space skipping (see file comment).
template <int MODE>
__device__ void walk_skip(const MarchParams& P, Sink& s, D3 o, D3 d, DevError* err) {
    if (P.n_steps == 0) return;
    const double R = double(P.res);
    const double EPS = 1e-6;  // fine cells; >> 1e-15 rounding, << 1 cell halo
    double A[3] = {(o.x - P.k.lo.x) * P.scale[0], (o.y - P.k.lo.y) * P.scale[1],
                   (o.z - P.k.lo.z) * P.scale[2]};
    double B[3] = {d.x * P.scale[0], d.y * P.scale[1], d.z * P.scale[2]};
    double tlo = P.near_, thi = P.far_;
#pragma unroll
    for (int a = 0; a < 3; ++a) {  // ray_aabb_intersect against [-EPS, R+EPS]^3
        if (B[a] == 0.0) {
            if (A[a] < -EPS || A[a] > R + EPS) return;
        } else {
            double ta = (-EPS - A[a]) / B[a], tb = (R + EPS - A[a]) / B[a];
            if (ta > tb) {
                double x = ta;
                ta = tb;
                tb = x;
            }
            tlo = fmax(tlo, ta);
            thi = fmin(thi, tb);
        }
    }
    if (!(tlo <= thi)) return;
    const double Bs = double(P.block);
    const int Rc = int(P.res_c);
    int c[3], stp[3];
    double tmax[3], tdel[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double pa = A[a] + B[a] * tlo;
        int ca = int(floor(pa / Bs));
        ca = ca < 0 ? 0 : (ca >= Rc ? Rc - 1 : ca);
        c[a] = ca;
        if (B[a] > 0.0) {
            stp[a] = 1;
            tmax[a] = (double(ca + 1) * Bs - A[a]) / B[a];
            tdel[a] = Bs / B[a];
        } else if (B[a] < 0.0) {
            stp[a] = -1;
            tmax[a] = (double(ca) * Bs - A[a]) / B[a];
            tdel[a] = -Bs / B[a];
        } else {
            stp[a] = 0;
            tmax[a] = INFINITY;
            tdel[a] = INFINITY;
        }
    }
    const double inv_step = 1.0 / P.step;
    const int64_t last = int64_t(P.n_steps) - 1;
    int64_t next_i = 0;
    double t = tlo;
    bool alive = true;
    for (int guard = 0; guard < 4 * (3 * Rc + 3); ++guard) {
        double tn = fmin(fmin(tmax[0], tmax[1]), fmin(tmax[2], thi));
        if (coarse_bit(P, c[0], c[1], c[2])) {
            double tb = fmax(tn, t);
            int64_t jlo = int64_t(floor((t - P.near_) * inv_step)) - 1;
            int64_t jhi = int64_t(floor((tb - P.near_) * inv_step)) + 1;
            if (jlo < next_i) jlo = next_i;
            if (jhi > last) jhi = last;
            for (int64_t j = jlo; j <= jhi; ++j)
                if (!eval_step<MODE>(P, s, o, d, uint64_t(j), err, &alive)) return;
            if (jhi + 1 > next_i) next_i = jhi + 1;
            if (next_i > last) return;
        }
        if (tn >= thi) return;
        if (tmax[0] <= tmax[1] && tmax[0] <= tmax[2]) {
            c[0] += stp[0];
            if (c[0] < 0 || c[0] >= Rc) return;
            tmax[0] += tdel[0];
        } else if (tmax[1] <= tmax[2]) {
            c[1] += stp[1];
            if (c[1] < 0 || c[1] >= Rc) return;
            tmax[1] += tdel[1];
        } else {
            c[2] += stp[2];
            if (c[2] < 0 || c[2] >= Rc) return;
            tmax[2] += tdel[2];
        }
        t = tn;
    }
}

// Bounded lattice, every step evaluated (sphere contraction / unsafe inputs).
template <int MODE>
__device__ void walk_dense(const MarchParams& P, Sink& s, D3 o, D3 d, DevError* err) {
    bool alive = true;
    for (uint64_t i = 0; i < P.n_steps; ++i)
        if (!eval_step<MODE>(P, s, o, d, i, err, &alive)) return;
}

// Cascade query of one midpoint: 1 occupied, 0 empty / outside every level, -1
// outside the outermost (AABB) level on an axis the ray does not come back along.
// The computed midpoint o + d m is monotone in m per axis (both roundings are),
// and so is the AABB contraction (x - lo) / size, so once the outermost level
// rejects it that way it rejects every later midpoint; the inner levels are
// nested inside it with a margin of whole cells (checked on the host).
__device__ __forceinline__ int cascade_query(const MarchParams& P, D3 p, D3 d) {
    int64_t c = cell_of_point(P.k, P.res, p);
    if (c >= 0) return fine_bit(P.bits, c);
    for (uint32_t l = 0; l < P.n_lv; ++l) {
        c = cell_of_point(P.lv_k[l], P.lv_res[l], p);
        if (c >= 0) return fine_bit(P.lv_bits[l], c);
    }
    if (P.exit_box) {
        const Contract& k = P.n_lv ? P.lv_k[P.n_lv - 1] : P.k;
        const D3 g = contract(k, p);
        if ((g.x > 1.0 && d.x >= 0.0) || (g.x < 0.0 && d.x <= 0.0) || (g.y > 1.0 && d.y >= 0.0) ||
            (g.y < 0.0 && d.y <= 0.0) || (g.z > 1.0 && d.z >= 0.0) || (g.z < 0.0 && d.z <= 0.0))
            return -1;
    }
    return 0;
}

// cascade_query that also reports the deciding level (0 = base) and its cell
__device__ __forceinline__ int cascade_locate(const MarchParams& P, D3 p, D3 d, int* lev, int64_t* cell) {
    int64_t c = cell_of_point(P.k, P.res, p);
    if (c >= 0) {
        *lev = 0, *cell = c;
        return fine_bit(P.bits, c);
    }
    for (uint32_t l = 0; l < P.n_lv; ++l) {
        c = cell_of_point(P.lv_k[l], P.lv_res[l], p);
        if (c >= 0) {
            *lev = int(l) + 1, *cell = c;
            return fine_bit(P.lv_bits[l], c);
        }
    }
    *lev = -1;
    if (P.exit_box) {
        const Contract& k = P.n_lv ? P.lv_k[P.n_lv - 1] : P.k;
        const D3 g = contract(k, p);
        if ((g.x > 1.0 && d.x >= 0.0) || (g.x < 0.0 && d.x <= 0.0) || (g.y > 1.0 && d.y >= 0.0) ||
            (g.y < 0.0 && d.y <= 0.0) || (g.z > 1.0 && d.z >= 0.0) || (g.z < 0.0 && d.z <= 0.0))
            return -1;
    }
    return 0;
}

// Geometric step growth outside the unit ball (ray_marching.cpp:88-106).
template <int MODE>
__device__ void walk_growth(const MarchParams& P, Sink& s, D3 o, D3 d, DevError* err) {
    double t = P.near_, dt = P.step;
    while (t < P.far_ && s.n_cand < P.max_cand) {
        double t1 = min_ref(t + dt, P.far_);
        if (!(t1 > t)) break;
        D3 mid = o + d * (0.5 * (t + t1));
        if (!finite3(mid)) {
            atomicMin(&err->key, march_err_key(s.ray, 0, ERR_NONFINITE_COORD));
            return;
        }
        int64_t c = cell_of_point(P.k, P.res, mid);
        if (c >= 0 && fine_bit(P.bits, c))
            if (!on_candidate<MODE>(P, s, s.n_cand, t, t1, mid, err)) return;
        t += dt;
        const D3 q = mid - P.ball_c;
        const double q2 = dot(q, q);  // norm() = sqrt(dot(q, q)), math.hpp:31
        const bool outside = P.ball_filter && q2 > P.ball_r2_hi   ? true
                             : P.ball_filter && q2 < P.ball_r2_lo ? false
                                                                  : sqrt(q2) > P.ball_r;
        if (outside)
            dt *= P.growth;
        else
            dt = P.step;
    }
}

// The accumulated-t walk of vmb_march_cascade (k_march instantiations with EXTM):
// the growth walk's arithmetic (t += dt, t1 = min(t + dt, far)) with NerfAcc's cone
// rule dt = min(max(t cone_angle, step), max_step) at each interval's t, or the
// growth rule (sphere level 0), over a cascade of nested levels.
template <int MODE>
__device__ void walk_ext(const MarchParams& P, Sink& s, D3 o, D3 d, DevError* err) {
    double t = P.near_, dt = P.step;
    while (t < P.far_ && s.n_cand < P.max_cand) {
        if (P.cone) dt = fmin(fmax(t * P.cone_angle, P.step), P.max_step);
        double t1 = min_ref(t + dt, P.far_);
        if (!(t1 > t)) break;
        D3 mid = o + d * (0.5 * (t + t1));
        if (!finite3(mid)) {
            atomicMin(&err->key, march_err_key(s.ray, 0, ERR_NONFINITE_COORD));
            return;
        }
        int lev;
        int64_t cell;
        const int q = cascade_locate(P, mid, d, &lev, &cell);
        if (q < 0) return;
        if (q && !on_candidate<MODE>(P, s, s.n_cand, t, t1, mid, err)) return;
        const double mt0 = 0.5 * (t + t1);
        t += dt;
        if (!P.grows) {
            // Empty-space skipping: the deciding level's cell is empty with distance
            // D >= 2 to its nearest occupied cell, so every point within D - 1 cells
            // of this midpoint (that is still decided by this level: inside its box,
            // outside the box of the level below) is an empty cell. The next steps
            // whose midpoints stay within that reach are not candidates: only their
            // t recurrence runs (t += dt, the same fp64 sequence), not their queries.
            // Bounds in fp32 cell units with 1e-3-cell margins (the positions'
            // rounding is ~1e-5 cells) and a 1e-4 relative shrink.
            if (P.ext_skip && q == 0 && lev >= 0) {
                const int D = __ldg((lev == 0 ? P.dist : P.lv_dist[lev - 1]) + cell);
                if (D >= 2) {
                    const auto& X = P.xs[lev];
                    const float Rl = float(lev == 0 ? P.res : P.lv_res[lev - 1]);
                    // cell coordinates from fp64 (a far-off box must not lose them to fp32)
                    const float u0 = float((mid.x - X.lo[0]) * X.scale[0]), B0 = float(d.x * X.scale[0]);
                    const float u1 = float((mid.y - X.lo[1]) * X.scale[1]), B1 = float(d.y * X.scale[1]);
                    const float u2 = float((mid.z - X.lo[2]) * X.scale[2]), B2 = float(d.z * X.scale[2]);
                    const float bmax = fmaxf(fmaxf(fabsf(B0), fabsf(B1)), fabsf(B2));
                    float lim = (float(D) - 1.001f) / bmax;  // bmax == 0: +inf
                    auto wall = [&](float u, float B) {     // stay inside this level's box
                        if (B > 0.0f) lim = fminf(lim, (Rl - 1e-3f - u) / B);
                        if (B < 0.0f) lim = fminf(lim, (u - 1e-3f) / -B);
                    };
                    wall(u0, B0), wall(u1, B1), wall(u2, B2);
                    if (lev > 0) {  // stay outside the box of the level below (L-inf gap)
                        const float gap = fmaxf(fmaxf(fmaxf(X.in_lo[0] - u0, u0 - X.in_hi[0]),
                                                      fmaxf(X.in_lo[1] - u1, u1 - X.in_hi[1])),
                                                fmaxf(X.in_lo[2] - u2, u2 - X.in_hi[2]));
                        lim = fminf(lim, (gap - 1e-3f) / bmax);
                    }
                    const double reach = double(lim) * 0.9999;
                    if (reach > 0.0) {
                        while (t < P.far_) {
                            if (P.cone) dt = fmin(fmax(t * P.cone_angle, P.step), P.max_step);
                            const double t1n = min_ref(t + dt, P.far_);
                            if (!(t1n > t) || 0.5 * (t + t1n) - mt0 > reach) break;
                            t += dt;
                        }
                    }
                }
            }
            continue;
        }
        const D3 b = mid - P.ball_c;
        const double b2 = dot(b, b);
        const bool outside = P.ball_filter && b2 > P.ball_r2_hi   ? true
                             : P.ball_filter && b2 < P.ball_r2_lo ? false
                                                                  : sqrt(b2) > P.ball_r;
        if (outside)
            dt *= P.growth;
        else
            dt = P.step;
    }
}

// ---------------------------------------------------------------------------
// Fast walk (AABB, bounded lattice): fp32 coarse DDA + FILTERED fp32 cell test.
//
// For lattice step j the cell coordinate along axis a is u_a = A_a + B_a * m_j
// (fine-cell units, A = (o - lo) R / size, B = d R / size, m_j the step midpoint).
// It is evaluated in fp32 with one FMA; the fp32 value differs from the real value
// by at most E = 2^-22 (2 max|A| + 5 max|B| M) (a >3x over-estimate of the
// rounding of A, B, m and the FMA; M = max(|near|, |far|)), while the reference's
// fp64 evaluation differs from the real value by ~1e-13 cells. Hence when every
// fp32 coordinate is more than E away from an integer, floor() of the fp32 value
// IS the reference's cell (and its in/out-of-domain decision). Otherwise — and
// for the last, possibly far-clamped step — the step is re-evaluated with the
// exact fp64 code (eval_step). Candidates always get exact t0/t1/midpoint.
// ---------------------------------------------------------------------------
template <int MODE, typename RT>
__device__ void walk_fast(const MarchParams& P, Sink& s, const RT* __restrict__ orig,
                          const RT* __restrict__ dirs, uint64_t r, DevError* err) {
    if (P.n_steps == 0) return;
    const float Rf = float(P.res);
    // Only fp32 state stays live in the loops; the fp64 ray is re-read from
    // global memory (L1) by the rare exact paths.
    float A[3], B[3], Q[3];
    // SolidSphere: the squared distance to the centre along the ray as a quadratic
    // in the midpoint parameter, |o + d m - c|^2 = a m^2 + b m + c0 (coefficients in
    // fp64, evaluated in fp32 by two FMAs), with its error bound sph_err:
    //   the midpoint's fp32 error |dm| <= 6 2^-24 M (M = max(|near|, |far|)) moves the
    //   quadratic by <= (2 a M + |b|) |dm|; the coefficients' rounding, the two FMAs'
    //   and r^2's add <= 4 2^-24 (a M^2 + |b| M + c0 + r^2); the reference's fp64
    //   evaluation is within ~1e-15 of it; a factor 4 of headroom on top.
    float sph_err = 0.0f;
    {
        const D3 o = load3(orig, r), d = load3(dirs, r);
        A[0] = float((o.x - P.k.lo.x) * P.scale[0]);
        A[1] = float((o.y - P.k.lo.y) * P.scale[1]);
        A[2] = float((o.z - P.k.lo.z) * P.scale[2]);
        B[0] = float(d.x * P.scale[0]);
        B[1] = float(d.y * P.scale[1]);
        B[2] = float(d.z * P.scale[2]);
        Q[0] = Q[1] = Q[2] = 0.0f;
        if (P.sphere_fast) {
            const D3 oc = o - d3(P.f.center[0], P.f.center[1], P.f.center[2]);
            const double qa = dot(d, d), qb = 2.0 * dot(oc, d), qc = dot(oc, oc);
            const double M = double(P.Mf), r2 = P.f.radius * P.f.radius;
            const double bound = (2.0 * qa * M + fabs(qb)) * 6.0 * M + 4.0 * (qa * M * M + fabs(qb) * M + qc + r2);
            Q[0] = float(qa), Q[1] = float(qb), Q[2] = float(qc);
            sph_err = float(4.0 * 0x1p-24 * bound * (1.0 + 1e-6)) + 1e-12f;
        }
    }
    // the loop evaluates v = u - 1/2 (cell coordinate minus one half): the cell is
    // rint(v), decided when every |v - rint(v)| <= 1/2 - E (one max, one compare)
    float Ah[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) Ah[a] = A[a] - 0.5f;
    if (mrsm(MODE)) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            WRC(a) = Ah[a];
            WRC(3 + a) = B[a];
            WRC(6 + a) = Q[a];
        }
    }
    // the constants where they are used: from the shared slot (RSMM) or registers
#define VM_RC(k, reg) (mrsm(MODE) ? WRC(k) : (reg))
    const float amax = fmaxf(fmaxf(fabsf(A[0]), fabsf(A[1])), fabsf(A[2]));
    const float bmax = fmaxf(fmaxf(fabsf(B[0]), fabsf(B[1])), fabsf(B[2]));
    // (scalings by powers of two are exact: x * 2^-22 == ldexpf(x, -22))
    // (+ 2^-24 (amax + 1): the rounding of A - 1/2)
    const float E = (2.0f * amax + 5.0f * bmax * P.Mf) * 0x1p-22f + (amax + 1.0f) * 0x1p-24f + 1e-6f;
    const bool fast_ok = E < 0.05f;
    const float half_E = 0.5f - E;
    const float EPSD = 1e-3f + 4.0f * E;  // guard for the fp32 clip
    // ray_aabb_intersect against the guarded bounding box of the occupied cells
    // (inside the domain [0, R]^3): every lattice step outside it is an empty cell
    // or outside the domain, so the walk covers only the clipped range (+2 steps)
    float tlo = P.near_f, thi = P.far_f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const uint32_t b0 = __ldg(P.bbox + a), b1 = __ldg(P.bbox + 3 + a);
        if (b0 >= b1) return;  // no occupied cell: no candidate anywhere
        const float lo = float(b0) - EPSD, hi = fminf(float(b1), Rf) + EPSD;
        if (B[a] == 0.0f) {
            if (A[a] < lo || A[a] > hi) return;
        } else {
            // approximate reciprocal (rel. error < 2^-22): the clipped range carries
            // EPSD cells and two lattice steps of slack on each side, against a t error
            // of ~1e-7 t (n_steps < 2^20 on this path: < 0.2 steps)
            float inv;
            asm("rcp.approx.f32 %0, %1;" : "=f"(inv) : "f"(B[a]));
            float ta = (lo - A[a]) * inv, tb = (hi - A[a]) * inv;
            tlo = fmaxf(tlo, fminf(ta, tb));
            thi = fminf(thi, fmaxf(ta, tb));
        }
    }
    if (!(tlo <= thi)) return;
    // Distance-map walk (replaces a coarse DDA): for lattice step j the fp32 cell
    // coordinate of its midpoint is within E of the real one. If that cell lies in
    // the domain and its L-inf distance to the nearest occupied cell is D >= 2,
    // every point within L = D - 1 - 2E - 0.01 cells of it is in an empty cell, so
    // the next floor(L / (bmax * step)) lattice steps are skipped unevaluated
    // (bmax * step = largest per-step move along any axis, in cells).
    const int last = int(P.n_steps) - 1;
    float inv_bms;  // approximate: jumps are cut by the 0.99999 factor below (1e-5 >> 2^-22)
    asm("rcp.approx.f32 %0, %1;" : "=f"(inv_bms) : "f"(fmaxf(bmax * P.step_f, 1e-30f)));
    const float jump_margin = 1.0f + 2.0f * E + 0.01f;
    const int Ri = int(P.res);
    int j = int(floorf((tlo - P.near_f) * P.inv_step_f)) - 2;
    int jend = int(floorf((thi - P.near_f) * P.inv_step_f)) + 2;
    if (j < 0) j = 0;
    if (jend > last) jend = last;
    bool alive = true;
    while (j <= jend) {
        const float m = fmaf(float(j), P.step_f, P.m0_f);
        const float v0 = fmaf(VM_RC(3, B[0]), m, VM_RC(0, Ah[0]));
        const float v1 = fmaf(VM_RC(4, B[1]), m, VM_RC(1, Ah[1]));
        const float v2 = fmaf(VM_RC(5, B[2]), m, VM_RC(2, Ah[2]));
        // |u| stays within a few cells of the domain here (the loop range is the
        // clipped lattice), so the float->int floor is exact and in range
        const int i0 = __float2int_rn(v0), i1 = __float2int_rn(v1), i2 = __float2int_rn(v2);
        const bool inside = unsigned(i0) < unsigned(Ri) && unsigned(i1) < unsigned(Ri) && unsigned(i2) < unsigned(Ri);
        int D = kDistCap;
        uint32_t cell = 0;
        if (inside) {
            cell = uint32_t(i0) + P.res * (uint32_t(i1) + P.res * uint32_t(i2));
            D = __ldg(P.dist + cell);
            if (D >= 2 && j != last) {
                const float Lj = float(D) - jump_margin;
                j += (Lj > 0.0f ? int(Lj * inv_bms * 0.99999f) : 0) + 1;
                continue;
            }
        }
        bool exact = !fast_ok || j == last;
        if (!exact) {
            const float r0 = v0 - float(i0), r1 = v1 - float(i1), r2 = v2 - float(i2);
            exact = fmaxf(fmaxf(fabsf(r0), fabsf(r1)), fabsf(r2)) > half_E;
        }
        if (exact) {
            if (!eval_step<MODE>(P, s, load3(orig, r), load3(dirs, r), uint64_t(j), err, &alive))
                return;
            ++j;
            continue;
        }
        if (!inside || D != 0) {  // outside the domain, or an empty cell
            ++j;
            continue;
        }
        // occupied cell: a candidate, with the reference's exact interval
        const double dj = double(j);  // double(j + 1) == dj + 1.0 exactly (j < 2^20): one I2F
        if (P.sphere_fast && s.filtering) {
            // Filtered SolidSphere test (fields.cpp:45): |p - c|^2 in fp32 from the
            // ray's quadratic, within sph_err; decided cases skip the fp64 midpoint
            // + sqrt.
            const float d2 = fmaf(fmaf(VM_RC(6, Q[0]), m, VM_RC(7, Q[1])), m, VM_RC(8, Q[2]));
            if (d2 > P.sph_r2 + sph_err || d2 < P.sph_r2 - sph_err) {
                if (s.n_cand >= P.max_cand) return;  // candidate cap
                uint32_t ci = s.n_cand++;
                const bool in = d2 < P.sph_r2;
                if (matab(MODE) && (s.at32 ? P.tab_same32 : true)) {
                    // The constant interior density from the table: alpha and the
                    // midpoint 0.5 (t0 + t1) of step j. sigma = 0 outside is never kept
                    // (alpha_thre >= 0); inside, the attribute-dtype sigma equals the
                    // march sigma, so the compositing T is the march's T (acc[0]
                    // follows it for the general path) and alpha is the same value.
                    if (!in) {
                        ++j;
                        continue;
                    }
                    const double a = walk_dyn_smem[2 * j];
                    if (a <= P.thr) {
                        ++j;
                        continue;
                    }
                    if (s.n_kept < s.buf_cap) s.buf[s.n_kept * s.buf_stride] = uint32_t(j);
                    if (mbase(MODE) == BUFFER_FWD) {  // rendering.cpp:50-58, in its operation order
                        const double w = s.T * a;
                        const double mid = walk_dyn_smem[2 * j + 1];  // (w 0.5)(t0 + t1) == w (0.5 (t0 + t1))
                        const double cr = s.at32 ? P.sph_rgb32[0] : P.f.rgb[0];
                        const double cg = s.at32 ? P.sph_rgb32[1] : P.f.rgb[1];
                        const double cb = s.at32 ? P.sph_rgb32[2] : P.f.rgb[2];
                        WACC(1) = WACC(1) + cr * w;
                        WACC(2) = WACC(2) + cg * w;
                        WACC(3) = WACC(3) + cb * w;
                        WACC(4) += w;
                        WACC(5) += w * mid;
                    }
                    s.n_kept++;
                    s.T *= 1.0 - a;
                    if (mbase(MODE) == BUFFER_FWD) WACC(0) = s.T;
                    if (s.T < P.eps) {
                        s.filtering = false;
                        if (!P.full) return;
                    }
                    ++j;
                    continue;
                }
                const double t0 = P.near_ + dj * P.step;
                const double t1 = min_ref(P.near_ + (dj + 1.0) * P.step, P.far_);
                const double sigma = in ? P.f.sigma : 0.0;
                // attribute-dtype roundings precomputed on the host (k_shade's AT(rgb), AT(sigma))
                const D3 rgb = !in ? d3(0.0, 0.0, 0.0)
                                   : s.at32 ? d3(P.sph_rgb32[0], P.sph_rgb32[1], P.sph_rgb32[2])
                                            : d3(P.f.rgb[0], P.f.rgb[1], P.f.rgb[2]);
                const double sg = !in ? 0.0 : s.at32 ? P.sph_sig32 : P.f.sigma;
                // alpha of step j for the constant interior density (table) or computed
                const double apre = matab(MODE) && in ? walk_dyn_smem[2 * j] : -1.0;
                if (!filter_sample<MODE>(P, s, uint64_t(j), ci, t0, t1, sigma, err, rgb, true, sg, apre))
                    return;
                ++j;
                continue;
            }
        }
        const double t0 = P.near_ + dj * P.step;
        const double t1 = min_ref(P.near_ + (dj + 1.0) * P.step, P.far_);
        D3 p = load3(orig, r) + load3(dirs, r) * (0.5 * (t0 + t1));
        if (!on_candidate<MODE>(P, s, uint64_t(j), t0, t1, p, err)) return;
        ++j;
    }
}

#undef VM_RC

__device__ __forceinline__ bool ray_safe(const MarchParams& P, D3 o, D3 d) {
    // Overflowing midpoints can only occur for astronomically large inputs; such
    // rays take the dense walk so every step is checked as the reference does.
    double mag = fmax(fmax(fabs(o.x), fabs(o.y)), fabs(o.z)) +
                 fmax(fmax(fabs(d.x), fabs(d.y)), fabs(d.z)) * fmax(fabs(P.near_), fabs(P.far_));
    return mag < 1e300;
}

template <int MODE, typename RT>
__device__ __forceinline__ void walk(const MarchParams& P, Sink& s, const RT* __restrict__ orig,
                                     const RT* __restrict__ dirs, uint64_t r, DevError* err) {
    bool safe;
    {
        const D3 o = load3(orig, r), d = load3(dirs, r);
        safe = ray_safe(P, o, d);
        if (mext(MODE)) {
            walk_ext<MODE>(P, s, o, d, err);
            return;
        }
        if (P.grows) {
            walk_growth<MODE>(P, s, o, d, err);
            return;
        }
        if (!(P.fast && safe)) {
            if (P.skip && safe)
                walk_skip<MODE>(P, s, o, d, err);
            else
                walk_dense<MODE>(P, s, o, d, err);
            return;
        }
    }
    walk_fast<MODE>(P, s, orig, dirs, r, err);
}

// ---------------------------------------------------------------------------
// Packed march, walk + expand:
//   k_march_walk   persistent warps steal 32-ray chunks from an atomic counter
//                  (no CTA barrier, no cross-CTA waiting: a warp that finishes
//                  early just takes the next chunk); each ray writes its kept
//                  count and the lattice indices of its first kWalkCap kept
//                  samples into a chunk-major scratch [chunk][k][lane] (u32).
//   scan           counts -> offsets (scan.cu)
//   k_march_expand warp per chunk; the chunk's samples are one contiguous output
//                  range, written coalesced: each lane finds the owning ray of its
//                  output slot by a shuffle binary search over the 32 offsets and
//                  re-materialises t0/t1 from the lattice index with the exact
//                  reference expressions.
//   k_march_fixup  re-walks the rare rays with more than kWalkCap kept samples.
// ---------------------------------------------------------------------------
#ifndef VMB_WALK_RSM
#define VMB_WALK_RSM 1
#endif
constexpr int kWalkCap = 32;  // >= the 28 kept samples of a sphere ray at config 2 (step sqrt(3)/1024)
// A/B build switches (make variant DEFS=...): the constant-density alpha table, the
// expansion's constant shading, and the two-pass march for every lattice
#ifndef VMB_ATAB
#define VMB_ATAB 1
#endif
#ifndef VMB_EXPAND_CONST
#define VMB_EXPAND_CONST 1
#endif
#ifndef VMB_MARCH_TWOPASS
#define VMB_MARCH_TWOPASS 0
#endif
#ifndef VMB_WALK_CLAIM
#define VMB_WALK_CLAIM 1
#endif
// chunks per work-stealing ticket (measured at config 5: 1 = 0.756, 2 = 0.757,
// 4 = 0.769 ms/step; an L1 prefetch of the next claimed chunk did not pay either)
constexpr int kClaim = VMB_WALK_CLAIM;

// FAST instantiates only walk_fast (+ its exact fallback and the dense walk for
// unsafe rays), so its register allocation is not the union of every walk.
#ifndef VMB_WALK_MINB
#define VMB_WALK_MINB (1024 / VMB_WALK_THREADS)  // 32 warps per SM: 64 registers
#endif
// Fused render_forward (vmb_march_render_field): for an analytic field the
// compositing of rendering.cpp:47-58 runs over exactly the kept samples, in order,
// with alpha from the shaded sigma. FwdAcc (k_march_fixup) and Sink::composite
// (k_march_walk, inline as samples are kept) repeat k_shade + k_forward's
// expressions (attributes rounded to the attribute dtype first), so the outputs
// are bit-identical to march -> shade -> render_forward. Inline compositing needs
// the shading position to be the march position (time_shift == identity).
template <typename AT, bool VOX>
struct FwdAcc {
    double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0, op = 0.0, dep = 0.0;
    template <typename RT>
    __device__ __forceinline__ void kept(const MarchParams& P, const RT* orig, const RT* dirs,
                                         uint64_t r, double t0, double t1, double time) {
        const D3 x = load3(orig, r) + load3(dirs, r) * (0.5 * (t0 + t1));
        D3 c;
        const double sg = double(AT(field_rgb_sigma_t<VOX>(P.f, time_shift(P.f, x, time), &c)));
        const double alpha = 1.0 - exp(-sg * (t1 - t0));
        const double w = T * alpha;
        cr = cr + double(AT(c.x)) * w;
        cg = cg + double(AT(c.y)) * w;
        cb = cb + double(AT(c.z)) * w;
        op += w;
        dep += w * 0.5 * (t0 + t1);
        T *= 1.0 - alpha;
    }
    __device__ __forceinline__ void store(uint64_t r, AT* color, AT* opacity, AT* depth) const {
        color[3 * r] = AT(cr);
        color[3 * r + 1] = AT(cg);
        color[3 * r + 2] = AT(cb);
        opacity[r] = AT(op);
        depth[r] = AT(dep);
    }
};

template <typename AT>
struct FwdOut {
    AT* color;
    AT* opacity;
    AT* depth;
    double time;
};

// FAST instantiates only walk_fast (+ its exact fallback and the dense walk for
// unsafe rays), so its register allocation is not the union of every walk.
template <typename RT, bool FAST, typename AT, bool FWD, bool VOX, bool ATAB = false, bool ATTR = false>
__global__ void __launch_bounds__(kAccStride, VMB_WALK_MINB) k_march_walk(
    MarchParams P, const RT* __restrict__ orig, const RT* __restrict__ dirs, uint64_t n_rays,
    uint32_t* __restrict__ counts, uint32_t* __restrict__ kept_idx, unsigned int* chunk_counter,
    uint64_t n_chunks, unsigned long long* emitted, DevError* err, FwdOut<AT> fo,
    uint32_t* __restrict__ chunk_tot, void* __restrict__ kept_attr) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    unsigned long long emit_local = 0;
    if (ATAB) {  // alpha per lattice step for the constant interior density (sphere)
        for (uint32_t j = threadIdx.x; j < P.atab_n; j += blockDim.x) {
            const double dj = double(j);
            const double t0 = P.near_ + dj * P.step;
            const double t1 = min_ref(P.near_ + (dj + 1.0) * P.step, P.far_);
            walk_dyn_smem[2 * j] = 1.0 - exp(-P.f.sigma * (t1 - t0));
            walk_dyn_smem[2 * j + 1] = 0.5 * (t0 + t1);
        }
        __syncthreads();
    }
    // chunks are claimed kClaim at a time (one atomic per claim)
    unsigned int chunk = 0, claim_end = 0;
    for (;;) {
        if (chunk == claim_end) {
            if (lane == 0) chunk = atomicAdd(chunk_counter, unsigned(kClaim));
            chunk = __shfl_sync(0xffffffffu, chunk, 0);
            claim_end = chunk + kClaim;
        }
        if (chunk >= n_chunks) break;
        const uint64_t r = uint64_t(chunk) * 32 + lane;
        uint32_t kept = 0;
        if (r < n_rays) {
            Sink s;
            s.ray = r;
            s.buf = kept_idx + uint64_t(chunk) * (kWalkCap * 32) + lane;
            s.buf_stride = 32;
            s.buf_cap = kWalkCap;
            s.at32 = sizeof(AT) == 4;
            if (ATTR)
                s.attr = static_cast<char*>(kept_attr) + (uint64_t(chunk) * (kWalkCap * 32) + lane) * 4 * sizeof(AT);
            if (FWD) {
                WACC(0) = 1.0;
#pragma unroll
                for (int k = 1; k < 6; ++k) WACC(k) = 0.0;
            }
            constexpr int M = (FWD ? BUFFER_FWD : BUFFER) | (VOX ? VOXM : 0) | (ATAB ? ATABM : 0) |
                              (FAST && VMB_WALK_RSM ? RSMM : 0) | (FWD && ATTR ? ATTRM : 0);
            if (FAST) {
                const D3 o = load3(orig, r), d = load3(dirs, r);
                // f32 rays (|o|, |d| < 3.5e38) cannot reach ray_safe's 1e300 bound
                // unless near/far are beyond 1e250 (P.f32_safe, set on the host)
                if ((sizeof(RT) == 4 && P.f32_safe) || ray_safe(P, o, d))
                    walk_fast<M>(P, s, orig, dirs, r, err);
                else
                    walk_dense<M>(P, s, o, d, err);
            } else {
                walk<M>(P, s, orig, dirs, r, err);
            }
            counts[r] = s.n_kept;
            kept = s.n_kept;
            emit_local += s.n_cand;
            if (FWD) {  // every kept sample was composited (rays over kWalkCap too)
                fo.color[3 * r] = AT(WACC(1));
                fo.color[3 * r + 1] = AT(WACC(2));
                fo.color[3 * r + 2] = AT(WACC(3));
                fo.opacity[r] = AT(WACC(4));
                fo.depth[r] = AT(WACC(5));
            }
        }
        // the chunk's sample total: the packing scans these (32x fewer than rays)
        const uint32_t tot = __reduce_add_sync(0xffffffffu, kept);
        if (lane == 0) chunk_tot[chunk] = tot;
        ++chunk;
    }
    if (emitted) {
        for (int o = 16; o > 0; o >>= 1) emit_local += __shfl_xor_sync(0xffffffffu, emit_local, o);
        if (lane == 0 && emit_local) atomicAdd(emitted, emit_local);
    }
}

// Optional fused shading of an analytic field (vmb_march_field_shaded): the
// expand kernel already holds each sample's ray and exact t0/t1, so it writes the
// field's rgb/sigma at the midpoint too — the expressions of shade_samples
// (voxmarch.cpp:235-251) / k_shade, without re-reading the packed samples.
template <typename RT, typename AT, bool VOX = false>
struct ShadeOut {
    const RT* orig;
    const RT* dirs;
    vmb_field f;
    double time;
    AT* rgb;
    AT* sig;
    __device__ __forceinline__ void shade(uint64_t r, uint64_t p, double t0, double t1) const {
        D3 o = d3(double(orig[3 * r]), double(orig[3 * r + 1]), double(orig[3 * r + 2]));
        D3 d = d3(double(dirs[3 * r]), double(dirs[3 * r + 1]), double(dirs[3 * r + 2]));
        shade_ray(o, d, p, t0, t1);
    }
    __device__ __forceinline__ void shade_ray(D3 o, D3 d, uint64_t p, double t0, double t1) const {
        D3 x = o + d * (0.5 * (t0 + t1));
        D3 c;
        double sigma = field_rgb_sigma_t<VOX>(f, time_shift(f, x, time), &c);
        rgb[3 * p] = AT(c.x);
        rgb[3 * p + 1] = AT(c.y);
        rgb[3 * p + 2] = AT(c.z);
        sig[p] = AT(sigma);
    }
};

// Per warp, software-pipelined over its chunks: while chunk c is expanded, the
// used kept-index rows of chunk c+1 (rows x 128 B, contiguous) are already in
// flight into the other shared-memory buffer (cp.async, 16 B per lane), its rays
// are in registers, and the counts/offsets of chunk c+2 are being loaded. Each
// lane holds its own ray; a sample's ray is handed to its lane by shuffles. The
// per-sample work touches registers/smem only, plus the coalesced output writes.
#ifndef VMB_EXPAND_WARPS
#define VMB_EXPAND_WARPS 12  // one CTA per SM; r2 sweep (config 5 step): 12 0.7077 ms, 16 0.7113, 14 0.7104, 10 0.7118, 6 0.7121
#endif
constexpr int kExpandWarps = VMB_EXPAND_WARPS;
#ifndef VMB_EXPAND_UNROLL
#define VMB_EXPAND_UNROLL 4
#endif
constexpr int kExpandUnroll = VMB_EXPAND_UNROLL;  // rounds per iteration of the constant-shading path
// per warp: two kept-index row buffers, the owner map, and the rows' two mbarriers
__host__ __device__ constexpr size_t expand_smem_of(int warps) {
    return size_t(warps) * (kWalkCap * 32 * (2 * sizeof(uint32_t) + sizeof(uint16_t)) + 2 * sizeof(uint64_t));
}
// Warps per expansion CTA: the variants that evaluate the field per sample (rays by
// shuffles, e.g. the Checker) are compute-heavier and run 16 (r2: Checker step
// 1.44 -> 1.37 ms); constant / copied attributes run kExpandWarps (12).
__host__ __device__ constexpr int expand_warps(bool shade, bool cst, bool attr) { return shade && !cst && !attr ? 16 : kExpandWarps; }
constexpr uint32_t kMaxAlphaTable = 1024;  // the fused backward's constant-density alpha table


// (an explicit minBlocksPerSM, even 1, changes the register allocation and costs
// ~25 us per step here: leave it unset unless tuning with -DVMB_EXPAND_MINB)
#ifdef VMB_EXPAND_MINB
#define VMB_EXPAND_BOUNDS __launch_bounds__(32 * expand_warps(SHADE, CONST, ATTR), VMB_EXPAND_MINB)
#else
#define VMB_EXPAND_BOUNDS __launch_bounds__(32 * expand_warps(SHADE, CONST, ATTR))
#endif
// Fused training step (vmb_march_render_backward_field_async): the expansion also
// runs render_backward (rendering.cpp:67-112) on the samples it has just written —
// t0/t1 from the lattice index, rgb/sigma from the shading — so nothing is read
// back. Per chunk (mapped: no ray above kWalkCap kept samples) two sweeps over its
// 32-slot rounds, one sample per lane: the forward sweep carries T (segmented
// product scan of 1 - alpha, the carry into round q kept by lane q), the reverse
// sweep recomputes T, takes the owner ray's upstream gradients by shuffles and
// accumulates the suffix of w v from the ray's end (segmented reverse sum scan),
// then writes every output of the slot. alpha = 1 - exp(-sigma delta) with sigma
// in the attribute dtype, as render_backward recomputes it from the stored sigma
// (for a constant field: a per-CTA table over the lattice). Chunks with a longer
// ray list their rays for k_backward_long after the fixup re-walk.
template <typename AT>
struct BwdOut {
    const AT* dc;
    const AT* dop;
    const AT* ddep;
    AT* g_rgb;
    AT* g_sig;
    uint32_t* list;         // rays of unmapped chunks (backward after the fixup)
    unsigned int* n_list;
    uint32_t atab_n;        // CONST: alpha table entries (lattice steps), 0 = compute
    double sig_at;          // CONST: the field's sigma in the attribute dtype
};

// CONST (shading of a UniformBox / SolidSphere whose kept samples are all inside):
// a kept sample has alpha > alpha_thre >= 0, so the march saw sigma > 0 at the
// sample's midpoint, i.e. the constant interior density — and shading evaluates
// the same field at the same point (time shift = identity), so rgb/sigma are the
// field's constants: no ray, no position, no test.
// ATTR: the walk left each kept sample's rgb/sigma beside its lattice index
// (ATTRM); they are copied instead of evaluating the field again.
template <typename RT, typename AT, bool SHADE, bool VOX, bool CONST = false, bool BWD = false, bool ATTR = false>
__global__ void VMB_EXPAND_BOUNDS k_march_expand(
    double near_, double far_, double step, const uint32_t* __restrict__ counts,
    const uint32_t* __restrict__ chunk_off, uint32_t* __restrict__ offsets,
    const uint32_t* __restrict__ kept_idx, uint64_t n_rays,
    double* __restrict__ ts, double* __restrict__ te, uint32_t* __restrict__ idx, uint64_t cap,
    uint32_t* __restrict__ overflow, unsigned int* n_overflow, ShadeOut<RT, AT, VOX> sh, BwdOut<AT> bo,
    const void* __restrict__ kept_attr) {
    griddep_wait();
    constexpr bool RAYS = SHADE && !CONST && !ATTR;  // the per-sample shading needs the ray
    constexpr int EW = expand_warps(SHADE, CONST, ATTR);
    using AT4 = std::conditional_t<sizeof(AT) == 4, float4, double4>;
    const AT4* attr = static_cast<const AT4*>(kept_attr);
    // dynamic shared memory (expand_smem_of(EW)): per warp, two kept-index row buffers and
    // the owner map of the chunk's output slots (lane | (k << 5), k = rank in the ray)
    extern __shared__ __align__(16) uint32_t expand_smem[];
    uint32_t(*s_idx)[2][kWalkCap * 32] = reinterpret_cast<uint32_t(*)[2][kWalkCap * 32]>(expand_smem);
    uint16_t(*s_map)[kWalkCap * 32] =
        reinterpret_cast<uint16_t(*)[kWalkCap * 32]>(expand_smem + EW * 2 * kWalkCap * 32);
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint64_t n_chunks = (n_rays + 31) / 32;
    const uint64_t wstride = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const uint64_t c0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    AT c_rgb[3] = {AT(0), AT(0), AT(0)}, c_sig = AT(0);
    if (CONST) {
        c_rgb[0] = AT(sh.f.rgb[0]), c_rgb[1] = AT(sh.f.rgb[1]), c_rgb[2] = AT(sh.f.rgb[2]);
        c_sig = AT(sh.f.sigma);
    }
    // the row buffers' mbarriers, then (BWD && CONST) alpha per lattice step
    unsigned long long* rbar = reinterpret_cast<unsigned long long*>(
        expand_smem + EW * (2 * kWalkCap * 32 + kWalkCap * 16)) + 2 * wib;
    double* atab = reinterpret_cast<double*>(expand_smem + EW * (2 * kWalkCap * 32 + kWalkCap * 16 + 4));
    if (BWD && CONST) {
        for (uint32_t j = threadIdx.x; j < bo.atab_n; j += blockDim.x) {
            const double dj = double(j);
            const double t0 = near_ + dj * step;
            const double t1 = min_ref(near_ + (dj + 1.0) * step, far_);
            atab[j] = 1.0 - exp(-bo.sig_at * (t1 - t0));
        }
        __syncthreads();
    }

    // chunk-local state: count/offset of this lane's ray, its ray (RT), and the
    // number of staged rows
    // (off: the chunk's first packed position, chunk_off[c]; a ray's own offset is
    // that plus the exclusive warp scan of the counts, written to offsets[])
    struct Stage {
        uint32_t cnt = 0u, off = 0u;
        RT o[3] = {}, d[3] = {};
    };
    auto load_meta = [&](uint64_t c, Stage& st) {
        const uint64_t r = c * 32 + lane;
        st.cnt = 0u;
        st.off = 0u;
        if (c < n_chunks) st.off = chunk_off[c];
        if (c < n_chunks && r < n_rays) st.cnt = counts[r];
    };
    auto load_rays = [&](uint64_t c, Stage& st) {
        const uint64_t r = c * 32 + lane;
        if (RAYS && c < n_chunks && r < n_rays) {
#pragma unroll
            for (int a = 0; a < 3; ++a) st.o[a] = sh.orig[3 * r + a], st.d[a] = sh.dirs[3 * r + a];
        }
    };
    // the chunk's used kept-index rows (rows x 128 B, contiguous, 16 B aligned): one
    // bulk copy issued by lane 0, completed on the buffer's mbarrier
    if (lane == 0) {
        mbar_init(&rbar[0]);
        mbar_init(&rbar[1]);
        mbar_fence_init();
    }
    __syncwarp();
    uint32_t rphase = 0u;  // bit b: parity of buffer b's next completion
    auto stage_rows = [&](uint64_t c, const Stage& st, int buf) {
        const uint32_t rows = c < n_chunks ? min(__reduce_max_sync(0xffffffffu, st.cnt), uint32_t(kWalkCap)) : 0u;
        if (lane == 0) {
            fence_proxy_async();  // the buffer's earlier reads happen before the copy
            mbar_expect(&rbar[buf], rows * 128u);
            if (rows) bulk_g2s(s_idx[wib][buf], kept_idx + c * (kWalkCap * 32), rows * 128u, &rbar[buf]);
        }
    };
    // one output slot p, owned by lane L (its k-th kept sample)
    auto emit = [&](uint64_t chunk, uint64_t p, int L, uint32_t i, D3 o, D3 d, uint32_t k = 0) {
        const double di = double(i);  // double(i + 1) == di + 1.0 exactly
        const double t0 = near_ + di * step;
        const double t1 = min_ref(near_ + (di + 1.0) * step, far_);
        ts[p] = t0;
        te[p] = t1;
        idx[p] = uint32_t(chunk * 32 + L);
        if (CONST) {
            sh.rgb[3 * p] = c_rgb[0];
            sh.rgb[3 * p + 1] = c_rgb[1];
            sh.rgb[3 * p + 2] = c_rgb[2];
            sh.sig[p] = c_sig;
        } else if (ATTR) {
            const AT4 a = attr[chunk * (kWalkCap * 32) + k * 32 + L];
            sh.rgb[3 * p] = a.x;
            sh.rgb[3 * p + 1] = a.y;
            sh.rgb[3 * p + 2] = a.z;
            sh.sig[p] = a.w;
        } else if (SHADE) {
            sh.shade_ray(o, d, p, t0, t1);
        }
    };

    Stage cur, nxt, nn;
    load_meta(c0, cur);
    load_rays(c0, cur);
    stage_rows(c0, cur, 0);
    load_meta(c0 + wstride, nxt);
    int buf = 0;
    uint16_t* mp = s_map[wib];
    for (uint64_t chunk = c0; chunk < n_chunks; chunk += wstride, buf ^= 1) {
        // pipeline: rows + rays of the next chunk, counts of the one after
        stage_rows(chunk + wstride, nxt, buf ^ 1);
        load_rays(chunk + wstride, nxt);
        load_meta(chunk + 2 * wstride, nn);

        const uint64_t r = chunk * 32 + lane;
        const bool valid = r < n_rays;
        if (!__any_sync(0xffffffffu, cur.cnt != 0u)) {  // no kept sample in the chunk: its offsets only
            if (valid) offsets[r] = cur.off;
            mbar_wait(&rbar[buf], (rphase >> buf) & 1u);  // the chunk's (empty) row stage
            rphase ^= 1u << buf;
            __syncwarp();
            cur = nxt;
            nxt = nn;
            continue;
        }
        const uint32_t cnt = cur.cnt;
        uint32_t incl = cnt;  // inclusive warp scan of the counts
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, dd);
            if (lane >= dd) incl += v;
        }
        const uint32_t off = valid ? cur.off + incl - cnt : 0xffffffffu;
        if (valid) offsets[r] = off;
        const bool big = cnt > uint32_t(kWalkCap);
        if (big) overflow[atomicAdd(n_overflow, 1u)] = uint32_t(r);
        const unsigned vmask = __ballot_sync(0xffffffffu, valid);
        const int last = 31 - __clz(vmask);
        const uint64_t base = __shfl_sync(0xffffffffu, off, 0);
        const uint64_t end = uint64_t(__shfl_sync(0xffffffffu, off, last)) +
                             __shfl_sync(0xffffffffu, cnt, last);
        const RT ox = cur.o[0], oy = cur.o[1], oz = cur.o[2];  // shuffled in the ray's own type
        const RT dx = cur.d[0], dy = cur.d[1], dz = cur.d[2];
        const bool mapped = !__any_sync(0xffffffffu, big);  // then end - base <= kWalkCap * 32
        if (mapped)  // lane-serial: one 16-bit entry per kept sample
            for (uint32_t k = 0; k < cnt; ++k) mp[off - uint32_t(base) + k] = uint16_t(lane | (k << 5));
        mbar_wait(&rbar[buf], (rphase >> buf) & 1u);  // this chunk's rows have landed
        rphase ^= 1u << buf;
        __syncwarp();
        const uint32_t* sk = s_idx[wib][buf];
        if (BWD && !mapped) {  // a ray above kWalkCap: the chunk's rays go to k_backward_long
            const unsigned lm = __ballot_sync(0xffffffffu, valid && cnt > 0u);
            unsigned at = 0;
            if (lane == 0) at = atomicAdd(bo.n_list, unsigned(__popc(lm)));
            at = __shfl_sync(0xffffffffu, at, 0);
            if ((lm >> lane) & 1u) bo.list[at + __popc(lm & ((1u << lane) - 1u))] = uint32_t(r);
        }
        if (BWD && mapped) {
            // upstream gradients of this lane's ray (rendering.cpp:101-102)
            double u_dcx = 0.0, u_dcy = 0.0, u_dcz = 0.0, u_dop = 0.0, u_ddep = 0.0;
            if (valid) {
                u_dcx = double(bo.dc[3 * r]), u_dcy = double(bo.dc[3 * r + 1]), u_dcz = double(bo.dc[3 * r + 2]);
                u_dop = double(bo.dop[r]), u_ddep = double(bo.ddep[r]);
            }
            const uint32_t n_rounds = uint32_t(end - base + 31) / 32;  // <= 32: mapped
            // one slot's sample: owner lane, rank, interval, alpha, rgb (rgb only when `col`)
            auto sample = [&](uint64_t p, bool in, int* L, uint32_t* k, double* t0, double* t1, double* a,
                              double c[3], bool col) {
                *L = 0, *k = 0;
                *t0 = 0.0, *t1 = 0.0, *a = 0.0;
                c[0] = c[1] = c[2] = 0.0;
                if (in) {
                    const uint32_t e = mp[p - base];
                    *L = int(e & 31u);
                    *k = e >> 5;
                }
                D3 o{}, d{};
                if (RAYS) {
                    o = d3(double(__shfl_sync(0xffffffffu, ox, *L)), double(__shfl_sync(0xffffffffu, oy, *L)),
                           double(__shfl_sync(0xffffffffu, oz, *L)));
                    d = d3(double(__shfl_sync(0xffffffffu, dx, *L)), double(__shfl_sync(0xffffffffu, dy, *L)),
                           double(__shfl_sync(0xffffffffu, dz, *L)));
                }
                if (!in) return;
                const uint32_t i = sk[*k * 32 + *L];
                const double di = double(i);
                *t0 = near_ + di * step;
                *t1 = min_ref(near_ + (di + 1.0) * step, far_);
                if (CONST) {
                    *a = i < bo.atab_n ? atab[i] : 1.0 - exp(-bo.sig_at * (*t1 - *t0));
                    if (col) c[0] = double(c_rgb[0]), c[1] = double(c_rgb[1]), c[2] = double(c_rgb[2]);
                } else if (!col) {  // forward sweep: shade (k_shade's expressions), keep rgb/sigma
                    AT cr, cg, cb, sga;
                    if (ATTR) {
                        const AT4 av = attr[chunk * (kWalkCap * 32) + *k * 32 + *L];
                        cr = av.x, cg = av.y, cb = av.z, sga = av.w;
                    } else {
                        const D3 x = o + d * (0.5 * (*t0 + *t1));
                        D3 cc;
                        const double sg = field_rgb_sigma_t<VOX>(sh.f, time_shift(sh.f, x, sh.time), &cc);
                        cr = AT(cc.x), cg = AT(cc.y), cb = AT(cc.z), sga = AT(sg);
                    }
                    if (p < cap) {
                        sh.rgb[3 * p] = cr;
                        sh.rgb[3 * p + 1] = cg;
                        sh.rgb[3 * p + 2] = cb;
                        sh.sig[p] = sga;
                    }
                    *a = 1.0 - exp(-double(sga) * (*t1 - *t0));
                } else if (p < cap) {  // reverse sweep: the attributes just written
                    c[0] = double(sh.rgb[3 * p]), c[1] = double(sh.rgb[3 * p + 1]), c[2] = double(sh.rgb[3 * p + 2]);
                    *a = 1.0 - exp(-double(sh.sig[p]) * (*t1 - *t0));
                }
            };
            double cin = 1.0, carry = 1.0;  // lane q: T carried into round q
            for (uint32_t q = 0; q < n_rounds; ++q) {
                if (uint32_t(lane) == q) cin = carry;
                const uint64_t p = base + 32 * q + lane;
                const bool in = p < end;
                int L;
                uint32_t k;
                double t0, t1, a, c[3];
                sample(p, in, &L, &k, &t0, &t1, &a, c, false);
                seg_excl_prod(in ? 1.0 - a : 1.0, !in || k == 0, carry);
            }
            double carryS = 0.0;  // suffix of w v beyond the current round
            for (uint32_t q = n_rounds; q-- > 0;) {
                double cT = __shfl_sync(0xffffffffu, cin, int(q));
                const uint64_t p = base + 32 * q + lane;
                const bool in = p < end;
                int L;
                uint32_t k;
                double t0, t1, a, c[3];
                sample(p, in, &L, &k, &t0, &t1, &a, c, true);
                const double tr = seg_excl_prod(in ? 1.0 - a : 1.0, !in || k == 0, cT);
                const double dcx = __shfl_sync(0xffffffffu, u_dcx, L), dcy = __shfl_sync(0xffffffffu, u_dcy, L);
                const double dcz = __shfl_sync(0xffffffffu, u_dcz, L), dop = __shfl_sync(0xffffffffu, u_dop, L);
                const double ddep = __shfl_sync(0xffffffffu, u_ddep, L);
                const uint32_t cntL = __shfl_sync(0xffffffffu, cnt, L);
                const double v = (dcx * c[0] + dcy * c[1] + dcz * c[2]) + dop + ddep * (0.5 * (t0 + t1));
                const double wgt = tr * a;
                const double later = seg_excl_sum_rev(in ? wgt * v : 0.0, !in || k + 1 == cntL, carryS);
                if (in && p < cap) {
                    ts[p] = t0;
                    te[p] = t1;
                    idx[p] = uint32_t(chunk * 32 + L);
                    if (CONST) {
                        sh.rgb[3 * p] = c_rgb[0];
                        sh.rgb[3 * p + 1] = c_rgb[1];
                        sh.rgb[3 * p + 2] = c_rgb[2];
                        sh.sig[p] = c_sig;
                    }
                    bo.g_rgb[3 * p] = AT(dcx * wgt);
                    bo.g_rgb[3 * p + 1] = AT(dcy * wgt);
                    bo.g_rgb[3 * p + 2] = AT(dcz * wgt);
                    bo.g_sig[p] = AT((t1 - t0) * (tr * (1.0 - a) * v - later));
                }
            }
        } else if (CONST && mapped) {  // no ray needed: kExpandUnroll independent 32-slot rounds per iteration
            for (uint64_t p0 = base; p0 < end; p0 += 32 * kExpandUnroll) {
                uint32_t e[kExpandUnroll], ii[kExpandUnroll];
#pragma unroll
                for (int q = 0; q < kExpandUnroll; ++q) {
                    const uint64_t pq = p0 + 32 * q + lane;
                    e[q] = pq < end && pq < cap ? mp[pq - base] | 0x80000000u : 0u;
                }
#pragma unroll
                for (int q = 0; q < kExpandUnroll; ++q)
                    ii[q] = e[q] ? sk[((e[q] >> 5) & 31u) * 32 + (e[q] & 31u)] : 0u;
#pragma unroll
                for (int q = 0; q < kExpandUnroll; ++q)
                    if (e[q]) emit(chunk, p0 + 32 * q + lane, int(e[q] & 31u), ii[q], D3{}, D3{});
            }
        } else
        for (uint64_t p0 = base; p0 < end; p0 += 32) {
            const uint64_t p = p0 + lane;
            const bool in = p < end && p < cap;
            int L = 0;
            uint32_t k = 0;
            if (mapped) {
                if (in) {
                    const uint32_t e = mp[p - base];
                    L = int(e & 31u);
                    k = e >> 5;
                }
            } else {
                // owner = largest lane L with off_L <= p (zero-count lanes share the
                // next lane's offset, so the largest such lane owns the slot)
#pragma unroll
                for (int stride = 16; stride > 0; stride >>= 1) {
                    int c = L + stride;
                    uint32_t v = __shfl_sync(0xffffffffu, off, c & 31);
                    if (c < 32 && uint64_t(v) <= p) L = c;
                }
                k = uint32_t(p - __shfl_sync(0xffffffffu, off, L));
            }
            D3 o{}, d{};
            if (RAYS) {
                o = d3(double(__shfl_sync(0xffffffffu, ox, L)), double(__shfl_sync(0xffffffffu, oy, L)),
                       double(__shfl_sync(0xffffffffu, oz, L)));
                d = d3(double(__shfl_sync(0xffffffffu, dx, L)), double(__shfl_sync(0xffffffffu, dy, L)),
                       double(__shfl_sync(0xffffffffu, dz, L)));
            }
            if (in && k < uint32_t(kWalkCap)) emit(chunk, p, L, sk[k * 32 + L], o, d, k);
        }
        __syncwarp();  // buffer `buf` and the map are refilled from the next chunk on
        cur = nxt;
        nxt = nn;
    }
    // the last prefetch (a chunk past the end: rows = 0) completes at once
    mbar_wait(&rbar[buf], (rphase >> buf) & 1u);
}

// Re-walks the (rare) rays whose kept samples overflowed the shared buffer.
template <typename RT, typename AT, bool SHADE, bool FWD, bool VOX>
__global__ void k_march_fixup(MarchParams P, const RT* __restrict__ orig, const RT* __restrict__ dirs,
                              const uint32_t* __restrict__ offsets, double* __restrict__ ts,
                              double* __restrict__ te, uint32_t* __restrict__ idx, uint64_t cap,
                              const uint32_t* __restrict__ overflow, const unsigned int* n_overflow,
                              DevError* err, ShadeOut<RT, AT, VOX> sh, FwdOut<AT> fo) {
    griddep_wait();
    const unsigned int n = *n_overflow;
    for (unsigned int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        uint64_t r = overflow[k];
        Sink s;
        s.ray = r;
        s.ts = ts;
        s.te = te;
        s.idx = idx;
        s.base = offsets[r];
        s.cap = cap;
        walk<FILL | (VOX ? VOXM : 0)>(P, s, orig, dirs, r, err);
        if (SHADE)
            for (uint64_t q = s.base; q < s.base + s.n_kept && q < cap; ++q) sh.shade(r, q, ts[q], te[q]);
        if (FWD) {  // walk_fast's t0/t1 of this ray, recomputed by the FILL walk
            FwdAcc<AT, VOX> acc;
            for (uint64_t q = s.base; q < s.base + s.n_kept && q < cap; ++q)
                acc.kept(P, orig, dirs, r, ts[q], te[q], fo.time);
            acc.store(r, fo.color, fo.opacity, fo.depth);
        }
    }
}

// two-pass walk kernel (count / fill): capped at 80 registers (6 CTAs/SM); the
// uncapped build took 120 (count) / 96 (fill) registers. Config 3 stand-in step
// 10.27 -> 9.86 ms (8 CTAs / 64 registers: 10.10 ms; later A/B at 9.30 ms: 5 CTAs
// 9.71, 7 CTAs 9.40).
#ifndef VMB_MARCH_MINB
#define VMB_MARCH_MINB 8  // 64 registers; config 3 (cascade, two-pass walk): 8.97 ms vs 9.04 (6), 9.58 (4)
#endif
#define VMB_MARCH_LB __launch_bounds__(128, VMB_MARCH_MINB)
template <typename RT, int MODE>
__global__ void VMB_MARCH_LB k_march(MarchParams P, const RT* __restrict__ orig,
                                               const RT* __restrict__ dirs, uint64_t n_rays,
                                               uint32_t* __restrict__ counts,
                                               const uint32_t* __restrict__ offsets,
                                               double* __restrict__ ts, double* __restrict__ te,
                                               uint32_t* __restrict__ idx, uint64_t cap,
                                               unsigned long long* emitted, DevError* err, uint32_t slab_cap = 0) {
    // SLABM (FILL): one pass instead of count + fill for long-ray walks — each ray
    // writes its first slab_cap kept intervals to its own slab [r slab_cap, (r + 1)
    // slab_cap) of ts/te/idx and its kept count; k_slab_gather packs them after the
    // scan. FILL with slab_cap > 0: the packed fill of the rays above slab_cap only.
    constexpr bool SLAB = mslab(MODE);
    griddep_wait();
    unsigned long long emit_local = 0;
    __shared__ double stg[mbase(MODE) == FILL ? 8 * kStgStride : 1];
    const bool vec = ((reinterpret_cast<uintptr_t>(ts) | reinterpret_cast<uintptr_t>(te) |
                       reinterpret_cast<uintptr_t>(idx)) & 15) == 0;
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rays;
         r += uint64_t(gridDim.x) * blockDim.x) {
        if (mbase(MODE) == FILL && !SLAB && slab_cap && counts[r] <= slab_cap) continue;
        Sink s;
        s.ray = r;
        if (mbase(MODE) == FILL) {
            s.ts = ts;
            s.te = te;
            s.idx = idx;
            s.base = SLAB ? r * slab_cap : offsets[r];
            s.cap = SLAB ? (r + 1) * slab_cap : cap;
            s.stg = stg + threadIdx.x;
            s.vec = vec;
        }
        walk<MODE & ~SLABM>(P, s, orig, dirs, r, err);
        if (mbase(MODE) == FILL) s.flush_tail();
        if (mbase(MODE) == COUNT || SLAB) counts[r] = s.n_kept;
        emit_local += s.n_cand;
    }
    if ((mbase(MODE) == COUNT || SLAB) && emitted) {
        for (int off = 16; off > 0; off >>= 1) emit_local += __shfl_xor_sync(0xffffffffu, emit_local, off);
        if ((threadIdx.x & 31) == 0 && emit_local) atomicAdd(emitted, emit_local);
    }
}

// The slab pass's packing: warp per ray, its min(count, slab_cap) intervals copied
// coalesced from the slab to the packed arrays at the ray's offset, with its index.
__global__ void k_slab_gather(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ offsets,
                              uint64_t n_rays, uint32_t slab_cap, const double* __restrict__ sts,
                              const double* __restrict__ ste, double* __restrict__ ts, double* __restrict__ te,
                              uint32_t* __restrict__ idx, uint64_t cap) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    for (uint64_t r = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n_rays;
         r += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint32_t n = min(__ldg(counts + r), slab_cap);
        const uint64_t o = __ldg(offsets + r), src = r * slab_cap;
        for (uint32_t k = uint32_t(lane); k < n; k += 32)
            if (o + k < cap) {
                ts[o + k] = __ldg(sts + src + k);
                te[o + k] = __ldg(ste + src + k);
                idx[o + k] = uint32_t(r);
            }
    }
}

// Alpha floor + T cut over host-evaluated candidate sigmas (ray_marching.cpp:118-137).
template <int MODE>
__global__ void k_filter(const uint32_t* __restrict__ c_off, const uint32_t* __restrict__ c_cnt,
                         uint64_t n_rays, const double* __restrict__ c_ts,
                         const double* __restrict__ c_te, const double* __restrict__ sig,
                         double eps, double thr, uint32_t* __restrict__ counts,
                         const uint32_t* __restrict__ offsets, double* __restrict__ ts,
                         double* __restrict__ te, uint32_t* __restrict__ idx, uint64_t cap,
                         DevError* err) {
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rays;
         r += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t b = c_off[r], n = c_cnt[r];
        uint64_t out = mbase(MODE) == FILL ? offsets[r] : 0;
        uint32_t kept = 0;
        double T = 1.0;
        for (uint64_t k = 0; k < n; ++k) {
            double sigma = sig[b + k];
            if (!isfinite(sigma) || sigma < 0.0) {
                atomicMin(&err->key, march_err_key(r, k, !isfinite(sigma) ? ERR_NONFINITE_SIGMA
                                                                          : ERR_NEGATIVE_SIGMA));
                break;
            }
            double t0 = c_ts[b + k], t1 = c_te[b + k];
            double alpha = 1.0 - exp(-sigma * (t1 - t0));
            if (alpha <= thr) continue;
            if (mbase(MODE) == FILL && out + kept < cap) {
                ts[out + kept] = t0;
                te[out + kept] = t1;
                idx[out + kept] = uint32_t(r);
            }
            ++kept;
            T *= 1.0 - alpha;
            if (T < eps) break;
        }
        if (mbase(MODE) == COUNT) counts[r] = kept;
    }
}

// march_uniform: every ray has the same lattice of n_eff steps.
__global__ void k_uniform(uint64_t n_rays, uint64_t n_eff, double near_, double far_, double step,
                          uint32_t* __restrict__ offsets, uint32_t* __restrict__ counts,
                          double* __restrict__ ts, double* __restrict__ te,
                          uint32_t* __restrict__ idx) {
    const uint64_t total = n_rays * n_eff;
    for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < n_rays;
         r += uint64_t(gridDim.x) * blockDim.x) {
        offsets[r] = uint32_t(r * n_eff);
        counts[r] = uint32_t(n_eff);
    }
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < total;
         s += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t r = s / n_eff, i = s - r * n_eff;
        ts[s] = near_ + double(i) * step;
        te[s] = min_ref(near_ + double(i + 1) * step, far_);
        idx[s] = uint32_t(r);
    }
}

int validate_config(const vmb_march_config* c) {  // ray_marching.cpp:12-22
    if (!(c->step_size > 0.0)) return fail(VMB_INVALID_ARGUMENT, "marching: step_size must be > 0");
    if (!(c->early_stop_eps >= 0.0 && c->early_stop_eps < 1.0))
        return fail(VMB_INVALID_ARGUMENT, "marching: early_stop_eps must be in [0,1)");
    if (!(c->alpha_thre >= 0.0 && c->alpha_thre < 1.0))
        return fail(VMB_INVALID_ARGUMENT, "marching: alpha_thre must be in [0,1)");
    if (c->max_samples_per_ray < 1)
        return fail(VMB_INVALID_ARGUMENT, "marching: max_samples_per_ray must be >= 1");
    if (!(c->unbounded_step_growth >= 1.0))
        return fail(VMB_INVALID_ARGUMENT, "marching: unbounded_step_growth must be >= 1");
    return VMB_OK;
}

// Effective lattice length: the first i with !(t1 > t0) ends every ray's walk
// (ray_marching.cpp:81), and it does not depend on the ray. Host arithmetic is
// plain IEEE double (compiled with -ffp-contract=off), identical to the device's.
uint64_t effective_steps(double near_, double far_, double step, uint64_t n, bool* exact) {
    *exact = true;
    if (n > (1ull << 26)) {  // too long to pre-check; the caller falls back to dense walks
        *exact = false;
        return n;
    }
    for (uint64_t i = 0; i < n; ++i) {
        double t0 = near_ + double(i) * step;
        double t1 = min_ref(near_ + double(i + 1) * step, far_);
        if (!(t1 > t0)) return i;
    }
    return n;
}

int march_params(const vmb_grid* g, const vmb_rays* rays, const vmb_march_config* cfg,
                 MarchParams* P) {
    int rc = validate_config(cfg);
    if (rc) return rc;
    if (!(rays->near_plane >= 0.0) || !(rays->far_plane > rays->near_plane))
        return fail(VMB_INVALID_ARGUMENT, "ray batch: requires far > near >= 0");
    *P = MarchParams{};
    P->k = g->k;
    P->res = g->res;
    P->bits = g->bits;
    P->coarse = g->coarse;
    P->grid = g;
    P->dist = g->dist;
    P->bbox = g->bbox;
    P->block = g->block;
    P->res_c = g->res_c;
    P->scale[0] = double(g->res) / g->k.size.x;
    P->scale[1] = double(g->res) / g->k.size.y;
    P->scale[2] = double(g->res) / g->k.size.z;
    P->near_ = rays->near_plane;
    P->far_ = rays->far_plane;
    P->step = cfg->step_size;
    P->grows = g->con.kind == VMB_CONTRACT_SPHERE && cfg->unbounded_step_growth > 1.0;
    P->growth = cfg->unbounded_step_growth;
    P->ball_c = g->k.center;
    P->ball_r = g->k.radius;
    {
        const double r = P->ball_r;
        P->ball_filter = r > 1e-100 && r < 1e100;
        P->ball_r2_lo = P->ball_filter ? r * r * (1.0 - 0x1p-40) : 0.0;
        P->ball_r2_hi = P->ball_filter ? r * r * (1.0 + 0x1p-40) : 0.0;
    }
    P->eps = cfg->early_stop_eps;
    P->thr = cfg->alpha_thre;
    P->max_cand = cfg->max_samples_per_ray;
    bool exact = true;
    uint64_t n = uniform_step_count(P->near_, P->far_, P->step);
    P->n_steps = effective_steps(P->near_, P->far_, P->step, n, &exact);
    P->skip = g->con.kind == VMB_CONTRACT_AABB && exact && !P->grows;
    // fp32 fast walk: lattice indices and step-range conversions stay well inside
    // fp32 resolution for lattices up to 2^20 steps.
    P->fast = P->skip && P->n_steps < (1ull << 20) && P->n_steps > 0 && g->res <= 1024;
    P->f32_safe = fmax(fabs(P->near_), fabs(P->far_)) < 1e250;
    P->step_f = float(P->step);
    P->m0_f = float(P->near_ + 0.5 * P->step);
    P->inv_step_f = float(1.0 / P->step);
    P->near_f = float(P->near_);
    P->far_f = float(P->far_);
    P->Mf = float(fmax(fabs(P->near_), fabs(P->far_)));
    return VMB_OK;
}

// The slab pass of a two-pass walk (k_march slab_mode): per-ray capacity and buffers
struct Slab {
    uint32_t cap = 0;  // 0: count + fill
    int mode = 0;      // 1: the slab pass (SLABM), 2: the fill of the rays above cap
    double* ts = nullptr;
    double* te = nullptr;
    uint32_t* idx = nullptr;
};

template <int MODE>
void launch_march(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, uint32_t* counts,
                  const uint32_t* offsets, vmb_samples* out, unsigned long long* emitted, Slab sl = Slab{});

template <int MODE>
void launch_march_rt(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, uint32_t* counts,
                     const uint32_t* offsets, vmb_samples* out, unsigned long long* emitted, Slab sl) {
    int blocks = grid_blocks(ctx, rays->n_rays, 128, 16);
    double* ts = sl.mode == 1 ? sl.ts : out ? out->d_t_starts : nullptr;
    double* te = sl.mode == 1 ? sl.te : out ? out->d_t_ends : nullptr;
    uint32_t* ix = sl.mode == 1 ? sl.idx : out ? out->d_ray_indices : nullptr;
    const uint64_t cap = out ? out->capacity : 0;
    if (rays->dtype == VMB_F32)
        launch_pdl(k_march<float, MODE>, dim3(blocks), dim3(128), 0, ctx->stream, P,
                   static_cast<const float*>(rays->d_origins), static_cast<const float*>(rays->d_directions),
                   rays->n_rays, counts, offsets, ts, te, ix, cap, emitted, ctx->d_err, sl.cap);
    else
        launch_pdl(k_march<double, MODE>, dim3(blocks), dim3(128), 0, ctx->stream, P,
                   static_cast<const double*>(rays->d_origins), static_cast<const double*>(rays->d_directions),
                   rays->n_rays, counts, offsets, ts, te, ix, cap, emitted, ctx->d_err, sl.cap);
}

// Long-ray walks (accumulated t: cascades, cone stepping, growth) pack in one walk:
// the slab pass, the scan, k_slab_gather, and a fill of the rays above the slab
// capacity only, instead of a count walk and a fill walk. Up to 256 intervals per
// ray and 6 GiB of slab; otherwise (or for short-ray walks) count + fill.
Slab make_slab(vmb_ctx* ctx, const MarchParams& P, uint64_t n_rays) {
#ifndef VMB_SLAB
#define VMB_SLAB 1
#endif
    Slab sl;
    if (!VMB_SLAB || !(P.accum || P.grows) || n_rays == 0) return sl;
    const uint64_t budget = 6ull << 30;  // 256 slots for up to 1.26M rays
    uint64_t cap = budget / (n_rays * (2 * sizeof(double) + 4));  // t0, t1, index per slot
    cap = cap > 256 ? 256 : cap & ~uint64_t(3);
    if (cap < 64) return sl;
    auto* b = static_cast<double*>(scratch(ctx, SCRATCH_SLAB, n_rays * cap * (2 * sizeof(double) + 4)));
    if (!b) {
        cudaGetLastError();  // fall back to count + fill
        return sl;
    }
    sl.cap = uint32_t(cap);
    sl.ts = b;
    sl.te = b + n_rays * cap;
    sl.idx = reinterpret_cast<uint32_t*>(b + 2 * n_rays * cap);
    return sl;
}

void slab_pack(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, vmb_samples* out, Slab sl) {
    const int blocks = grid_blocks(ctx, rays->n_rays * 32, 256, 8);
    launch_pdl(k_slab_gather, dim3(blocks), dim3(256), 0, ctx->stream, out->d_counts, out->d_offsets, rays->n_rays,
               sl.cap, sl.ts, sl.te, out->d_t_starts, out->d_t_ends, out->d_ray_indices, out->capacity);
    sl.mode = 2;
    launch_march<FILL>(ctx, P, rays, out->d_counts, out->d_offsets, out, nullptr, sl);
}

// walk_skip reads the grid's coarse bits: the paths that may take it build them first
int ensure_skip_structures(vmb_ctx* ctx, const MarchParams& P) {
    return P.skip && !P.fast ? grid_ensure_coarse(ctx, P.grid) : VMB_OK;
}

template <int MODE>
void launch_march(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, uint32_t* counts,
                  const uint32_t* offsets, vmb_samples* out, unsigned long long* emitted, Slab sl) {
    if (ensure_skip_structures(ctx, P)) return;
    if (MODE == FILL && sl.mode == 1) {  // the slab pass: long-ray (accumulated-t / growth) walks only
        if (P.accum && P.f.kind == VMB_FIELD_VOXEL)
            launch_march_rt<FILL | SLABM | VOXM | EXTM>(ctx, P, rays, counts, offsets, out, emitted, sl);
        else if (P.accum)
            launch_march_rt<FILL | SLABM | EXTM>(ctx, P, rays, counts, offsets, out, emitted, sl);
        else if (P.f.kind == VMB_FIELD_VOXEL)
            launch_march_rt<FILL | SLABM | VOXM>(ctx, P, rays, counts, offsets, out, emitted, sl);
        else
            launch_march_rt<FILL | SLABM>(ctx, P, rays, counts, offsets, out, emitted, sl);
        return;
    }
    if (P.accum && P.f.kind == VMB_FIELD_VOXEL)
        launch_march_rt<MODE | VOXM | EXTM>(ctx, P, rays, counts, offsets, out, emitted, sl);
    else if (P.accum)
        launch_march_rt<MODE | EXTM>(ctx, P, rays, counts, offsets, out, emitted, sl);
    else if (P.f.kind == VMB_FIELD_VOXEL)
        launch_march_rt<MODE | VOXM>(ctx, P, rays, counts, offsets, out, emitted, sl);
    else
        launch_march_rt<MODE>(ctx, P, rays, counts, offsets, out, emitted, sl);
}

std::string march_error_text(const DevError& e) {
    uint64_t ray = e.key >> 32, low = e.key & 0xffffffffull;
    if (low == 0) return "non-finite coordinate";
    uint64_t sample = (low >> 2) - 1;
    int kind = int(low & 3);
    return std::string(kind == ERR_NONFINITE_SIGMA ? "marching: non-finite density at ray "
                                                   : "marching: negative density at ray ") +
           std::to_string(ray) + " sample " + std::to_string(sample);
}

int report_march_error(vmb_ctx* ctx) {
    DevError err;
    int rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key == ~0ull) return VMB_OK;
    uint64_t low = err.key & 0xffffffffull;
    return fail(low == 0 ? VMB_INVALID_ARGUMENT : VMB_RUNTIME, march_error_text(err));
}

// Filtered fp32 density decisions are used for a well-scaled SolidSphere field.
void set_sphere_fast(MarchParams* P) {
    const vmb_field& f = P->f;
    double cmax = fmax(fmax(fabs(f.center[0]), fabs(f.center[1])), fabs(f.center[2]));
    P->sphere_fast = P->fast && f.kind == VMB_FIELD_SOLID_SPHERE && f.radius > 0.0 &&
                     f.radius < 1e6 && cmax < 1e6 && std::isfinite(f.sigma) && f.sigma >= 0.0;
    for (int a = 0; a < 3; ++a) P->sph_c[a] = float(f.center[a]);
    P->sph_r = float(f.radius);
    P->sph_r2 = P->sph_r * P->sph_r;
    P->sph_cmax = float(cmax);
    P->sph_sig32 = double(float(f.sigma));
    for (int a = 0; a < 3; ++a) P->sph_rgb32[a] = double(float(f.rgb[a]));
    // inside the sphere sigma is one constant, so alpha depends only on the lattice
    // step: k_march_walk tabulates it per CTA (built with -DVMB_ATAB=0: off)
    P->atab_n = P->sphere_fast && VMB_ATAB && P->n_steps <= 1024 ? uint32_t(P->n_steps) : 0u;
    P->tab_same32 = double(float(f.sigma)) == f.sigma;
}


// vmb_march_ext -> MarchParams: stacked levels and the cone rule (vmb_march_cascade).
int apply_ext(const vmb_grid* g, const vmb_march_ext* x, const vmb_march_config* cfg, MarchParams* P) {
    if (!x) return VMB_OK;
    if (x->n_levels > uint32_t(kMaxLevels - 1))
        return fail(VMB_INVALID_ARGUMENT, "cascade: at most 7 levels above level 0");
    if (x->n_levels && !x->levels) return fail(VMB_INVALID_ARGUMENT, "cascade: levels required");
    if (x->cone) {
        if (!(x->cone_angle >= 0.0) || !std::isfinite(x->cone_angle))
            return fail(VMB_INVALID_ARGUMENT, "cascade: cone_angle must be finite and >= 0");
        if (!(x->max_step >= cfg->step_size))
            return fail(VMB_INVALID_ARGUMENT, "cascade: max_step must be >= step_size");
        if (P->grows)
            return fail(VMB_INVALID_ARGUMENT, "cascade: cone stepping and unbounded_step_growth > 1 are exclusive");
    }
    const vmb_grid* prev = g;
    for (uint32_t l = 0; l < x->n_levels; ++l) {
        const vmb_grid* L = x->levels[l];
        if (!L) return fail(VMB_INVALID_ARGUMENT, "cascade: levels required");
        if (prev->con.kind != VMB_CONTRACT_AABB || L->con.kind != VMB_CONTRACT_AABB)
            return fail(VMB_INVALID_ARGUMENT, "cascade: stacked levels must be AABB grids");
        // strictly nested with a margin far above the contraction's rounding
        for (int a = 0; a < 3; ++a) {
            const double m = 1e-9 * (1.0 + fmax(fmax(fabs(L->con.box_min[a]), fabs(L->con.box_max[a])),
                                                fmax(fabs(prev->con.box_min[a]), fabs(prev->con.box_max[a]))));
            if (!(L->con.box_min[a] < prev->con.box_min[a] - m && L->con.box_max[a] > prev->con.box_max[a] + m))
                return fail(VMB_INVALID_ARGUMENT, "cascade: each level must strictly contain the level below");
        }
        P->lv_k[l] = L->k;
        P->lv_res[l] = L->res;
        P->lv_bits[l] = L->bits;
        P->lv_dist[l] = L->dist;
        prev = L;
    }
    // walk_ext's empty-space skipping: every level an AABB grid, no step growth
    P->ext_skip = !P->grows && g->con.kind == VMB_CONTRACT_AABB;
    for (uint32_t l = 0; P->ext_skip && l <= x->n_levels; ++l) {
        const vmb_grid* L = l == 0 ? g : x->levels[l - 1];
        auto& X = P->xs[l];
        for (int a = 0; a < 3; ++a) {
            const double sz = L->con.box_max[a] - L->con.box_min[a];
            if (!(sz > 0.0) || !std::isfinite(sz)) P->ext_skip = false;
            X.lo[a] = L->con.box_min[a];
            X.scale[a] = double(L->res) / sz;
            X.in_lo[a] = 1.0f, X.in_hi[a] = 0.0f;  // level 0: no level below (gap unused)
            if (l > 0) {
                const vmb_grid* B = l == 1 ? g : x->levels[l - 2];
                X.in_lo[a] = float((B->con.box_min[a] - L->con.box_min[a]) * double(L->res) / sz);
                X.in_hi[a] = float((B->con.box_max[a] - L->con.box_min[a]) * double(L->res) / sz);
            }
        }
    }
    P->n_lv = x->n_levels;
    P->cone = x->cone != 0;
    P->cone_angle = x->cone_angle;
    P->max_step = x->max_step;
    P->accum = P->n_lv > 0 || P->cone || P->grows;
    P->exit_box = P->accum && prev->con.kind == VMB_CONTRACT_AABB;
    if (P->accum) P->skip = P->fast = false;
    return VMB_OK;
}

// Points -> occupancy under the cascade rule (the finest level containing each).
__global__ void k_cascade_query(MarchParams P, const double* __restrict__ pts, uint64_t n,
                                uint8_t* __restrict__ out, DevError* err) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        D3 p = d3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        if (!finite3(p)) {
            atomicMin(&err->key, (unsigned long long)i);
            out[i] = 0;
            continue;
        }
        out[i] = uint8_t(cascade_query(P, p, d3(0.0, 0.0, 0.0)) > 0);
    }
}

// A build with -DVMB_MARCH_TWOPASS=1 forces the count -> scan -> fill pipeline (A/B).
bool use_fused(const MarchParams& P) { return !P.grows && !P.accum && !VMB_MARCH_TWOPASS; }

// Optional analytic-field shading fused into the packing (vmb_march_field_shaded).
struct ShadeReq {
    bool on = false;
    vmb_field f{};
    double time = 0.0;
    void* rgb = nullptr;
    void* sig = nullptr;
    int dtype = VMB_F32;
    // fused render_forward (requires on): per-ray outputs in dtype
    bool fwd = false;
    void* color = nullptr;
    void* opacity = nullptr;
    void* depth = nullptr;
    // fused render_backward (requires fwd): upstream gradients in, gradients out
    bool bwd = false;
    const void* dc = nullptr;
    const void* dop = nullptr;
    const void* ddep = nullptr;
    void* g_rgb = nullptr;
    void* g_sig = nullptr;
};

template <typename AT>
FwdOut<AT> fwd_out(const ShadeReq& sr) {
    return FwdOut<AT>{static_cast<AT*>(sr.color), static_cast<AT*>(sr.opacity),
                      static_cast<AT*>(sr.depth), sr.time};
}

// Resident CTAs per SM of one expansion kernel (persistent grid), after opting it
// in to its dynamic shared memory — once per kernel (the kernel is the
// template argument: instantiations share one function type).

template <auto K, size_t SMEM, int W>
int expand_per_sm() {
    static const int n = [] {
        cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM));
        int m = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, K, 32 * W, SMEM);
        return m < 1 ? 2 : m;
    }();
    return n;
}

// Constant shading (see k_march_expand): every kept sample is inside a constant
// analytic field; needs the alpha floor, a positive density and an identity time shift.
bool const_shading(const MarchParams& P, const ShadeReq& sr) {
    const vmb_field& f = sr.f;
    bool ident = std::isfinite(sr.time) && (sr.time == 0.0 || (f.velocity[0] == 0.0 && f.velocity[1] == 0.0 &&
                                                                f.velocity[2] == 0.0));
    for (int a = 0; a < 3; ++a) ident = ident && std::isfinite(f.velocity[a]);
    return sr.on && f.kind != VMB_FIELD_VOXEL && P.filter && P.thr >= 0.0 && ident && std::isfinite(f.sigma) &&
           f.sigma > 0.0 && (f.kind == VMB_FIELD_SOLID_SPHERE || f.kind == VMB_FIELD_UNIFORM_BOX) &&
           VMB_EXPAND_CONST;
}

template <typename RT, typename AT, bool SHADE, bool FWD, bool VOX>
void launch_expand_fixup(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, vmb_samples* out,
                         const uint32_t* kept_idx, uint32_t* overflow, unsigned int* n_overflow,
                         uint64_t n_chunks, const ShadeReq& sr, const uint32_t* chunk_off, uint32_t* bwd_list,
                         const void* kept_attr) {
    ShadeOut<RT, AT, VOX> sh{static_cast<const RT*>(rays->d_origins), static_cast<const RT*>(rays->d_directions),
                        sr.f, sr.time, static_cast<AT*>(sr.rgb), static_cast<AT*>(sr.sig)};
    BwdOut<AT> bo{};
    if (sr.bwd) {
        bo = BwdOut<AT>{static_cast<const AT*>(sr.dc), static_cast<const AT*>(sr.dop), static_cast<const AT*>(sr.ddep),
                        static_cast<AT*>(sr.g_rgb), static_cast<AT*>(sr.g_sig), bwd_list + 4,
                        reinterpret_cast<unsigned int*>(bwd_list), 0u, double(AT(sr.f.sigma))};
        bo.atab_n = P.n_steps <= kMaxAlphaTable ? uint32_t(P.n_steps) : 0u;
    }
    auto launch = [&](auto kernel, int per_sm, size_t smem, int w) {
        launch_pdl(kernel, dim3(grid_blocks(ctx, n_chunks * 32, 32 * w, per_sm)), dim3(32 * w), smem, ctx->stream,
                   P.near_, P.far_, P.step, out->d_counts, chunk_off, out->d_offsets, kept_idx, rays->n_rays,
                   out->d_t_starts, out->d_t_ends, out->d_ray_indices, out->capacity, overflow, n_overflow, sh, bo,
                   kept_attr);
    };
    // one expansion variant: its warps per CTA and dynamic shared memory (+ the
    // constant-density alpha table for the fused backward)
    auto go = [&](auto kernel, auto CST, auto BWDC, auto ATTRC) {
        constexpr bool C = decltype(CST)::value, B = decltype(BWDC)::value, A = decltype(ATTRC)::value;
        constexpr int W = expand_warps(SHADE, C, A);
        constexpr size_t SM = expand_smem_of(W) + (B && C ? kMaxAlphaTable * sizeof(double) : 0);
        launch(kernel, expand_per_sm<k_march_expand<RT, AT, SHADE, VOX, C, B, A>, SM, W>(), SM, W);
    };
    const bool cst = SHADE && !VOX && const_shading(P, sr);
    bool plain = true;
    if constexpr (FWD && SHADE) {
        if (sr.bwd) {
            plain = false;
            zero_words_async(ctx, bwd_list, 1);
            if (cst)
                go(k_march_expand<RT, AT, SHADE, VOX, true, true>, std::true_type{}, std::true_type{},
                   std::false_type{});
            else if (kept_attr)
                go(k_march_expand<RT, AT, SHADE, VOX, false, true, true>, std::false_type{}, std::true_type{},
                   std::true_type{});
            else
                go(k_march_expand<RT, AT, SHADE, VOX, false, true>, std::false_type{}, std::true_type{},
                   std::false_type{});
        } else if (kept_attr) {
            plain = false;
            go(k_march_expand<RT, AT, SHADE, VOX, false, false, true>, std::false_type{}, std::false_type{},
               std::true_type{});
        }
    }
    if (plain && cst)
        go(k_march_expand<RT, AT, SHADE, VOX, true>, std::true_type{}, std::false_type{}, std::false_type{});
    else if (plain)
        go(k_march_expand<RT, AT, SHADE, VOX, false>, std::false_type{}, std::false_type{}, std::false_type{});
    launch_pdl(k_march_fixup<RT, AT, SHADE, FWD, VOX>, dim3(ctx->num_sms * 2), dim3(128), 0, ctx->stream, P, sh.orig,
               sh.dirs, out->d_offsets, out->d_t_starts, out->d_t_ends, out->d_ray_indices, out->capacity, overflow,
               n_overflow, ctx->d_err, sh, fwd_out<AT>(sr));
    if (sr.bwd) {  // the rays of chunks with a ray above kWalkCap samples, after the fixup
        vmb_packed_view v{out->d_offsets, out->d_counts, rays->n_rays, out->d_t_starts, out->d_t_ends, out->capacity};
        backward_listed(ctx, &v, sr.rgb, sr.sig, sr.dc, sr.dop, sr.ddep, sr.g_rgb, sr.g_sig, bwd_list + 4,
                        reinterpret_cast<const unsigned int*>(bwd_list), sr.dtype);
    }
}

template <typename RT>
void dispatch_expand(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, vmb_samples* out,
                     const uint32_t* kept_idx, uint32_t* overflow, unsigned int* n_overflow,
                     uint64_t n_chunks, const ShadeReq& sr, const uint32_t* chunk_off, uint32_t* bwd_list,
                     const void* kept_attr) {
#define VMB_EXPAND(AT, SH, FW, VX) \
    launch_expand_fixup<RT, AT, SH, FW, VX>(ctx, P, rays, out, kept_idx, overflow, n_overflow, n_chunks, sr, \
                                            chunk_off, bwd_list, kept_attr)
    const bool vox = P.f.kind == VMB_FIELD_VOXEL;
    if (!sr.on)
        vox ? VMB_EXPAND(float, false, false, true) : VMB_EXPAND(float, false, false, false);
    else if (sr.dtype == VMB_F32 && vox)
        sr.fwd ? VMB_EXPAND(float, true, true, true) : VMB_EXPAND(float, true, false, true);
    else if (sr.dtype == VMB_F32)
        sr.fwd ? VMB_EXPAND(float, true, true, false) : VMB_EXPAND(float, true, false, false);
    else if (vox)
        sr.fwd ? VMB_EXPAND(double, true, true, true) : VMB_EXPAND(double, true, false, true);
    else
        sr.fwd ? VMB_EXPAND(double, true, true, false) : VMB_EXPAND(double, true, false, false);
#undef VMB_EXPAND
}

// walk -> scan -> expand (+shade) -> fixup; the sample total lands in d_total.
int launch_fused(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, vmb_samples* out,
                 unsigned long long* d_total, unsigned long long* emitted, const ShadeReq& sr) {
    if (int rc = ensure_skip_structures(ctx, P)) return rc;
    const uint64_t n = rays->n_rays;
    const uint64_t n_chunks = (n + 31) / 32;
    // head: [chunk claim, overflow count, scan ticket, pad] + the single-pass scan's
    // status words (one per tile of chunk totals), all zeroed before the walk
    const uint64_t scan_tiles = scan_onepass_tiles(n_chunks);
    const bool onepass = scan_tiles <= 1024;
    const size_t head = onepass ? (16 + 8 * scan_tiles + 15) / 16 * 16 : 16;
    const size_t idx_bytes = n_chunks * kWalkCap * 32 * sizeof(uint32_t);
    // the walk keeps each kept sample's rgb/sigma for the stored voxel field (ATTRM):
    // 16-32 B of scratch per sample instead of a second trilinear stencil (voxel
    // config 5 step 3.01 -> 2.19 ms); an analytic field shades cheaper than the
    // round trip (Checker 1.45 -> 1.56 ms with it)
    const bool attr_on = sr.on && sr.fwd && P.f.kind == VMB_FIELD_VOXEL;
    const size_t attr_bytes = attr_on ? n_chunks * kWalkCap * 32 * 4 * (sr.dtype == VMB_F32 ? 4 : 8) : 0;
    const size_t misc = n * 4 + 8 * n_chunks + (sr.bwd ? 16 + 4 * n : 0) + 64;
    char* base = static_cast<char*>(scratch(ctx, SCRATCH_MARCH, head + idx_bytes + attr_bytes + misc + 256));
    if (!base) return VMB_CUDA;
    auto* counters = reinterpret_cast<unsigned int*>(base);  // [chunk, overflow, scan ticket]
    auto* scan_status = reinterpret_cast<unsigned long long*>(base + 16);
    auto* kept_idx = reinterpret_cast<uint32_t*>(base + head);
    void* kept_attr = attr_on ? static_cast<void*>(base + head + idx_bytes) : nullptr;  // 16 B aligned
    char* rest = base + head + idx_bytes + attr_bytes;
    auto* overflow = reinterpret_cast<uint32_t*>(rest);
    auto* chunk_tot = reinterpret_cast<uint32_t*>(rest + n * 4);  // per-chunk totals
    auto* chunk_off = chunk_tot + n_chunks;                       // and their scan
    auto* bwd_list = chunk_off + n_chunks;  // fused backward: [count, pad x3, rays...]
    zero_words_async(ctx, base, int(head / 4));
    if (n == 0) {
        cudaMemsetAsync(d_total, 0, 8, ctx->stream);
        cudaError_t e = cudaGetLastError();
        return e == cudaSuccess ? VMB_OK : cuda_fail(e, "march");
    }
    // persistent grid: exactly the resident capacity of the device
    auto launch_walk = [&](auto kernel, auto* o, auto* d, auto fo) {
        int per_sm = 0;
        const size_t dyn = size_t(P.atab_n) * 2 * sizeof(double);  // read only by ATAB kernels: alpha, midpoint
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kAccStride, dyn);
        if (per_sm < 1) per_sm = 4;
        launch_pdl(kernel, dim3(ctx->num_sms * per_sm), dim3(kAccStride), dyn, ctx->stream, P, o, d, n, out->d_counts,
                   kept_idx, counters, n_chunks, emitted, ctx->d_err, fo, chunk_tot, kept_attr);
    };
    auto walk_vox = [&](auto* o, auto* d, auto VOXC) {
        using RT = std::remove_const_t<std::remove_pointer_t<decltype(o)>>;
        constexpr bool VX = decltype(VOXC)::value;
        const bool f64 = sr.dtype == VMB_F64;
        if (P.fast && P.atab_n && !VX) {  // SolidSphere: alpha table
            if (!sr.fwd)
                launch_walk(k_march_walk<RT, true, float, false, false, true>, o, d, FwdOut<float>{});
            else if (f64)
                launch_walk(k_march_walk<RT, true, double, true, false, true>, o, d, fwd_out<double>(sr));
            else
                launch_walk(k_march_walk<RT, true, float, true, false, true>, o, d, fwd_out<float>(sr));
        } else if (P.fast) {
            if (!sr.fwd)
                launch_walk(k_march_walk<RT, true, float, false, VX>, o, d, FwdOut<float>{});
            else if (f64)
                attr_on ? launch_walk(k_march_walk<RT, true, double, true, VX, false, true>, o, d, fwd_out<double>(sr))
                        : launch_walk(k_march_walk<RT, true, double, true, VX>, o, d, fwd_out<double>(sr));
            else
                attr_on ? launch_walk(k_march_walk<RT, true, float, true, VX, false, true>, o, d, fwd_out<float>(sr))
                        : launch_walk(k_march_walk<RT, true, float, true, VX>, o, d, fwd_out<float>(sr));
        } else {
            if (!sr.fwd)
                launch_walk(k_march_walk<RT, false, float, false, VX>, o, d, FwdOut<float>{});
            else if (f64)
                attr_on ? launch_walk(k_march_walk<RT, false, double, true, VX, false, true>, o, d, fwd_out<double>(sr))
                        : launch_walk(k_march_walk<RT, false, double, true, VX>, o, d, fwd_out<double>(sr));
            else
                attr_on ? launch_walk(k_march_walk<RT, false, float, true, VX, false, true>, o, d, fwd_out<float>(sr))
                        : launch_walk(k_march_walk<RT, false, float, true, VX>, o, d, fwd_out<float>(sr));
        }
    };
    auto walk_rt = [&](auto* o, auto* d) {
        if (P.f.kind == VMB_FIELD_VOXEL)
            walk_vox(o, d, std::true_type{});
        else
            walk_vox(o, d, std::false_type{});
    };
    if (rays->dtype == VMB_F32)
        walk_rt(static_cast<const float*>(rays->d_origins), static_cast<const float*>(rays->d_directions));
    else
        walk_rt(static_cast<const double*>(rays->d_origins), static_cast<const double*>(rays->d_directions));
    // offsets: the scan of the walk's per-chunk totals, then within each chunk the
    // expansion's warp scan (it writes out->d_offsets)
    int rc = onepass ? scan_counts_onepass(ctx, chunk_tot, n_chunks, chunk_off, d_total, counters + 2, scan_status)
                     : scan_counts(ctx, chunk_tot, n_chunks, chunk_off, d_total);
    if (rc) return rc;
    if (rays->dtype == VMB_F32)
        dispatch_expand<float>(ctx, P, rays, out, kept_idx, overflow, counters + 1, n_chunks, sr, chunk_off, bwd_list,
                               kept_attr);
    else
        dispatch_expand<double>(ctx, P, rays, out, kept_idx, overflow, counters + 1, n_chunks, sr, chunk_off,
                                bwd_list, kept_attr);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "march");
}

// Packed march shared by march_field and march_candidates: the fused single-pass
// kernel when possible, else count -> scan -> (sync) -> fill.
int march_packed(vmb_ctx* ctx, const MarchParams& P, const vmb_rays* rays, vmb_samples* out,
                 uint64_t* h_n, vmb_march_stats* stats, const ShadeReq& sr = ShadeReq{}) {
    if (!out || !out->d_offsets || !out->d_counts)
        return fail(VMB_INVALID_ARGUMENT, "march: output offsets/counts required");
    int rc = reset_error(ctx);
    if (rc) return rc;
    cudaMemsetAsync(ctx->d_u64 + 1, 0, 8, ctx->stream);
    if (use_fused(P)) {
        rc = launch_fused(ctx, P, rays, out, ctx->d_u64, stats ? ctx->d_u64 + 1 : nullptr, sr);
        if (rc) return rc;
        cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 16, cudaMemcpyDeviceToHost, ctx->stream);
        rc = report_march_error(ctx);  // synchronizes
        if (rc) return rc;
        uint64_t total = ctx->h_u64[0];
        *h_n = total;
        if (stats) {
            stats->samples_emitted = ctx->h_u64[1];
            stats->samples_kept = total;
        }
        if (total > 0xffffffffull)
            return fail(VMB_INVALID_ARGUMENT, "pack: sample count exceeds 32-bit index range");
        if (total > out->capacity) return fail(VMB_CAPACITY, "march: sample capacity too small");
        return VMB_OK;
    }
    Slab sl = make_slab(ctx, P, rays->n_rays);
    sl.mode = 1;
    if (sl.cap)
        launch_march<FILL>(ctx, P, rays, out->d_counts, nullptr, out, stats ? ctx->d_u64 + 1 : nullptr, sl);
    else if (rays->n_rays)
        launch_march<COUNT>(ctx, P, rays, out->d_counts, nullptr, nullptr, stats ? ctx->d_u64 + 1 : nullptr);
    rc = scan_counts(ctx, out->d_counts, rays->n_rays, out->d_offsets, ctx->d_u64);
    if (rc) return rc;
    cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 16, cudaMemcpyDeviceToHost, ctx->stream);
    rc = report_march_error(ctx);  // synchronizes
    if (rc) return rc;
    uint64_t total = ctx->h_u64[0];
    *h_n = total;
    if (stats) {
        stats->samples_emitted = ctx->h_u64[1];
        stats->samples_kept = total;
    }
    if (total > 0xffffffffull) return fail(VMB_INVALID_ARGUMENT, "pack: sample count exceeds 32-bit index range");
    if (total > out->capacity) return fail(VMB_CAPACITY, "march: sample capacity too small");
    if (total && sl.cap)
        slab_pack(ctx, P, rays, out, sl);
    else if (total)
        launch_march<FILL>(ctx, P, rays, out->d_counts, out->d_offsets, out, nullptr);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "march fill");
    if (sr.on && sr.fwd && total) {  // long-ray batches: one shade + composite pass
        vmb_packed_view v{out->d_offsets, out->d_counts, rays->n_rays, out->d_t_starts,
                          out->d_t_ends, total};
        rc = shade_forward_long(ctx, rays, &sr.f, sr.time, &v, sr.rgb, sr.sig, sr.color, sr.opacity,
                                sr.depth, sr.dtype);
        if (rc != 1) return rc;
    }
    if (sr.on && total) {
        rc = vmb_shade_field(ctx, rays, &sr.f, sr.time, out->d_ray_indices, out->d_t_starts,
                             out->d_t_ends, total, sr.rgb, sr.sig, sr.dtype);
        if (rc) return rc;
    }
    if (sr.fwd) {  // growth walks are sequential per ray: composite with the render kernel
        vmb_packed_view v{out->d_offsets, out->d_counts, rays->n_rays, out->d_t_starts,
                          out->d_t_ends, total};
        return vmb_render_forward(ctx, &v, sr.rgb, sr.sig, sr.color, sr.opacity, sr.depth, sr.dtype);
    }
    return VMB_OK;
}

}  // namespace
}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_march_field_shaded(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays, const vmb_field* f,
                           const vmb_march_config* cfg, vmb_samples* out, void* d_rgbs, void* d_sigmas,
                           int dtype, double time, uint64_t* h_n, vmb_march_stats* stats) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = stats != nullptr;
    set_sphere_fast(&P);
    ShadeReq sr;
    sr.on = true;
    sr.f = *f;
    sr.time = time;
    sr.rgb = d_rgbs;
    sr.sig = d_sigmas;
    sr.dtype = dtype;
    return march_packed(ctx, P, rays, out, h_n, stats, sr);
}

int vmb_march_render_field(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays, const vmb_field* f,
                           const vmb_march_config* cfg, vmb_samples* out, void* d_rgbs, void* d_sigmas,
                           void* d_color, void* d_opacity, void* d_depth, int dtype, double time,
                           uint64_t* h_n, vmb_march_stats* stats) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = stats != nullptr;
    set_sphere_fast(&P);
    ShadeReq sr;
    sr.on = true;
    sr.f = *f;
    sr.time = time;
    sr.rgb = d_rgbs;
    sr.sig = d_sigmas;
    sr.dtype = dtype;
    // Inline compositing shades at the march position: p - velocity * time must be
    // p itself (up to the sign of zero, which no field distinguishes).
    bool ident = std::isfinite(time) && (time == 0.0 || (f->velocity[0] == 0.0 &&
                                                          f->velocity[1] == 0.0 && f->velocity[2] == 0.0));
    for (int a = 0; a < 3; ++a) ident = ident && std::isfinite(f->velocity[a]);
    if (!ident) {  // shaded march, then the render kernel
        rc = march_packed(ctx, P, rays, out, h_n, stats, sr);
        if (rc) return rc;
        vmb_packed_view v{out->d_offsets, out->d_counts, rays->n_rays, out->d_t_starts, out->d_t_ends, *h_n};
        return vmb_render_forward(ctx, &v, d_rgbs, d_sigmas, d_color, d_opacity, d_depth, dtype);
    }
    sr.fwd = true;
    sr.color = d_color;
    sr.opacity = d_opacity;
    sr.depth = d_depth;
    return march_packed(ctx, P, rays, out, h_n, stats, sr);
}

int vmb_march_field(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays, const vmb_field* f,
                    const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n,
                    vmb_march_stats* stats) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = stats != nullptr;
    set_sphere_fast(&P);
    return march_packed(ctx, P, rays, out, h_n, stats);
}

int vmb_march_field_async(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                          const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out,
                          uint64_t* d_n) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = false;
    set_sphere_fast(&P);
    if (use_fused(P))
        return launch_fused(ctx, P, rays, out, reinterpret_cast<unsigned long long*>(d_n), nullptr,
                            ShadeReq{});
    Slab sl = make_slab(ctx, P, rays->n_rays);
    sl.mode = 1;
    if (sl.cap)
        launch_march<FILL>(ctx, P, rays, out->d_counts, nullptr, out, nullptr, sl);
    else if (rays->n_rays)
        launch_march<COUNT>(ctx, P, rays, out->d_counts, nullptr, nullptr, nullptr);
    rc = scan_counts(ctx, out->d_counts, rays->n_rays, out->d_offsets,
                     reinterpret_cast<unsigned long long*>(d_n));
    if (rc) return rc;
    if (rays->n_rays && sl.cap)
        slab_pack(ctx, P, rays, out, sl);
    else if (rays->n_rays)
        launch_march<FILL>(ctx, P, rays, out->d_counts, out->d_offsets, out, nullptr);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "march async");
}

int vmb_march_render_field_async(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays, const vmb_field* f,
                                 const vmb_march_config* cfg, vmb_samples* out, void* d_rgbs, void* d_sigmas,
                                 void* d_color, void* d_opacity, void* d_depth, int dtype, double time,
                                 uint64_t* d_n) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = false;
    set_sphere_fast(&P);
    bool ident = std::isfinite(time) && (time == 0.0 || (f->velocity[0] == 0.0 &&
                                                          f->velocity[1] == 0.0 && f->velocity[2] == 0.0));
    for (int a = 0; a < 3; ++a) ident = ident && std::isfinite(f->velocity[a]);
    if (!ident || !use_fused(P)) {  // the synchronous path, then publish the total on the device
        uint64_t n = 0;
        rc = vmb_march_render_field(ctx, g, rays, f, cfg, out, d_rgbs, d_sigmas, d_color, d_opacity, d_depth,
                                    dtype, time, &n, nullptr);
        if (rc && rc != VMB_CAPACITY) return rc;
        cudaError_t e = cudaMemcpyAsync(d_n, &n, 8, cudaMemcpyHostToDevice, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        return e == cudaSuccess ? VMB_OK : cuda_fail(e, "march async");
    }
    ShadeReq sr;
    sr.on = true;
    sr.f = *f;
    sr.time = time;
    sr.rgb = d_rgbs;
    sr.sig = d_sigmas;
    sr.dtype = dtype;
    sr.fwd = true;
    sr.color = d_color;
    sr.opacity = d_opacity;
    sr.depth = d_depth;
    return launch_fused(ctx, P, rays, out, reinterpret_cast<unsigned long long*>(d_n), nullptr, sr);
}

int vmb_cascade_level_box(const vmb_contraction* base, uint32_t level, vmb_contraction* out) {
    if (!base || !out || base->kind != VMB_CONTRACT_AABB)
        return fail(VMB_INVALID_ARGUMENT, "cascade: level 0 must be an AABB contraction");
    if (level >= uint32_t(kMaxLevels)) return fail(VMB_INVALID_ARGUMENT, "cascade: at most 7 levels above level 0");
    *out = *base;
    const double s = ldexp(1.0, int(level));
    for (int a = 0; a < 3; ++a) {
        const double c = 0.5 * (base->box_min[a] + base->box_max[a]);
        const double h = 0.5 * (base->box_max[a] - base->box_min[a]);
        out->box_min[a] = c - h * s;
        out->box_max[a] = c + h * s;
    }
    return VMB_OK;
}

int vmb_cascade_query(vmb_ctx* ctx, const vmb_grid* g, const vmb_march_ext* ext, const double* d_points,
                      uint64_t n, uint8_t* d_out) {
    MarchParams P{};
    P.k = g->k;
    P.res = g->res;
    P.bits = g->bits;
    vmb_march_config cfg{1.0, 1e-4, 1e-2, 1, 0, 1.0};
    if (int rc = apply_ext(g, ext, &cfg, &P)) return rc;
    P.exit_box = false;
    if (!n) return VMB_OK;
    int rc = reset_error(ctx);
    if (rc) return rc;
    k_cascade_query<<<grid_blocks(ctx, n, 256), 256, 0, ctx->stream>>>(P, d_points, n, d_out, ctx->d_err);
    DevError err;
    rc = read_error(ctx, &err);
    if (rc) return rc;
    if (err.key != ~0ull) return fail(VMB_INVALID_ARGUMENT, "non-finite coordinate");
    return VMB_OK;
}

int vmb_march_cascade(vmb_ctx* ctx, const vmb_grid* g, const vmb_march_ext* ext, const vmb_rays* rays,
                      const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n,
                      vmb_march_stats* stats) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if ((rc = apply_ext(g, ext, cfg, &P))) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = stats != nullptr;
    set_sphere_fast(&P);
    return march_packed(ctx, P, rays, out, h_n, stats);
}

int vmb_march_render_cascade(vmb_ctx* ctx, const vmb_grid* g, const vmb_march_ext* ext, const vmb_rays* rays,
                             const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out, void* d_rgbs,
                             void* d_sigmas, void* d_color, void* d_opacity, void* d_depth, int dtype, double time,
                             uint64_t* h_n, vmb_march_stats* stats) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if ((rc = apply_ext(g, ext, cfg, &P))) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = stats != nullptr;
    set_sphere_fast(&P);
    ShadeReq sr;
    sr.on = true;
    sr.f = *f;
    sr.time = time;
    sr.rgb = d_rgbs;
    sr.sig = d_sigmas;
    sr.dtype = dtype;
    sr.fwd = true;
    sr.color = d_color;
    sr.opacity = d_opacity;
    sr.depth = d_depth;
    return march_packed(ctx, P, rays, out, h_n, stats, sr);
}

int vmb_march_render_backward_field_async(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                                          const vmb_field* f, const vmb_march_config* cfg, vmb_samples* out,
                                          void* d_rgbs, void* d_sigmas, void* d_color, void* d_opacity, void* d_depth,
                                          const void* d_grad_color, const void* d_grad_opacity,
                                          const void* d_grad_depth, void* d_grad_rgbs, void* d_grad_sigmas,
                                          int dtype, double time, uint64_t* d_n) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    if (int frc = check_field(f)) return frc;
    P.f = *f;
    P.filter = true;
    P.full = false;
    set_sphere_fast(&P);
    bool ident = std::isfinite(time) && (time == 0.0 || (f->velocity[0] == 0.0 &&
                                                          f->velocity[1] == 0.0 && f->velocity[2] == 0.0));
    for (int a = 0; a < 3; ++a) ident = ident && std::isfinite(f->velocity[a]);
    if (!ident || !use_fused(P)) {  // march + render_forward, then render_backward on the result
        rc = vmb_march_render_field_async(ctx, g, rays, f, cfg, out, d_rgbs, d_sigmas, d_color, d_opacity, d_depth,
                                          dtype, time, d_n);
        if (rc) return rc;
        uint64_t n = 0;
        cudaError_t e = cudaMemcpyAsync(&n, d_n, 8, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(e, "march");
        vmb_packed_view v{out->d_offsets, out->d_counts, rays->n_rays, out->d_t_starts, out->d_t_ends,
                          n < out->capacity ? n : out->capacity};
        return vmb_render_backward(ctx, &v, d_rgbs, d_sigmas, d_grad_color, d_grad_opacity, d_grad_depth,
                                   d_grad_rgbs, d_grad_sigmas, dtype);
    }
    ShadeReq sr;
    sr.on = true;
    sr.f = *f;
    sr.time = time;
    sr.rgb = d_rgbs;
    sr.sig = d_sigmas;
    sr.dtype = dtype;
    sr.fwd = true;
    sr.color = d_color;
    sr.opacity = d_opacity;
    sr.depth = d_depth;
    sr.bwd = true;
    sr.dc = d_grad_color;
    sr.dop = d_grad_opacity;
    sr.ddep = d_grad_depth;
    sr.g_rgb = d_grad_rgbs;
    sr.g_sig = d_grad_sigmas;
    return launch_fused(ctx, P, rays, out, reinterpret_cast<unsigned long long*>(d_n), nullptr, sr);
}

int vmb_march_check(vmb_ctx* ctx) {  // reports the recorded error once, then clears the record
    int rc = report_march_error(ctx);
    int rr = reset_error(ctx);
    return rc ? rc : rr;
}

int vmb_march_candidates(vmb_ctx* ctx, const vmb_grid* g, const vmb_rays* rays,
                         const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n) {
    MarchParams P;
    int rc = march_params(g, rays, cfg, &P);
    if (rc) return rc;
    P.filter = false;
    P.full = true;
    return march_packed(ctx, P, rays, out, h_n, nullptr);
}

int vmb_march_filter(vmb_ctx* ctx, const vmb_packed_view* c, const double* sig,
                     const vmb_march_config* cfg, vmb_samples* out, uint64_t* h_n) {
    int rc = validate_config(cfg);
    if (rc) return rc;
    rc = reset_error(ctx);
    if (rc) return rc;
    int blocks = grid_blocks(ctx, c->n_rays, 128, 16);
    if (c->n_rays)
        k_filter<COUNT><<<blocks, 128, 0, ctx->stream>>>(
            c->d_offsets, c->d_counts, c->n_rays, c->d_t_starts, c->d_t_ends, sig, cfg->early_stop_eps,
            cfg->alpha_thre, out->d_counts, nullptr, nullptr, nullptr, nullptr, 0, ctx->d_err);
    rc = scan_counts(ctx, out->d_counts, c->n_rays, out->d_offsets, ctx->d_u64);
    if (rc) return rc;
    cudaMemcpyAsync(ctx->h_u64, ctx->d_u64, 8, cudaMemcpyDeviceToHost, ctx->stream);
    rc = report_march_error(ctx);
    if (rc) return rc;
    *h_n = ctx->h_u64[0];
    if (*h_n > out->capacity) return fail(VMB_CAPACITY, "march: sample capacity too small");
    if (*h_n)
        k_filter<FILL><<<blocks, 128, 0, ctx->stream>>>(
            c->d_offsets, c->d_counts, c->n_rays, c->d_t_starts, c->d_t_ends, sig, cfg->early_stop_eps,
            cfg->alpha_thre, nullptr, out->d_offsets, out->d_t_starts, out->d_t_ends,
            out->d_ray_indices, out->capacity, ctx->d_err);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "march filter");
}

int vmb_march_uniform(vmb_ctx* ctx, const vmb_rays* rays, const vmb_march_config* cfg,
                      vmb_samples* out, uint64_t* h_n) {
    int rc = validate_config(cfg);
    if (rc) return rc;
    if (!(rays->near_plane >= 0.0) || !(rays->far_plane > rays->near_plane))
        return fail(VMB_INVALID_ARGUMENT, "ray batch: requires far > near >= 0");
    bool exact;
    uint64_t n = uniform_step_count(rays->near_plane, rays->far_plane, cfg->step_size);
    uint64_t n_eff = effective_steps(rays->near_plane, rays->far_plane, cfg->step_size, n, &exact);
    if (!exact) return fail(VMB_NOT_SUPPORTED, "march_uniform: lattice longer than 2^26 steps");
    uint64_t total = rays->n_rays * n_eff;
    *h_n = total;
    if (total > 0xffffffffull) return fail(VMB_INVALID_ARGUMENT, "pack: sample count exceeds 32-bit index range");
    if (total > out->capacity) return fail(VMB_CAPACITY, "march: sample capacity too small");
    uint64_t work = total > rays->n_rays ? total : rays->n_rays;
    if (work)
        k_uniform<<<grid_blocks(ctx, work, 256), 256, 0, ctx->stream>>>(
            rays->n_rays, n_eff, rays->near_plane, rays->far_plane, cfg->step_size, out->d_offsets,
            out->d_counts, out->d_t_starts, out->d_t_ends, out->d_ray_indices);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? VMB_OK : cuda_fail(e, "march uniform");
}

}  // extern "C"
