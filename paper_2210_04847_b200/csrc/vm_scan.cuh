// vm_scan.cuh — segmented warp scans along rays (shared by ops.cu and the fused
// training step in march.cu). One sample per lane; a ray is a segment, the scans
// continue across rounds of 32 samples through a carry.
#pragma once

namespace vmb {

// Exclusive segmented product of m over the warp's 32 lanes (head flag at each
// ray's first sample), continuing `carry` (the running product of the ray that is
// open at lane 0) — returns T before this lane's sample, updates carry.
__device__ __forceinline__ double seg_excl_prod(double m, bool head, double& carry) {
    double x = m;
    int f = head;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, d);
        const int g = __shfl_up_sync(0xffffffffu, f, d);
        if (lane >= d) {
            if (!f) x = y * x;
            f |= g;
        }
    }
    if (!f) x = carry * x;  // the segment open at lane 0 continues the previous round
    double t = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) t = carry;
    if (head) t = 1.0;
    carry = __shfl_sync(0xffffffffu, x, 31);
    return t;
}

// Reverse segmented scan of affine maps (c, m): inclusive V_i = c_i + m_i V_{i+1}
// within a ray (tail flag at its last sample), continuing `carry` (V at lane 0 of
// the next round, for the ray still open at lane 31). Returns the EXCLUSIVE value
// W_i = V_{i+1} (0 at a tail) and updates carry for the previous round. With m = 1
// it is the suffix sum of c accumulated from the ray's end.
__device__ __forceinline__ double seg_excl_affine_rev(double c, double m, bool tail, double& carry) {
    int f = tail;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double c2 = __shfl_down_sync(0xffffffffu, c, d);
        const double m2 = __shfl_down_sync(0xffffffffu, m, d);
        const int g = __shfl_down_sync(0xffffffffu, f, d);
        if (lane + d < 32) {
            if (!f) {
                c = c + m * c2;
                m = m * m2;
            }
            f |= g;
        }
    }
    const double v = f ? c : c + m * carry;  // inclusive V_i
    double w = __shfl_down_sync(0xffffffffu, v, 1);
    if (lane == 31) w = carry;
    if (tail) w = 0.0;
    carry = __shfl_sync(0xffffffffu, v, 0);
    return w;
}

// seg_excl_affine_rev with m = 1: sum of c over the later samples of the ray.
__device__ __forceinline__ double seg_excl_sum_rev(double c, bool tail, double& carry) {
    int f = tail;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double c2 = __shfl_down_sync(0xffffffffu, c, d);
        const int g = __shfl_down_sync(0xffffffffu, f, d);
        if (lane + d < 32) {
            if (!f) c = c + c2;
            f |= g;
        }
    }
    const double v = f ? c : c + carry;
    double w = __shfl_down_sync(0xffffffffu, v, 1);
    if (lane == 31) w = carry;
    if (tail) w = 0.0;
    carry = __shfl_sync(0xffffffffu, v, 0);
    return w;
}

}  // namespace vmb
