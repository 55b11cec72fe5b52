// camera.cu — pinhole cameras and device ray generation (scene_camera.cpp:10-63).
//
// generate_rays is the benchmark's ray source: producing the
// rays on the device removes their host->device copy (24 B/ray in f32, 48 B/ray
// in f64). One thread per pixel evaluates the reference's fp64 expressions in the
// same order (file compiled with --fmad=false), so f64 directions are the
// reference's bit for bit; f32 output is that value rounded once.
#include "vm_internal.h"

namespace vmb {
namespace {

// Mat3 * Vec3 (math.hpp:78-80): row dot products, left to right.
VM_HD D3 mat_vec(const double* m, D3 v) {
    return d3(m[0] * v.x + m[1] * v.y + m[2] * v.z, m[3] * v.x + m[4] * v.y + m[5] * v.z,
              m[6] * v.x + m[7] * v.y + m[8] * v.z);
}
VM_HD D3 col_of(const double* m, int i) { return d3(m[i], m[3 + i], m[6 + i]); }
VM_HD D3 cross3(D3 a, D3 b) {  // math.hpp:27-29
    return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
VM_HD D3 div3(D3 a, double s) { return d3(a.x / s, a.y / s, a.z / s); }
VM_HD D3 normalize3(D3 a) { return div3(a, norm(a)); }  // math.hpp:31

template <typename T>
__global__ void k_generate_rays(vmb_camera cam, uint64_t first, uint64_t n, T* __restrict__ o,
                                T* __restrict__ d) {
    const double cx = 0.5 * cam.width;
    const double cy = 0.5 * cam.height;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t px = first + i;  // row-major pixel index
        const int row = int(px / uint64_t(cam.width));
        const int col = int(px - uint64_t(row) * uint64_t(cam.width));
        // pixel centres; image row 0 is the top of the frame (scene_camera.cpp:56-58)
        const D3 dir_cam = d3((double(col) + 0.5 - cx) / cam.focal, (cy - (double(row) + 0.5)) / cam.focal, -1.0);
        const D3 w = normalize3(mat_vec(cam.rotation, dir_cam));
        o[3 * i] = T(cam.position[0]);
        o[3 * i + 1] = T(cam.position[1]);
        o[3 * i + 2] = T(cam.position[2]);
        d[3 * i] = T(w.x);
        d[3 * i + 1] = T(w.y);
        d[3 * i + 2] = T(w.z);
    }
}

}  // namespace
}  // namespace vmb

using namespace vmb;

extern "C" {

int vmb_camera_validate(const vmb_camera* c) {
    if (!c) return fail(VMB_INVALID_ARGUMENT, "camera: null");
    if (c->width <= 0 || c->height <= 0)
        return fail(VMB_INVALID_ARGUMENT, "camera: image dimensions must be positive");
    if (!(c->focal > 0.0)) return fail(VMB_INVALID_ARGUMENT, "camera: focal must be > 0");
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double dd = dot(col_of(c->rotation, i), col_of(c->rotation, j)) - (i == j ? 1.0 : 0.0);
            if (std::abs(dd) > 1e-6) return fail(VMB_INVALID_ARGUMENT, "camera: rotation is not orthonormal");
        }
    const double det = dot(col_of(c->rotation, 0), cross3(col_of(c->rotation, 1), col_of(c->rotation, 2)));
    if (std::abs(det - 1.0) > 1e-6) return fail(VMB_INVALID_ARGUMENT, "camera: rotation determinant must be +1");
    return VMB_OK;
}

int vmb_camera_look_at(const double eye[3], const double target[3], const double up[3], double focal,
                       int32_t width, int32_t height, vmb_camera* out) {
    const D3 e = d3(eye[0], eye[1], eye[2]), t = d3(target[0], target[1], target[2]);
    const D3 offset = e - t;
    if (norm(offset) < 1e-12) return fail(VMB_INVALID_ARGUMENT, "look_at: eye and target coincide");
    const D3 z = normalize3(offset);  // the camera looks down -z, toward the target
    D3 x = cross3(d3(up[0], up[1], up[2]), z);
    if (norm(x) < 1e-9) return fail(VMB_INVALID_ARGUMENT, "look_at: up is parallel to view direction");
    x = normalize3(x);
    const D3 y = cross3(z, x);
    vmb_camera c{};
    const double cols[3][3] = {{x.x, x.y, x.z}, {y.x, y.y, y.z}, {z.x, z.y, z.z}};
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) c.rotation[3 * r + k] = cols[k][r];  // Mat3::from_columns
    c.position[0] = e.x, c.position[1] = e.y, c.position[2] = e.z;
    c.focal = focal;
    c.width = width;
    c.height = height;
    int rc = vmb_camera_validate(&c);
    if (rc) return rc;
    *out = c;
    return VMB_OK;
}

int vmb_generate_rays_range(vmb_ctx* ctx, const vmb_camera* camera, double near_plane, double far_plane,
                            int dtype, uint64_t first_ray, uint64_t n_rays, void* d_origins, void* d_directions,
                            vmb_rays* out_rays) {
    int rc = vmb_camera_validate(camera);
    if (rc) return rc;
    // RayBatch::create (core_types.cpp:13-20). Directions are unit by construction
    // (normalize of a vector with |z| = 1); only the shared origin can be non-finite.
    if (!(near_plane >= 0.0) || !(far_plane > near_plane))
        return fail(VMB_INVALID_ARGUMENT, "ray batch: requires far > near >= 0");
    if (uint64_t(camera->width) * uint64_t(camera->height) > 0 &&
        !(std::isfinite(camera->position[0]) && std::isfinite(camera->position[1]) &&
          std::isfinite(camera->position[2])))
        return fail(VMB_INVALID_ARGUMENT, "ray batch: non-finite ray at index 0");
    if (dtype != VMB_F32 && dtype != VMB_F64) return fail(VMB_INVALID_ARGUMENT, "generate_rays: dtype");
    const uint64_t total = uint64_t(camera->width) * uint64_t(camera->height);
    if (first_ray > total || n_rays > total - first_ray)
        return fail(VMB_INVALID_ARGUMENT, "generate_rays: ray range outside the image");
    const uint64_t n = n_rays;
    if (n) {
        const int blocks = grid_blocks(ctx, n, 256, 8);
        if (dtype == VMB_F32)
            k_generate_rays<float><<<blocks, 256, 0, ctx->stream>>>(
                *camera, first_ray, n, static_cast<float*>(d_origins), static_cast<float*>(d_directions));
        else
            k_generate_rays<double><<<blocks, 256, 0, ctx->stream>>>(
                *camera, first_ray, n, static_cast<double*>(d_origins), static_cast<double*>(d_directions));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "generate_rays");
    }
    if (out_rays) {
        *out_rays = vmb_rays{d_origins, d_directions, int32_t(dtype), 0, n, near_plane, far_plane};
    }
    return VMB_OK;
}

int vmb_generate_rays(vmb_ctx* ctx, const vmb_camera* camera, double near_plane, double far_plane, int dtype,
                      void* d_origins, void* d_directions, vmb_rays* out_rays) {
    const uint64_t n = camera && camera->width > 0 && camera->height > 0
                           ? uint64_t(camera->width) * uint64_t(camera->height)
                           : 0;
    return vmb_generate_rays_range(ctx, camera, near_plane, far_plane, dtype, 0, n, d_origins, d_directions,
                                   out_rays);
}

}  // extern "C"
