/*
 * vmb200_types.h — plain-old-data descriptors shared by the B200 C ABI
 * (include/vmb200.h) and the CPU oracle (oracle/vm_oracle.h).
 *
 * Every struct is a flat C layout (no pointers, explicit padding) so it can be
 * passed by pointer across the C ABI, through ctypes, and copied verbatim into
 * CUDA constant/parameter space.
 *
 * Reference types each descriptor stands in for (paths under /root/reference):
 *   vmb_contraction   <- voxmarch::Contraction      proj/include/voxmarch/contraction.hpp:14-29
 *   vmb_field         <- voxmarch::AnalyticField    proj/include/voxmarch/fields.hpp:17-37
 *                        (+ TimeConditionedField     proj/include/voxmarch/fields.hpp:123-129)
 *   vmb_march_config  <- voxmarch::MarchingConfig   proj/include/voxmarch/ray_marching.hpp:11-17
 *   vmb_march_stats   <- voxmarch::MarchStats       proj/include/voxmarch/ray_marching.hpp:26-29
 */
#ifndef VMB200_TYPES_H
#define VMB200_TYPES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes of every C-ABI entry point. The C++ facade maps them back to
 * the reference's exception types: INVALID_ARGUMENT -> std::invalid_argument,
 * RUNTIME -> std::runtime_error (throw sites in proj/src). */
enum {
    VMB_OK = 0,
    VMB_INVALID_ARGUMENT = 1,
    VMB_RUNTIME = 2,
    VMB_CUDA = 3,          /* CUDA/driver failure (no device, OOM, launch error) */
    VMB_NOT_SUPPORTED = 4, /* combination not implemented on this path */
    VMB_CAPACITY = 5       /* caller-provided output too small; required size returned */
};

/* Contraction kinds, same numeric tags as Contraction::Kind (contraction.hpp:15). */
enum { VMB_CONTRACT_AABB = 0, VMB_CONTRACT_SPHERE = 1 };

typedef struct vmb_contraction {
    int32_t kind;
    int32_t pad_;
    double box_min[3]; /* AabbNormalize */
    double box_max[3];
    double center[3];  /* SphereContract */
    double radius;
} vmb_contraction;

/* Density/appearance fields: the analytic fields (fields.hpp:17-37,
 * fields.cpp:39-73) and the stored TrilinearVoxelField (fields.hpp:55-111,
 * fields.cpp:95-168) — raw density [R^3] and raw rgb [R^3][3] per lattice vertex,
 * x-fastest, fp64, trilinear + softplus/sigmoid, zero outside box_min..box_max.
 * The voxel pointers are device pointers for vmb_* calls (host pointers for
 * the CPU oracle). */
enum { VMB_FIELD_UNIFORM_BOX = 0, VMB_FIELD_SOLID_SPHERE = 1, VMB_FIELD_CHECKER = 2,
       VMB_FIELD_VOXEL = 3 };

typedef struct vmb_field {
    int32_t kind;
    int32_t pad_;
    double box_min[3]; /* UniformBox::box */
    double box_max[3];
    double center[3];  /* SolidSphere::center */
    double radius;     /* SolidSphere::radius */
    double sigma;      /* all kinds */
    double rgb[3];     /* UniformBox/SolidSphere rgb; Checker rgb_a */
    double rgb_b[3];   /* Checker rgb_b */
    double period;     /* Checker period */
    double velocity[3];/* TimeConditionedField velocity (fields.cpp:264-271); zero = static */
    const double* vox_density; /* TrilinearVoxelField::raw_density_ [R^3] */
    const double* vox_color;   /* TrilinearVoxelField::raw_color_ [R^3][3] */
    uint32_t vox_resolution;   /* vertices per axis (>= 2); box_min/box_max = its box */
    uint32_t pad2_;
} vmb_field;

typedef struct vmb_march_config {
    double step_size;
    double early_stop_eps;
    double alpha_thre;
    uint32_t max_samples_per_ray;
    uint32_t pad_;
    double unbounded_step_growth;
} vmb_march_config;

typedef struct vmb_march_stats {
    uint64_t samples_emitted;
    uint64_t samples_kept;
} vmb_march_stats;

/* Storage precision of ray / attribute / output arrays on the device. Ray
 * marching and compositing always compute in fp64 (SURVEY §0.3 precision
 * hazard); this only selects the element type of the arrays in HBM. */
enum { VMB_F32 = 0, VMB_F64 = 1 };

/* TrilinearVoxelField::backward modes (fields.cpp:170-211). DETERMINISTIC folds
 * each vertex's contributions in sample order exactly like the reference (bitwise
 * equal); ATOMIC uses fp64 atomics (last-bit differences, faster). */
enum { VMB_GRAD_DETERMINISTIC = 0, VMB_GRAD_ATOMIC = 1 };

/* PinholeCamera (scene_camera.hpp:12-19): OpenGL convention (looks down -z, +y
 * up, square pixels); rotation is the row-major world-from-camera Mat3
 * (math.hpp:63-76, m[3*row+col]); position is the eye. */
typedef struct vmb_camera {
    double rotation[9];
    double position[3];
    double focal;  /* pixels */
    int32_t width;
    int32_t height;
} vmb_camera;

#ifdef __cplusplus
}
#endif

#endif /* VMB200_TYPES_H */
