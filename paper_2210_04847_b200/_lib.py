"""ctypes binding of the C ABI (include/vmb200.h) of libvoxmarch_b200.so.

Loading never falls back to anything: if the CUDA library is missing the import
of :func:`lib` raises, and every compute entry point needs a CUDA device
(``vmb_ctx_create`` fails loudly without one).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# VMB_LIB_PATH selects an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("VMB_LIB_PATH") or os.path.join(HERE, "lib", "libvoxmarch_b200.so")

VMB_OK, VMB_INVALID_ARGUMENT, VMB_RUNTIME, VMB_CUDA, VMB_NOT_SUPPORTED, VMB_CAPACITY = range(6)
VMB_F32, VMB_F64 = 0, 1
VMB_GRAD_DETERMINISTIC, VMB_GRAD_ATOMIC = 0, 1


class Contraction(C.Structure):
    """vmb_contraction <- voxmarch::Contraction (contraction.hpp:14-29)."""
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("box_min", C.c_double * 3),
                ("box_max", C.c_double * 3), ("center", C.c_double * 3), ("radius", C.c_double)]

    @staticmethod
    def aabb(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
        c = Contraction()
        c.kind = 0
        c.box_min[:] = [float(v) for v in lo]
        c.box_max[:] = [float(v) for v in hi]
        return c

    @staticmethod
    def sphere(center, radius):
        c = Contraction()
        c.kind = 1
        c.center[:] = [float(v) for v in center]
        c.radius = float(radius)
        return c


class Field(C.Structure):
    """vmb_field <- voxmarch::AnalyticField (fields.hpp:17-37) + time translation."""
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("box_min", C.c_double * 3),
                ("box_max", C.c_double * 3), ("center", C.c_double * 3), ("radius", C.c_double),
                ("sigma", C.c_double), ("rgb", C.c_double * 3), ("rgb_b", C.c_double * 3),
                ("period", C.c_double), ("velocity", C.c_double * 3),
                ("vox_density", C.c_void_p), ("vox_color", C.c_void_p), ("vox_resolution", C.c_uint32),
                ("pad2_", C.c_uint32)]

    @staticmethod
    def sphere(center=(0.5, 0.5, 0.5), radius=0.2, sigma=1.0, rgb=(1.0, 1.0, 1.0),
               velocity=(0.0, 0.0, 0.0)):
        f = Field()
        f.kind = 1
        f.center[:] = [float(v) for v in center]
        f.radius, f.sigma = float(radius), float(sigma)
        f.rgb[:] = [float(v) for v in rgb]
        f.velocity[:] = [float(v) for v in velocity]
        return f

    @staticmethod
    def box(lo, hi, sigma=1.0, rgb=(1.0, 1.0, 1.0), velocity=(0.0, 0.0, 0.0)):
        f = Field()
        f.kind = 0
        f.box_min[:] = [float(v) for v in lo]
        f.box_max[:] = [float(v) for v in hi]
        f.sigma = float(sigma)
        f.rgb[:] = [float(v) for v in rgb]
        f.velocity[:] = [float(v) for v in velocity]
        return f

    @staticmethod
    def checker(period=0.125, sigma=1.0, rgb_a=(1.0, 1.0, 1.0), rgb_b=(0.0, 0.0, 0.0)):
        f = Field()
        f.kind = 2
        f.period, f.sigma = float(period), float(sigma)
        f.rgb[:] = [float(v) for v in rgb_a]
        f.rgb_b[:] = [float(v) for v in rgb_b]
        return f

    @staticmethod
    def voxel(resolution, box_min, box_max, density_ptr, color_ptr, velocity=(0.0, 0.0, 0.0)):
        """TrilinearVoxelField (fields.hpp:55-111): raw density [R^3] / rgb [R^3][3] arrays
        (device pointers for the product, host pointers for the oracle)."""
        f = Field()
        f.kind = 3
        f.box_min[:] = [float(v) for v in box_min]
        f.box_max[:] = [float(v) for v in box_max]
        f.vox_resolution = int(resolution)
        f.vox_density, f.vox_color = density_ptr, color_ptr
        f.velocity[:] = [float(v) for v in velocity]
        return f


class MarchConfig(C.Structure):
    """vmb_march_config <- voxmarch::MarchingConfig (ray_marching.hpp:11-17)."""
    _fields_ = [("step_size", C.c_double), ("early_stop_eps", C.c_double),
                ("alpha_thre", C.c_double), ("max_samples_per_ray", C.c_uint32),
                ("pad_", C.c_uint32), ("unbounded_step_growth", C.c_double)]

    def __init__(self, step_size=1.6914558667664816e-3, early_stop_eps=1e-4, alpha_thre=1e-2,
                 max_samples_per_ray=2048, unbounded_step_growth=1.0):
        super().__init__(step_size, early_stop_eps, alpha_thre, max_samples_per_ray, 0,
                         unbounded_step_growth)


class MarchStats(C.Structure):
    _fields_ = [("samples_emitted", C.c_uint64), ("samples_kept", C.c_uint64)]


class Rays(C.Structure):
    _fields_ = [("d_origins", C.c_void_p), ("d_directions", C.c_void_p), ("dtype", C.c_int32),
                ("pad_", C.c_int32), ("n_rays", C.c_uint64), ("near_plane", C.c_double),
                ("far_plane", C.c_double)]


class Camera(C.Structure):
    """vmb_camera <- voxmarch::PinholeCamera (scene_camera.hpp:12-19)."""
    _fields_ = [("rotation", C.c_double * 9), ("position", C.c_double * 3), ("focal", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Samples(C.Structure):
    _fields_ = [("d_offsets", C.c_void_p), ("d_counts", C.c_void_p), ("d_t_starts", C.c_void_p),
                ("d_t_ends", C.c_void_p), ("d_ray_indices", C.c_void_p), ("capacity", C.c_uint64)]


class PackedView(C.Structure):
    _fields_ = [("d_offsets", C.c_void_p), ("d_counts", C.c_void_p), ("n_rays", C.c_uint64),
                ("d_t_starts", C.c_void_p), ("d_t_ends", C.c_void_p), ("n_samples", C.c_uint64)]


class MarchExt(C.Structure):
    """vmb_march_ext: stacked grid levels (NerfAcc cascades) and cone stepping."""
    _fields_ = [("levels", C.c_void_p), ("n_levels", C.c_uint32), ("cone", C.c_int32),
                ("cone_angle", C.c_double), ("max_step", C.c_double)]


P = C.POINTER
VP, U64, I32, D = C.c_void_p, C.c_uint64, C.c_int, C.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "vmb_last_error": (C.c_char_p, []),
    "vmb_version": (C.c_char_p, []),
    "vmb_device_count": (I32, [P(I32)]),
    "vmb_ctx_create": (I32, [I32, P(VP)]),
    "vmb_ctx_destroy": (I32, [VP]),
    "vmb_ctx_set_stream": (I32, [VP, VP]),
    "vmb_ctx_stream": (VP, [VP]),
    "vmb_ctx_synchronize": (I32, [VP]),
    "vmb_malloc": (I32, [VP, U64, P(VP)]),
    "vmb_free": (I32, [VP, VP]),
    "vmb_host_alloc": (I32, [U64, P(VP)]),
    "vmb_host_free": (I32, [VP]),
    "vmb_memcpy_h2d": (I32, [VP, VP, VP, U64]),
    "vmb_memcpy_d2h": (I32, [VP, VP, VP, U64]),
    "vmb_memcpy_d2h_async": (I32, [VP, VP, VP, U64]),
    "vmb_memcpy_d2d": (I32, [VP, VP, VP, U64]),
    "vmb_memset": (I32, [VP, VP, I32, U64]),
    "vmb_event_record": (I32, [VP, I32]),
    "vmb_ctx_wait": (I32, [VP, VP, I32]),
    "vmb_graph_begin": (I32, [VP]),
    "vmb_graph_end": (I32, [VP, P(VP)]),
    "vmb_graph_launch": (I32, [VP, VP]),
    "vmb_graph_destroy": (I32, [VP]),
    "vmb_event_elapsed_ms": (I32, [VP, I32, I32, P(C.c_float)]),
    "vmb_shard_range": (I32, [U64, I32, I32, P(U64), P(U64)]),
    "vmb_rays_validate": (I32, [VP, P(Rays)]),
    "vmb_field_query": (I32, [VP, P(Field), VP, U64, D, VP, VP]),
    "vmb_voxel_field_backward": (I32, [VP, P(Field), VP, U64, VP, VP, I32, VP, VP, I32]),
    "vmb_voxel_field_backward_samples": (I32, [VP, P(Field), P(Rays), VP, VP, VP, U64, D, VP, VP, I32, VP,
                                               VP, I32]),
    "vmb_adam_step": (I32, [VP, U64, VP, VP, VP, VP, D, D, D, D, U64]),
    "vmb_comm_allreduce_sum_f64": (I32, [VP, VP, U64]),
    "vmb_loss_mse_background": (I32, [VP, VP, VP, VP, U64, I32, VP, VP, VP, P(D)]),
    "vmb_gather_rays": (I32, [VP, VP, VP, VP, VP, U64, I32, VP, VP, VP]),
    "vmb_camera_validate": (I32, [P(Camera)]),
    "vmb_camera_look_at": (I32, [P(C.c_double), P(C.c_double), P(C.c_double), C.c_double, I32, I32,
                                 P(Camera)]),
    "vmb_generate_rays": (I32, [VP, P(Camera), C.c_double, C.c_double, I32, VP, VP, P(Rays)]),
    "vmb_generate_rays_range": (I32, [VP, P(Camera), C.c_double, C.c_double, I32, U64, U64, VP, VP, P(Rays)]),
    "vmb_uniform_step_count": (U64, [D, D, D]),
    "vmb_cascade_level_box": (I32, [P(Contraction), C.c_uint32, P(Contraction)]),
    "vmb_cascade_query": (I32, [VP, VP, P(MarchExt), VP, U64, VP]),
    "vmb_march_cascade": (I32, [VP, VP, P(MarchExt), P(Rays), P(Field), P(MarchConfig), P(Samples), P(U64),
                                P(MarchStats)]),
    "vmb_march_render_cascade": (I32, [VP, VP, P(MarchExt), P(Rays), P(Field), P(MarchConfig), P(Samples), VP, VP,
                                       VP, VP, VP, I32, D, P(U64), P(MarchStats)]),
    "vmb_render_weight_from_density": (I32, [VP, P(PackedView), VP, VP, VP, VP, I32]),
    "vmb_render_weight_from_density_backward": (I32, [VP, P(PackedView), VP, VP, VP, VP, VP, I32]),
    "vmb_render_weight_from_alpha": (I32, [VP, P(PackedView), VP, VP, VP, I32]),
    "vmb_render_weight_from_alpha_backward": (I32, [VP, P(PackedView), VP, VP, VP, VP, I32]),
    "vmb_render_transmittance_from_alpha": (I32, [VP, P(PackedView), VP, VP, I32]),
    "vmb_render_transmittance_from_alpha_backward": (I32, [VP, P(PackedView), VP, VP, VP, I32]),
    "vmb_accumulate_along_rays": (I32, [VP, P(PackedView), VP, VP, U64, VP, I32]),
    "vmb_accumulate_along_rays_backward": (I32, [VP, P(PackedView), VP, VP, U64, VP, VP, VP, I32]),
    "vmb_ray_aabb_intersect": (I32, [VP, P(Rays), VP, U64, D, VP, VP, VP]),
    "vmb_pack": (I32, [VP, VP, U64, VP, VP, U64, P(U64)]),
    "vmb_validate": (I32, [VP, P(PackedView), VP, U64, U64, U64, P(I32)]),
    "vmb_contract": (I32, [VP, P(Contraction), VP, U64, VP]),
    "vmb_invert_grid_point": (I32, [VP, P(Contraction), VP, U64, VP, VP]),
    "vmb_grid_create": (I32, [VP, C.c_uint32, P(Contraction), D, D, D, P(VP)]),
    "vmb_grid_destroy": (I32, [VP]),
    "vmb_grid_clone": (I32, [VP, VP, P(VP)]),
    "vmb_grid_info": (I32, [VP, P(C.c_uint32), P(Contraction), P(D), P(D), P(D)]),
    "vmb_grid_update_field": (I32, [VP, VP, P(Field), P(D), U64, D, I32, U64]),
    "vmb_grid_probe_field_range": (I32, [VP, VP, P(Field), P(D), U64, I32, U64, U64, U64, VP]),
    "vmb_grid_probe_points": (I32, [VP, VP, I32, U64, VP, VP, P(U64)]),
    "vmb_grid_accumulate": (I32, [VP, VP, VP, VP, U64, VP]),
    "vmb_grid_apply": (I32, [VP, VP, VP, D]),
    "vmb_grid_seed_mask": (I32, [VP, VP, VP]),
    "vmb_grid_occupied_count": (I32, [VP, VP, P(U64)]),
    "vmb_grid_query": (I32, [VP, VP, VP, U64, VP]),
    "vmb_grid_read": (I32, [VP, VP, VP, VP]),
    "vmb_grid_write": (I32, [VP, VP, VP, VP]),
    "vmb_grid_read_distance": (I32, [VP, VP, VP, P(C.c_uint32)]),
    "vmb_grid_occupied_bbox": (I32, [VP, VP, VP]),
    "vmb_grid_device_bits": (VP, [VP]),
    "vmb_grid_device_cache": (VP, [VP]),
    "vmb_march_field": (I32, [VP, VP, P(Rays), P(Field), P(MarchConfig), P(Samples), P(U64),
                              P(MarchStats)]),
    "vmb_march_field_shaded": (I32, [VP, VP, P(Rays), P(Field), P(MarchConfig), P(Samples), VP, VP,
                                     I32, D, P(U64), P(MarchStats)]),
    "vmb_march_render_field": (I32, [VP, VP, P(Rays), P(Field), P(MarchConfig), P(Samples), VP, VP,
                                     VP, VP, VP, I32, D, P(U64), P(MarchStats)]),
    "vmb_march_field_async": (I32, [VP, VP, P(Rays), P(Field), P(MarchConfig), P(Samples), VP]),
    "vmb_march_render_field_async": (I32, [VP, VP, P(Rays), P(Field), P(MarchConfig), P(Samples), VP, VP, VP, VP,
                                           VP, I32, D, VP]),
    "vmb_march_check": (I32, [VP]),
    "vmb_march_render_backward_field_async": (I32, [VP, VP, P(Rays), P(Field), P(MarchConfig), P(Samples), VP, VP,
                                                    VP, VP, VP, VP, VP, VP, VP, VP, I32, D, VP]),
    "vmb_march_candidates": (I32, [VP, VP, P(Rays), P(MarchConfig), P(Samples), P(U64)]),
    "vmb_march_filter": (I32, [VP, P(PackedView), VP, P(MarchConfig), P(Samples), P(U64)]),
    "vmb_march_uniform": (I32, [VP, P(Rays), P(MarchConfig), P(Samples), P(U64)]),
    "vmb_shade_field": (I32, [VP, P(Rays), P(Field), D, VP, VP, VP, U64, VP, VP, I32]),
    "vmb_transmittance": (I32, [VP, P(PackedView), VP, VP, I32]),
    "vmb_render_forward": (I32, [VP, P(PackedView), VP, VP, VP, VP, VP, I32]),
    "vmb_render_backward": (I32, [VP, P(PackedView), VP, VP, VP, VP, VP, VP, VP, I32]),
    "vmb_render_attribute": (I32, [VP, P(PackedView), VP, VP, U64, VP, I32]),
    "vmb_comm_unique_id": (I32, [VP]),
    "vmb_comm_init": (I32, [VP, VP, I32, I32]),
    "vmb_comm_destroy": (I32, [VP]),
    "vmb_comm_allreduce_max_f64": (I32, [VP, VP, U64]),
    "vmb_comm_allgather_f64": (I32, [VP, VP, U64]),
}

_LIB = None


class VmbError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.msg = msg


def lib():
    """Load libvoxmarch_b200.so (raises if it was not built: no fallback path)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"CUDA library missing: {LIB_PATH} — run `make` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _LIB = h
    return _LIB


def check(rc: int):
    """Raise the reference's exception type for a VMB status code."""
    if rc == VMB_OK:
        return
    msg = lib().vmb_last_error().decode()
    if rc == VMB_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == VMB_RUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    raise VmbError(rc, msg)
