"""Python mirror of the reference's hot-path API, executed by the B200 library.

Names, argument meaning and errors follow namespace ``voxmarch`` of the reference
(proj/include/voxmarch/*.hpp) exactly like the C++ facade
(include/voxmarch/voxmarch.hpp) does: value semantics over host numpy arrays,
``ValueError`` where the reference throws ``std::invalid_argument`` and
``RuntimeError`` for ``std::runtime_error``, with identical messages. Every
computation runs in the CUDA kernels of libvoxmarch_b200.so; host code only
moves data and calls user callbacks (SigmaFn / DensityBatchFn), as the reference
API requires.

The device-resident layer underneath (:class:`Device`, :class:`DeviceArray`,
:func:`march_device` ...) is what bench.py times.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field as dc_field
from typing import Callable, Optional

import numpy as np

from ._lib import (VMB_CAPACITY, VMB_F32, VMB_F64, Camera, Contraction, Field, MarchConfig, MarchExt,
                   MarchStats, PackedView, Rays, Samples, VmbError, check, lib)

__all__ = ["Device", "DeviceArray", "default_device", "Contraction", "Field", "MarchConfig",
           "MarchStats", "RayBatch", "PackedSamples", "OccupancyGrid", "march", "march_uniform",
           "uniform_step_count", "pack", "validate", "transmittance", "render_forward",
           "render_backward", "render_attribute", "contract", "invert_grid_point",
           "DevicePacked", "march_device", "shade_device", "render_forward_device",
           "render_backward_device", "shard_range", "Camera", "look_at", "generate_rays_device",
           "generate_rays", "VoxelField", "field_query_device"]


# ====================================================================== device layer
class Device:
    """A CUDA context of the library (vmb_ctx): device, stream, scratch, error record."""

    def __init__(self, index: int = 0):
        self.lib = lib()
        self.h = C.c_void_p()
        check(self.lib.vmb_ctx_create(index, C.byref(self.h)))
        self.index = index

    def close(self):
        if self.h:
            self.lib.vmb_ctx_destroy(self.h)
            self.h = C.c_void_p()

    # No __del__: device arrays may be garbage-collected after their context (cycle
    # collection order is arbitrary), so a context lives until close() or exit.

    def sync(self):
        check(self.lib.vmb_ctx_synchronize(self.h))

    def empty(self, shape, dtype) -> "DeviceArray":
        return DeviceArray(self, shape, dtype)

    def zeros(self, shape, dtype) -> "DeviceArray":
        a = DeviceArray(self, shape, dtype)
        check(self.lib.vmb_memset(self.h, a.ptr, 0, a.nbytes))
        return a

    def upload(self, host, dtype=None) -> "DeviceArray":
        host = np.ascontiguousarray(host if dtype is None else np.asarray(host, dtype=dtype))
        a = DeviceArray(self, host.shape, host.dtype)
        check(self.lib.vmb_memcpy_h2d(self.h, a.ptr, host.ctypes.data, host.nbytes))
        return a

    def record(self, slot: int):
        check(self.lib.vmb_event_record(self.h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        check(self.lib.vmb_event_elapsed_ms(self.h, a, b, C.byref(ms)))
        return float(ms.value)


class DeviceArray:
    """Owning device allocation with a numpy-like shape/dtype."""

    def __init__(self, dev: Device, shape, dtype):
        self.dev = dev
        self.shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        self.dtype = np.dtype(dtype)
        self.nbytes = int(np.prod(self.shape, dtype=np.int64)) * self.dtype.itemsize
        p = C.c_void_p()
        check(dev.lib.vmb_malloc(dev.h, max(self.nbytes, 16), C.byref(p)))
        self.ptr = p.value

    def free(self):
        if self.ptr and self.dev.h:
            self.dev.lib.vmb_free(self.dev.h, self.ptr)
        self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def numpy(self, count: Optional[int] = None) -> np.ndarray:
        shape = self.shape if count is None else (count,) + self.shape[1:]
        out = np.empty(shape, self.dtype)
        if out.nbytes:
            check(self.dev.lib.vmb_memcpy_d2h(self.dev.h, out.ctypes.data, self.ptr, out.nbytes))
        return out

    def copy_from(self, host: np.ndarray):
        host = np.ascontiguousarray(host, dtype=self.dtype)
        assert host.nbytes <= self.nbytes
        check(self.dev.lib.vmb_memcpy_h2d(self.dev.h, self.ptr, host.ctypes.data, host.nbytes))


_DEFAULT: Optional[Device] = None


def default_device() -> Device:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Device(0)
    return _DEFAULT


def shard_range(n: int, nranks: int, rank: int):
    """Rank's contiguous slice of n units (host-only; parallel.hpp:28-35 split)."""
    b, e = C.c_uint64(), C.c_uint64()
    check(lib().vmb_shard_range(n, nranks, rank, C.byref(b), C.byref(e)))
    return int(b.value), int(e.value)


def _dt(dtype) -> int:
    return VMB_F32 if np.dtype(dtype) == np.float32 else VMB_F64


def device_rays(dev: Device, origins: DeviceArray, dirs: DeviceArray, near: float,
                far: float) -> Rays:
    return Rays(origins.ptr, dirs.ptr, _dt(origins.dtype), 0, origins.shape[0], near, far)


@dataclass
class DevicePacked:
    """Device PackedSamples (caller-owned buffers, capacity protocol)."""
    offsets: DeviceArray
    counts: DeviceArray
    t_starts: DeviceArray
    t_ends: DeviceArray
    ray_indices: DeviceArray
    n_rays: int
    n_samples: int = 0

    @staticmethod
    def allocate(dev: Device, n_rays: int, capacity: int) -> "DevicePacked":
        cap = max(int(capacity), 1)
        return DevicePacked(dev.empty(max(n_rays, 1), np.uint32), dev.empty(max(n_rays, 1), np.uint32),
                            dev.empty(cap, np.float64), dev.empty(cap, np.float64),
                            dev.empty(cap, np.uint32), n_rays)

    @property
    def capacity(self) -> int:
        return self.t_starts.shape[0]

    def samples_struct(self) -> Samples:
        return Samples(self.offsets.ptr, self.counts.ptr, self.t_starts.ptr, self.t_ends.ptr,
                       self.ray_indices.ptr, self.capacity)

    def view(self) -> PackedView:
        return PackedView(self.offsets.ptr, self.counts.ptr, self.n_rays, self.t_starts.ptr,
                          self.t_ends.ptr, self.n_samples)

    def to_host(self) -> "PackedSamples":
        n, s = self.n_rays, self.n_samples
        return PackedSamples(self.offsets.numpy(n), self.counts.numpy(n), self.t_starts.numpy(s),
                             self.t_ends.numpy(s), self.ray_indices.numpy(s))


def march_device(dev: Device, grid: "OccupancyGrid", rays: Rays, field: Field, cfg: MarchConfig,
                 out: DevicePacked, stats: Optional[MarchStats] = None) -> DevicePacked:
    """vmb_march_field into caller buffers; grows them once on VMB_CAPACITY."""
    n = C.c_uint64()
    smp = out.samples_struct()
    rc = dev.lib.vmb_march_field(dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                 C.byref(smp), C.byref(n), C.byref(stats) if stats is not None else None)
    if rc == VMB_CAPACITY:
        grown = DevicePacked.allocate(dev, out.n_rays, int(n.value * 1.25) + 1024)
        out.t_starts, out.t_ends, out.ray_indices = grown.t_starts, grown.t_ends, grown.ray_indices
        smp = out.samples_struct()
        rc = dev.lib.vmb_march_field(dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                     C.byref(smp), C.byref(n),
                                     C.byref(stats) if stats is not None else None)
    check(rc)
    out.n_samples = int(n.value)
    return out


def march_shaded_device(dev: Device, grid: "OccupancyGrid", rays: Rays, field: Field,
                        cfg: MarchConfig, out: DevicePacked, rgbs: DeviceArray, sigmas: DeviceArray,
                        time: float = 0.0, stats: Optional[MarchStats] = None) -> DevicePacked:
    """vmb_march_field_shaded: march + analytic shading fused (buffers must be large enough)."""
    n = C.c_uint64()
    smp = out.samples_struct()
    check(dev.lib.vmb_march_field_shaded(dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                         C.byref(smp), rgbs.ptr, sigmas.ptr, _dt(rgbs.dtype), time,
                                         C.byref(n), C.byref(stats) if stats is not None else None))
    out.n_samples = int(n.value)
    return out


def march_render_device(dev: Device, grid: "OccupancyGrid", rays: Rays, field: Field,
                        cfg: MarchConfig, out: DevicePacked, rgbs: DeviceArray, sigmas: DeviceArray,
                        color: DeviceArray, opacity: DeviceArray, depth: DeviceArray,
                        time: float = 0.0, stats: Optional[MarchStats] = None) -> DevicePacked:
    """vmb_march_render_field: march + analytic shading + render_forward fused."""
    n = C.c_uint64()
    smp = out.samples_struct()
    check(dev.lib.vmb_march_render_field(dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                         C.byref(smp), rgbs.ptr, sigmas.ptr, color.ptr, opacity.ptr,
                                         depth.ptr, _dt(rgbs.dtype), time, C.byref(n),
                                         C.byref(stats) if stats is not None else None))
    out.n_samples = int(n.value)
    return out


def march_render_backward_device(dev: Device, grid: "OccupancyGrid", rays: Rays, field: Field,
                                 cfg: MarchConfig, out: DevicePacked, rgbs: DeviceArray, sigmas: DeviceArray,
                                 color: DeviceArray, opacity: DeviceArray, depth: DeviceArray, d_color, d_opacity,
                                 d_depth, g_rgbs: DeviceArray, g_sigmas: DeviceArray, n_dev: DeviceArray,
                                 time: float = 0.0):
    """vmb_march_render_backward_field_async: the whole training step (march + shading
    + render_forward + render_backward) on the context's stream; the sample total
    stays on the device (n_dev, u64); errors are deferred to vmb_march_check. The
    upstream gradients are device arrays (or objects with .ptr) in rgbs' dtype."""
    smp = out.samples_struct()
    check(dev.lib.vmb_march_render_backward_field_async(
        dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg), C.byref(smp), rgbs.ptr, sigmas.ptr, color.ptr,
        opacity.ptr, depth.ptr, d_color.ptr, d_opacity.ptr, d_depth.ptr, g_rgbs.ptr, g_sigmas.ptr, _dt(rgbs.dtype),
        time, n_dev.ptr))
    out.n_samples = out.capacity
    return out


def shade_device(dev: Device, rays: Rays, field: Field, packed: DevicePacked, rgbs: DeviceArray,
                 sigmas: DeviceArray, time: float = 0.0):
    check(dev.lib.vmb_shade_field(dev.h, C.byref(rays), C.byref(field), time,
                                  packed.ray_indices.ptr, packed.t_starts.ptr, packed.t_ends.ptr,
                                  packed.n_samples, rgbs.ptr, sigmas.ptr, _dt(rgbs.dtype)))


def render_forward_device(dev: Device, packed: DevicePacked, rgbs: DeviceArray, sigmas: DeviceArray,
                          color: DeviceArray, opacity: DeviceArray, depth: DeviceArray):
    v = packed.view()
    check(dev.lib.vmb_render_forward(dev.h, C.byref(v), rgbs.ptr, sigmas.ptr, color.ptr, opacity.ptr,
                                     depth.ptr, _dt(rgbs.dtype)))


def render_backward_device(dev: Device, packed: DevicePacked, rgbs: DeviceArray, sigmas: DeviceArray,
                           d_color: DeviceArray, d_opacity: DeviceArray, d_depth: DeviceArray,
                           g_rgbs: DeviceArray, g_sigmas: DeviceArray):
    v = packed.view()
    check(dev.lib.vmb_render_backward(dev.h, C.byref(v), rgbs.ptr, sigmas.ptr, d_color.ptr,
                                      d_opacity.ptr, d_depth.ptr, g_rgbs.ptr, g_sigmas.ptr,
                                      _dt(rgbs.dtype)))


# ====================================================================== cameras
def look_at(eye, target, up, focal: float, width: int, height: int) -> Camera:
    """voxmarch::look_at (scene_camera.cpp:25-44), host-side, exact fp64."""
    d3 = lambda v: (C.c_double * 3)(*[float(x) for x in v])
    cam = Camera()
    check(lib().vmb_camera_look_at(d3(eye), d3(target), d3(up), float(focal), int(width), int(height),
                                   C.byref(cam)))
    return cam


def generate_rays_device(dev: Device, cam: Camera, near: float, far: float, dtype=np.float32,
                         origins: Optional["DeviceArray"] = None, dirs: Optional["DeviceArray"] = None):
    """vmb_generate_rays: one ray per pixel on the device (scene_camera.cpp:46-63).
    Returns (Rays, origins, dirs); the arrays may be passed in to be reused."""
    n = max(cam.width, 0) * max(cam.height, 0)
    origins = origins if origins is not None else dev.empty(n * 3, dtype)
    dirs = dirs if dirs is not None else dev.empty(n * 3, dtype)
    rays = Rays()
    check(dev.lib.vmb_generate_rays(dev.h, C.byref(cam), float(near), float(far), _dt(dtype), origins.ptr,
                                    dirs.ptr, C.byref(rays)))
    return rays, origins, dirs


def generate_rays(cam: Camera, near: float, far: float, dev: Optional[Device] = None) -> "RayBatch":
    """voxmarch::generate_rays: the batch on the device (f64), as a RayBatch."""
    dev = dev or default_device()
    rays, o, d = generate_rays_device(dev, cam, near, far, np.float64)
    n = int(rays.n_rays)
    return RayBatch(o.numpy(3 * n).reshape(n, 3), d.numpy(3 * n).reshape(n, 3), near, far)


# ====================================================================== fields
def field_query_device(dev: Device, field: Field, points: "DeviceArray", n: int, time: float = 0.0,
                       rgb: bool = True):
    """vmb_field_query: sigma [n] (and rgb [n][3]) f64 on the device."""
    sig = dev.empty(n, np.float64)
    col = dev.empty(n * 3, np.float64) if rgb else None
    check(dev.lib.vmb_field_query(dev.h, C.byref(field), points.ptr, n, float(time), sig.ptr,
                                  col.ptr if col is not None else None))
    return sig, col


class VoxelField:
    """voxmarch::TrilinearVoxelField (fields.hpp:55-111) with its parameters in HBM
    (raw density [R^3] and raw rgb [R^3][3], f64, x-fastest). `field` is the
    vmb_field descriptor every march / shade / grid-update entry point accepts."""

    MAGIC, VERSION = b"VXFD", 1

    def __init__(self, resolution: int, box_min, box_max, dev: Optional[Device] = None):
        if resolution < 2:
            raise ValueError("voxel field: resolution must be >= 2 vertices per axis")
        lo, hi = [float(v) for v in box_min], [float(v) for v in box_max]
        if not all(b > a for a, b in zip(lo, hi)):
            raise ValueError("aabb max must be strictly greater than min")
        self.dev = dev or default_device()
        self.resolution, self.box_min, self.box_max = int(resolution), lo, hi
        nv = self.n_vertices
        self.d_density = self.dev.zeros(nv, np.float64)
        self.d_color = self.dev.zeros(3 * nv, np.float64)
        self.field = Field.voxel(self.resolution, lo, hi, self.d_density.ptr, self.d_color.ptr)

    @property
    def n_vertices(self) -> int:
        return self.resolution ** 3

    def vertex_index(self, ix, iy, iz) -> int:
        return int(ix) + self.resolution * (int(iy) + self.resolution * int(iz))

    def set_params(self, raw_density=None, raw_color=None):
        if raw_density is not None:
            self.d_density.copy_from(np.asarray(raw_density, np.float64).ravel())
        if raw_color is not None:
            self.d_color.copy_from(np.asarray(raw_color, np.float64).ravel())

    def raw_density(self) -> np.ndarray:
        return self.d_density.numpy()

    def raw_color(self) -> np.ndarray:
        return self.d_color.numpy()

    def zero_gradients(self):
        nv = self.n_vertices
        return self.dev.zeros(nv, np.float64), self.dev.zeros(3 * nv, np.float64)

    def query_rgb_sigma(self, positions, time: float = 0.0):
        p = _f64(positions).reshape(-1, 3)
        dp = self.dev.upload(p)
        sig, col = field_query_device(self.dev, self.field, dp, len(p), time, True)
        return col.numpy().reshape(-1, 3), sig.numpy()

    def query_density(self, positions, time: float = 0.0):
        p = _f64(positions).reshape(-1, 3)
        sig, _ = field_query_device(self.dev, self.field, self.dev.upload(p), len(p), time, False)
        return sig.numpy()

    def backward(self, positions, d_rgbs, d_sigmas, accum=None, mode: int = 0):
        """Accumulate the parameter gradient (host arrays in, device accumulators
        (d_density, d_color) out); mode 0 = deterministic (reference order)."""
        p = _f64(positions).reshape(-1, 3)
        if len(d_rgbs) != len(p) or len(d_sigmas) != len(p):
            raise ValueError("voxel field: gradient length mismatch")
        acc = accum if accum is not None else self.zero_gradients()
        gr, gs = self.dev.upload(_f64(d_rgbs).reshape(-1, 3)), self.dev.upload(_f64(d_sigmas))
        dp = self.dev.upload(p)
        check(self.dev.lib.vmb_voxel_field_backward(self.dev.h, C.byref(self.field), dp.ptr, len(p), gr.ptr,
                                                    gs.ptr, VMB_F64, acc[0].ptr, acc[1].ptr, int(mode)))
        self.dev.sync()
        return acc

    # VXFD (fields.cpp:224-262): magic, u32 version, u32 resolution, box f64 x6,
    # raw density then raw color as f32.
    def save(self, path: str):
        import struct
        with open(path, "wb") as fh:
            fh.write(self.MAGIC + struct.pack("<II", self.VERSION, self.resolution))
            fh.write(struct.pack("<6d", *self.box_min, *self.box_max))
            fh.write(self.raw_density().astype("<f4").tobytes())
            fh.write(self.raw_color().astype("<f4").tobytes())

    @staticmethod
    def load(path: str, dev: Optional[Device] = None) -> "VoxelField":
        import struct
        with open(path, "rb") as fh:
            if fh.read(4) != VoxelField.MAGIC:
                raise RuntimeError("voxel field: bad magic")
            hdr = fh.read(8)
            if len(hdr) < 8:
                raise RuntimeError("voxel field: truncated stream")
            version, res = struct.unpack("<II", hdr)
            if version != VoxelField.VERSION:
                raise RuntimeError("voxel field: unsupported version")
            box = fh.read(48)
            if len(box) < 48:
                raise RuntimeError("voxel field: truncated stream")
            b = struct.unpack("<6d", box)
            vf = VoxelField(res, b[:3], b[3:], dev)
            nv = vf.n_vertices
            dens, col = fh.read(4 * nv), fh.read(12 * nv)
            if len(dens) < 4 * nv or len(col) < 12 * nv:
                raise RuntimeError("voxel field: truncated stream")
            vf.set_params(np.frombuffer(dens, "<f4").astype(np.float64),
                          np.frombuffer(col, "<f4").astype(np.float64))
            return vf


# ====================================================================== reference mirror
def _v3(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
    return a


@dataclass
class RayBatch:
    """voxmarch::RayBatch (core_types.hpp:15-25): AoS f64 origins/directions, shared near/far."""
    origins: np.ndarray
    directions: np.ndarray
    near: float = 0.0
    far: float = 1.0

    @staticmethod
    def create(origins, directions, near, far, dev: Optional[Device] = None) -> "RayBatch":
        o, d = _v3(origins), _v3(directions)
        if len(o) != len(d):
            raise ValueError("ray batch: origins/directions size mismatch")
        rb = RayBatch(o, d, float(near), float(far))
        dev = dev or default_device()
        do, dd = dev.upload(o), dev.upload(d)
        check(dev.lib.vmb_rays_validate(dev.h, C.byref(device_rays(dev, do, dd, near, far))))
        return rb

    @property
    def n_rays(self):
        return len(self.origins)


@dataclass
class PackedSamples:
    """voxmarch::PackedSamples (core_types.hpp:29-38)."""
    offsets: np.ndarray = dc_field(default_factory=lambda: np.zeros(0, np.uint32))
    counts: np.ndarray = dc_field(default_factory=lambda: np.zeros(0, np.uint32))
    t_starts: np.ndarray = dc_field(default_factory=lambda: np.zeros(0))
    t_ends: np.ndarray = dc_field(default_factory=lambda: np.zeros(0))
    ray_indices: np.ndarray = dc_field(default_factory=lambda: np.zeros(0, np.uint32))

    @property
    def n_rays(self):
        return len(self.counts)

    @property
    def n_samples(self):
        return len(self.t_starts)

    def to_device(self, dev: Device) -> DevicePacked:
        n, s = self.n_rays, self.n_samples
        dp = DevicePacked(dev.upload(_u32(self.offsets) if n else np.zeros(1, np.uint32)),
                          dev.upload(_u32(self.counts) if n else np.zeros(1, np.uint32)),
                          dev.upload(_f64(self.t_starts) if s else np.zeros(1)),
                          dev.upload(_f64(self.t_ends) if s else np.zeros(1)),
                          dev.upload(_u32(self.ray_indices) if len(self.ray_indices) else np.zeros(1, np.uint32)),
                          n, s)
        return dp


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def uniform_step_count(near: float, far: float, step: float) -> int:
    """ray_marching.cpp:51-55."""
    return int(lib().vmb_uniform_step_count(near, far, step))


def pack(counts, dev: Optional[Device] = None):
    """core_types.cpp:30-48 -> (offsets, ray_indices)."""
    dev = dev or default_device()
    counts = _u32(counts)
    n = len(counts)
    total = int(counts.astype(np.uint64).sum())
    dc = dev.upload(counts if n else np.zeros(1, np.uint32))
    off = dev.empty(max(n, 1), np.uint32)
    cap = total if total <= 0xFFFFFFFF else 0
    idx = dev.empty(max(cap, 1), np.uint32)
    t = C.c_uint64()
    check(dev.lib.vmb_pack(dev.h, dc.ptr, n, off.ptr, idx.ptr if cap or not total else None, cap,
                           C.byref(t)))
    return off.numpy(n), idx.numpy(int(t.value))


_VALIDATE = [None, "length mismatch", "offset mismatch", "non-positive interval",
             "non-monotone t_starts", "overlapping intervals", "partition mismatch"]


def validate(p: PackedSamples, dev: Optional[Device] = None) -> Optional[str]:
    """core_types.cpp:50-78: first violated invariant or None."""
    dev = dev or default_device()
    n_off, n_cnt = len(p.offsets), len(p.counts)
    if n_off != n_cnt:
        return "length mismatch"
    d = p.to_device(dev)
    v = PackedView(d.offsets.ptr, d.counts.ptr, n_cnt, d.t_starts.ptr, d.t_ends.ptr, len(p.t_starts))
    res = C.c_int()
    check(dev.lib.vmb_validate(dev.h, C.byref(v), d.ray_indices.ptr, n_off, len(p.ray_indices),
                               len(p.t_ends), C.byref(res)))
    return _VALIDATE[res.value]


def contract(con: Contraction, points, dev: Optional[Device] = None) -> np.ndarray:
    dev = dev or default_device()
    x = _v3(points)
    dx, out = dev.upload(x if len(x) else np.zeros((1, 3))), dev.empty(max(len(x), 1) * 3, np.float64)
    check(dev.lib.vmb_contract(dev.h, C.byref(con), dx.ptr, len(x), out.ptr))
    return out.numpy(len(x) * 3).reshape(-1, 3)


def invert_grid_point(con: Contraction, g, dev: Optional[Device] = None):
    dev = dev or default_device()
    x = _v3(g)
    dx = dev.upload(x if len(x) else np.zeros((1, 3)))
    out, valid = dev.empty(max(len(x), 1) * 3, np.float64), dev.empty(max(len(x), 1), np.uint8)
    check(dev.lib.vmb_invert_grid_point(dev.h, C.byref(con), dx.ptr, len(x), out.ptr, valid.ptr))
    return out.numpy(len(x) * 3).reshape(-1, 3), valid.numpy(len(x)).astype(bool)


class OccupancyGrid:
    """voxmarch::OccupancyGrid (occupancy_grid.hpp:24-89), resident in HBM."""

    def __init__(self, resolution: int, contraction: Contraction, alpha_threshold: float = 1e-2,
                 reference_step: float = 0.0, initial_density: float = 0.0,
                 dev: Optional[Device] = None):
        self.dev = dev or default_device()
        self.h = C.c_void_p()
        check(self.dev.lib.vmb_grid_create(self.dev.h, int(resolution), C.byref(contraction),
                                           alpha_threshold, reference_step, initial_density,
                                           C.byref(self.h)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.dev.lib.vmb_grid_destroy(h)
            self.h = None

    def _info(self):
        res, con = C.c_uint32(), Contraction()
        thr, ref, thd = C.c_double(), C.c_double(), C.c_double()
        check(self.dev.lib.vmb_grid_info(self.h, C.byref(res), C.byref(con), C.byref(thr),
                                         C.byref(ref), C.byref(thd)))
        return res.value, con, thr.value, ref.value, thd.value

    @property
    def resolution(self):
        return self._info()[0]

    @property
    def contraction(self):
        return self._info()[1]

    @property
    def alpha_threshold(self):
        return self._info()[2]

    @property
    def reference_step(self):
        return self._info()[3]

    def threshold_density(self):
        return self._info()[4]

    @property
    def n_cells(self):
        return self.resolution ** 3

    def cell_index(self, ix, iy, iz):
        r = self.resolution
        return ix + r * (iy + r * iz)

    def bits(self) -> np.ndarray:
        n = self.n_cells
        b = np.zeros((n + 7) // 8, np.uint8)
        check(self.dev.lib.vmb_grid_read(self.dev.h, self.h, b.ctypes.data, None))
        return np.unpackbits(b, bitorder="little")[:n]

    def distance_map(self) -> np.ndarray:
        """The marcher's capped L-inf distance map (u8 per cell) and its cap."""
        d = np.zeros(self.n_cells, np.uint8)
        cap = C.c_uint32()
        check(self.dev.lib.vmb_grid_read_distance(self.dev.h, self.h, d.ctypes.data, C.byref(cap)))
        return d, int(cap.value)

    def occupied_bbox(self) -> np.ndarray:
        """The marcher's ray clip box: occupied cells' {min xyz, max+1 xyz} (u32[6])."""
        b = np.zeros(6, np.uint32)
        check(self.dev.lib.vmb_grid_occupied_bbox(self.dev.h, self.h, b.ctypes.data))
        return b

    def packed_bits(self) -> np.ndarray:
        b = np.zeros((self.n_cells + 7) // 8, np.uint8)
        check(self.dev.lib.vmb_grid_read(self.dev.h, self.h, b.ctypes.data, None))
        return b

    def density_cache(self) -> np.ndarray:
        c = np.zeros(self.n_cells)
        check(self.dev.lib.vmb_grid_read(self.dev.h, self.h, None, c.ctypes.data))
        return c

    def bit(self, cell):
        return bool(self.bits()[cell])

    def occupied_fraction(self) -> float:
        cnt = C.c_uint64()
        check(self.dev.lib.vmb_grid_occupied_count(self.dev.h, self.h, C.byref(cnt)))
        return float(cnt.value) / float(self.n_cells)

    def query(self, points) -> np.ndarray:
        x = _v3(points)
        dx, out = self.dev.upload(x if len(x) else np.zeros((1, 3))), self.dev.empty(max(len(x), 1), np.uint8)
        check(self.dev.lib.vmb_grid_query(self.dev.h, self.h, dx.ptr, len(x), out.ptr))
        return out.numpy(len(x)).astype(bool)

    # -------------------------------------------------------------- updates
    def update_field(self, field: Field, ema_decay: float, jitter_seed: Optional[int] = None,
                     timestamps=(0.0,)):
        """Device fast path: analytic field evaluated inside the probe kernel."""
        ts = _f64(timestamps)
        check(self.dev.lib.vmb_grid_update_field(
            self.dev.h, self.h, C.byref(field), ts.ctypes.data_as(C.POINTER(C.c_double)), len(ts),
            ema_decay, jitter_seed is not None, 0 if jitter_seed is None else int(jitter_seed)))

    def update(self, density_fn: Callable, ema_decay: float, jitter_seed: Optional[int] = None):
        """OccupancyGrid::update with a host DensityBatchFn (occupancy_grid.cpp:91-96)."""
        self.update_over_time(lambda p, t: density_fn(p), (0.0,), ema_decay, jitter_seed)

    def update_over_time(self, density_fn: Callable, timestamps, ema_decay: float,
                         jitter_seed: Optional[int] = None):
        """occupancy_grid.cpp:98-144 with a host TimeDensityBatchFn(points, t)."""
        ts = list(timestamps)
        if not ts:
            raise ValueError("occupancy grid: timestamps must be non-empty")
        if not (0.0 <= ema_decay <= 1.0):
            raise ValueError("occupancy grid: ema_decay must be in [0,1]")
        dev, n = self.dev, self.n_cells
        pts, cells = dev.empty(n * 3, np.float64), dev.empty(n, np.uint32)
        m = C.c_uint64()
        check(dev.lib.vmb_grid_probe_points(dev.h, self.h, jitter_seed is not None,
                                            0 if jitter_seed is None else int(jitter_seed),
                                            pts.ptr, cells.ptr, C.byref(m)))
        m = int(m.value)
        host_pts = pts.numpy(m * 3).reshape(m, 3)
        probed = dev.zeros(n, np.float64)
        dens_d = dev.empty(max(m, 1), np.float64)
        for t in ts:
            dens = np.asarray(density_fn(host_pts, t), dtype=np.float64)
            if len(dens) != m:
                raise RuntimeError("occupancy grid: density_fn returned wrong batch size")
            if m:
                dens_d.copy_from(dens)
            check(dev.lib.vmb_grid_accumulate(dev.h, self.h, dens_d.ptr, cells.ptr, m, probed.ptr))
        check(dev.lib.vmb_grid_apply(dev.h, self.h, probed.ptr, ema_decay))

    def cell_world_box(self, ix, iy, iz):
        """occupancy_grid.cpp:152-163 (AABB grids): world-space (lo, hi) of a cell."""
        res, con = self.resolution, self.contraction
        lo = np.array([ix / res, iy / res, iz / res], float)
        hi = np.array([(ix + 1) / res, (iy + 1) / res, (iz + 1) / res], float)
        w, valid = invert_grid_point(con, np.stack([lo, hi]), self.dev)
        return (w[0], w[1]) if valid.all() else None

    def seed_occupancy(self, occupied: Callable):
        """seed_occupancy: predicate over cell world boxes -> cache/bits (AABB only)."""
        con = self.contraction
        if con.kind != 0:
            raise ValueError("seed_occupancy: supported for AabbNormalize grids only")
        res = self.resolution
        idx = np.arange(res, dtype=np.float64)
        lo_g = idx / res
        hi_g = (idx + 1) / res
        mn, mx = np.array(con.box_min[:]), np.array(con.box_max[:])
        size = mx - mn
        mask = np.zeros(res ** 3, np.uint8)
        c = 0
        for iz in range(res):
            for iy in range(res):
                for ix in range(res):
                    lo = mn + np.array([lo_g[ix], lo_g[iy], lo_g[iz]]) * size
                    hi = mn + np.array([hi_g[ix], hi_g[iy], hi_g[iz]]) * size
                    mask[c] = bool(occupied((lo, hi)))
                    c += 1
        self.seed_mask(mask)

    def seed_mask(self, mask):
        m = self.dev.upload(np.ascontiguousarray(mask, dtype=np.uint8))
        check(self.dev.lib.vmb_grid_seed_mask(self.dev.h, self.h, m.ptr))

    def write(self, packed_bits=None, cache=None):
        b = None if packed_bits is None else np.ascontiguousarray(packed_bits, dtype=np.uint8)
        c = None if cache is None else _f64(cache)
        check(self.dev.lib.vmb_grid_write(self.dev.h, self.h, None if b is None else b.ctypes.data,
                                          None if c is None else c.ctypes.data))

    # -------------------------------------------------------------- OGRD I/O
    def save(self, path: str):
        """OGRD v1 (occupancy_grid.cpp:177-207); the bit section is the device layout."""
        res, con, thr, ref, _ = self._info()
        with open(path, "wb") as f:
            f.write(b"OGRD")
            f.write(np.uint32(1).tobytes())
            f.write(np.uint32(res).tobytes())
            f.write(np.uint8(con.kind).tobytes())
            if con.kind == 0:
                f.write(np.array(con.box_min[:] + con.box_max[:], np.float64).tobytes())
            else:
                f.write(np.array(con.center[:] + [con.radius], np.float64).tobytes())
            f.write(np.array([thr, ref], np.float64).tobytes())
            f.write(self.density_cache().astype(np.float32).tobytes())
            f.write(self.packed_bits().tobytes())

    @staticmethod
    def load(path: str, dev: Optional[Device] = None) -> "OccupancyGrid":
        """occupancy_grid.cpp:209-236: header, f32 cache, stored bits (not recomputed)."""
        data = open(path, "rb").read()
        if data[:4] != b"OGRD":
            raise RuntimeError("occupancy grid: bad magic")
        off = 4
        if np.frombuffer(data, np.uint32, 1, off)[0] != 1:
            raise RuntimeError("occupancy grid: unsupported version")
        res = int(np.frombuffer(data, np.uint32, 1, off + 4)[0])
        tag = data[off + 8]
        off += 9
        if tag == 0:
            v = np.frombuffer(data, np.float64, 6, off)
            con = Contraction.aabb(v[:3], v[3:])
            off += 48
        elif tag == 1:
            v = np.frombuffer(data, np.float64, 4, off)
            con = Contraction.sphere(v[:3], v[3])
            off += 32
        else:
            raise RuntimeError("occupancy grid: unknown contraction tag")
        thr, ref = np.frombuffer(data, np.float64, 2, off)
        off += 16
        n = res ** 3
        if len(data) < off + 4 * n + (n + 7) // 8:
            raise RuntimeError("occupancy grid: truncated stream")
        cache = np.frombuffer(data, np.float32, n, off).astype(np.float64)
        bits = np.frombuffer(data, np.uint8, (n + 7) // 8, off + 4 * n)
        g = OccupancyGrid(res, con, float(thr), float(ref), 0.0, dev)
        g.write(bits, cache)
        return g


# ---------------------------------------------------------------------- marching
def _rays_on_device(dev: Device, rays: RayBatch):
    do, dd = dev.upload(rays.origins if rays.n_rays else np.zeros((1, 3))), \
        dev.upload(rays.directions if rays.n_rays else np.zeros((1, 3)))
    r = Rays(do.ptr, dd.ptr, VMB_F64, 0, rays.n_rays, rays.near, rays.far)
    return r, (do, dd)


def _packed_call(dev: Device, fn, n_rays: int, guess: int) -> DevicePacked:
    out = DevicePacked.allocate(dev, n_rays, max(guess, 1))
    n = C.c_uint64()
    smp = out.samples_struct()
    rc = fn(smp, n)
    if rc == VMB_CAPACITY:
        out = DevicePacked.allocate(dev, n_rays, int(n.value))
        smp = out.samples_struct()
        rc = fn(smp, n)
    check(rc)
    out.n_samples = int(n.value)
    return out


def march(rays: RayBatch, grid: OccupancyGrid, sigma_fn, config: MarchConfig, n_threads: int = 1,
          stats: Optional[MarchStats] = None) -> PackedSamples:
    """ray_marching.hpp:40-42. ``sigma_fn`` is a device-evaluable :class:`Field` (fused
    kernel) or a host callable ``(t_starts, t_ends, ray_indices) -> sigmas`` invoked
    once per ray on that ray's grid-passing candidates, as the reference does."""
    dev = grid.dev
    r, keep = _rays_on_device(dev, rays)
    if isinstance(sigma_fn, Field):
        st = MarchStats()
        out = _packed_call(dev, lambda smp, n: dev.lib.vmb_march_field(
            dev.h, grid.h, C.byref(r), C.byref(sigma_fn), C.byref(config), C.byref(smp), C.byref(n),
            C.byref(st)), rays.n_rays, 32 * max(rays.n_rays, 1))
        if stats is not None:
            stats.samples_emitted, stats.samples_kept = st.samples_emitted, st.samples_kept
        return out.to_host()
    # generic path: device candidates -> host callback per ray -> device filter
    cand = _packed_call(dev, lambda smp, n: dev.lib.vmb_march_candidates(
        dev.h, grid.h, C.byref(r), C.byref(config), C.byref(smp), C.byref(n)),
        rays.n_rays, 64 * max(rays.n_rays, 1))
    hc = cand.to_host()
    sig = np.zeros(max(hc.n_samples, 1))
    for ray in range(hc.n_rays):
        b, c = int(hc.offsets[ray]), int(hc.counts[ray])
        if c == 0:
            continue
        vals = np.asarray(sigma_fn(hc.t_starts[b:b + c], hc.t_ends[b:b + c],
                                   np.full(c, ray, np.uint32)), dtype=np.float64)
        if len(vals) != c:
            # sigma errors of earlier rays take precedence (ray order); check them first
            _filter(dev, cand, sig, config, upto_ray=ray)
            raise RuntimeError(f"marching: sigma_fn returned {len(vals)} values for {c} samples")
        sig[b:b + c] = vals
    out = _filter(dev, cand, sig, config)
    if stats is not None:
        stats.samples_emitted, stats.samples_kept = hc.n_samples, out.n_samples
    return out.to_host()


def _filter(dev: Device, cand: DevicePacked, sig: np.ndarray, config: MarchConfig,
            upto_ray: Optional[int] = None) -> DevicePacked:
    n_rays = cand.n_rays if upto_ray is None else upto_ray
    ds = dev.upload(sig)
    v = PackedView(cand.offsets.ptr, cand.counts.ptr, n_rays, cand.t_starts.ptr, cand.t_ends.ptr,
                   cand.n_samples)
    return _packed_call(dev, lambda smp, n: dev.lib.vmb_march_filter(
        dev.h, C.byref(v), ds.ptr, C.byref(config), C.byref(smp), C.byref(n)), n_rays,
        max(cand.n_samples, 1))


def march_uniform(rays: RayBatch, config: MarchConfig, dev: Optional[Device] = None) -> PackedSamples:
    dev = dev or default_device()
    r, keep = _rays_on_device(dev, rays)
    guess = rays.n_rays * uniform_step_count(rays.near, rays.far, config.step_size)
    return _packed_call(dev, lambda smp, n: dev.lib.vmb_march_uniform(
        dev.h, C.byref(r), C.byref(config), C.byref(smp), C.byref(n)), rays.n_rays, guess).to_host()


# ---------------------------------------------------------------------- rendering
def _check_lengths(p: PackedSamples, rgbs, sigmas):
    if len(rgbs) != p.n_samples or len(sigmas) != p.n_samples:
        raise ValueError("rendering: attribute length mismatch")


def transmittance(p: PackedSamples, sigmas, dev: Optional[Device] = None) -> np.ndarray:
    if len(sigmas) != p.n_samples:
        raise ValueError("rendering: sigma length mismatch")
    dev = dev or default_device()
    d = p.to_device(dev)
    ds = dev.upload(_f64(sigmas) if p.n_samples else np.zeros(1))
    out = dev.zeros(max(p.n_samples, 1), np.float64)  # rendering.cpp:22: zero where no ray covers
    v = d.view()
    check(dev.lib.vmb_transmittance(dev.h, C.byref(v), ds.ptr, out.ptr, VMB_F64))
    return out.numpy(p.n_samples)


def render_forward(p: PackedSamples, rgbs, sigmas, n_threads: int = 1, dev: Optional[Device] = None,
                   dtype=np.float64):
    """rendering.cpp:35-65 -> (color[n,3], opacity[n], depth[n])."""
    _check_lengths(p, rgbs, sigmas)
    dev = dev or default_device()
    d = p.to_device(dev)
    n, s = p.n_rays, p.n_samples
    dr = dev.upload(np.asarray(rgbs, dtype).reshape(-1, 3) if s else np.zeros((1, 3), dtype))
    ds = dev.upload(np.asarray(sigmas, dtype) if s else np.zeros(1, dtype))
    col, op, dep = dev.empty(max(n, 1) * 3, dtype), dev.empty(max(n, 1), dtype), dev.empty(max(n, 1), dtype)
    v = d.view()
    check(dev.lib.vmb_render_forward(dev.h, C.byref(v), dr.ptr, ds.ptr, col.ptr, op.ptr, dep.ptr, _dt(dtype)))
    return col.numpy(n * 3).reshape(n, 3), op.numpy(n), dep.numpy(n)


def render_backward(p: PackedSamples, rgbs, sigmas, d_color, d_opacity, d_depth, n_threads: int = 1,
                    dev: Optional[Device] = None, dtype=np.float64):
    """rendering.cpp:67-112 -> (d_rgbs[s,3], d_sigmas[s])."""
    _check_lengths(p, rgbs, sigmas)
    n, s = p.n_rays, p.n_samples
    if len(d_color) != n or len(d_opacity) != n or len(d_depth) != n:
        raise ValueError("rendering: upstream gradient length mismatch")
    dev = dev or default_device()
    d = p.to_device(dev)
    up = lambda a, k=1: dev.upload(np.asarray(a, dtype).reshape(-1) if len(a) else np.zeros(k, dtype))  # noqa: E731
    dr, ds = up(rgbs, 3), up(sigmas)
    dc, do, dd = up(d_color, 3), up(d_opacity), up(d_depth)
    gr, gs = dev.zeros(max(s, 1) * 3, dtype), dev.zeros(max(s, 1), dtype)  # rendering.cpp:78-79
    v = d.view()
    check(dev.lib.vmb_render_backward(dev.h, C.byref(v), dr.ptr, ds.ptr, dc.ptr, do.ptr, dd.ptr,
                                      gr.ptr, gs.ptr, _dt(dtype)))
    return gr.numpy(s * 3).reshape(s, 3), gs.numpy(s)


def render_attribute(p: PackedSamples, sigmas, values, dim: int, dev: Optional[Device] = None):
    """rendering.cpp:114-134 -> out[n*dim]."""
    if len(sigmas) != p.n_samples:
        raise ValueError("rendering: sigma length mismatch")
    values = _f64(values).reshape(-1)
    if dim == 0 or len(values) != p.n_samples * dim:
        raise ValueError("rendering: value length mismatch")
    dev = dev or default_device()
    d = p.to_device(dev)
    ds = dev.upload(_f64(sigmas) if p.n_samples else np.zeros(1))
    dv = dev.upload(values if len(values) else np.zeros(1))
    out = dev.empty(max(p.n_rays * dim, 1), np.float64)
    v = d.view()
    check(dev.lib.vmb_render_attribute(dev.h, C.byref(v), ds.ptr, dv.ptr, dim, out.ptr, VMB_F64))
    return out.numpy(p.n_rays * dim)


# ---------------------------------------------------------------------- NerfAcc operators
# Host mirrors of nerfacc.volrend's standalone functions over packed samples
# (include/vmb200.h "NerfAcc operators"); arrays come back as numpy. Gradients
# take the upstream gradient of each output (None = 0) and return the input's.
def _opt_upload(dev, a, dtype, n):
    if a is None:
        return None
    a = np.asarray(a, dtype).reshape(-1)
    if len(a) != n:
        raise ValueError("rendering: upstream gradient length mismatch")
    return dev.upload(a if len(a) else np.zeros(1, dtype))


def _ptr(a):
    return a.ptr if a is not None else None


def _per_sample(dev, p: PackedSamples, x, dtype, what="sigma"):
    x = np.asarray(x, dtype).reshape(-1)
    if len(x) != p.n_samples:
        raise ValueError(f"rendering: {what} length mismatch")
    return dev.upload(x if len(x) else np.zeros(1, dtype))


def render_weight_from_density(p: PackedSamples, sigmas, dev: Optional[Device] = None, dtype=np.float64):
    """-> (weights, transmittance, alphas) per sample; rendering.cpp:47-58 per sample."""
    dev = dev or default_device()
    d, s = p.to_device(dev), p.n_samples
    ds = _per_sample(dev, p, sigmas, dtype)
    w, t, a = (dev.empty(max(s, 1), dtype) for _ in range(3))
    v = d.view()
    check(dev.lib.vmb_render_weight_from_density(dev.h, C.byref(v), ds.ptr, w.ptr, t.ptr, a.ptr, _dt(dtype)))
    return w.numpy(s), t.numpy(s), a.numpy(s)


def render_weight_from_density_backward(p: PackedSamples, sigmas, g_weights=None, g_trans=None, g_alphas=None,
                                        dev: Optional[Device] = None, dtype=np.float64):
    """-> dL/dsigmas."""
    dev = dev or default_device()
    d, s = p.to_device(dev), p.n_samples
    ds = _per_sample(dev, p, sigmas, dtype)
    gw, gt, ga = (_opt_upload(dev, g, dtype, s) for g in (g_weights, g_trans, g_alphas))
    out = dev.zeros(max(s, 1), dtype)
    v = d.view()
    check(dev.lib.vmb_render_weight_from_density_backward(dev.h, C.byref(v), ds.ptr, _ptr(gw), _ptr(gt), _ptr(ga),
                                                          out.ptr, _dt(dtype)))
    return out.numpy(s)


def render_weight_from_alpha(p: PackedSamples, alphas, dev: Optional[Device] = None, dtype=np.float64):
    """-> (weights, transmittance)."""
    dev = dev or default_device()
    d, s = p.to_device(dev), p.n_samples
    da = _per_sample(dev, p, alphas, dtype, "alpha")
    w, t = dev.empty(max(s, 1), dtype), dev.empty(max(s, 1), dtype)
    v = d.view()
    check(dev.lib.vmb_render_weight_from_alpha(dev.h, C.byref(v), da.ptr, w.ptr, t.ptr, _dt(dtype)))
    return w.numpy(s), t.numpy(s)


def render_weight_from_alpha_backward(p: PackedSamples, alphas, g_weights=None, g_trans=None,
                                      dev: Optional[Device] = None, dtype=np.float64):
    """-> dL/dalphas."""
    dev = dev or default_device()
    d, s = p.to_device(dev), p.n_samples
    da = _per_sample(dev, p, alphas, dtype, "alpha")
    gw, gt = (_opt_upload(dev, g, dtype, s) for g in (g_weights, g_trans))
    out = dev.zeros(max(s, 1), dtype)
    v = d.view()
    check(dev.lib.vmb_render_weight_from_alpha_backward(dev.h, C.byref(v), da.ptr, _ptr(gw), _ptr(gt), out.ptr,
                                                        _dt(dtype)))
    return out.numpy(s)


def render_transmittance_from_alpha(p: PackedSamples, alphas, dev: Optional[Device] = None, dtype=np.float64):
    """-> transmittance (exclusive product of 1 - alpha along each ray)."""
    dev = dev or default_device()
    d, s = p.to_device(dev), p.n_samples
    da = _per_sample(dev, p, alphas, dtype, "alpha")
    t = dev.empty(max(s, 1), dtype)
    v = d.view()
    check(dev.lib.vmb_render_transmittance_from_alpha(dev.h, C.byref(v), da.ptr, t.ptr, _dt(dtype)))
    return t.numpy(s)


def render_transmittance_from_alpha_backward(p: PackedSamples, alphas, g_trans, dev: Optional[Device] = None,
                                             dtype=np.float64):
    """-> dL/dalphas."""
    return render_weight_from_alpha_backward(p, alphas, None, g_trans, dev=dev, dtype=dtype)


def accumulate_along_rays(p: PackedSamples, weights, values=None, dim: int = 1, dev: Optional[Device] = None,
                          dtype=np.float64):
    """-> out[n_rays, dim] = per-ray sum of weights * values (values None: sum of weights)."""
    if dim == 0:
        raise ValueError("rendering: value length mismatch")
    dev = dev or default_device()
    d, s, n = p.to_device(dev), p.n_samples, p.n_rays
    dw = _per_sample(dev, p, weights, dtype, "weight")
    dv = None
    if values is not None:
        values = np.asarray(values, dtype).reshape(-1)
        if len(values) != s * dim:
            raise ValueError("rendering: value length mismatch")
        dv = dev.upload(values if len(values) else np.zeros(1, dtype))
    out = dev.empty(max(n * dim, 1), dtype)
    v = d.view()
    check(dev.lib.vmb_accumulate_along_rays(dev.h, C.byref(v), dw.ptr, _ptr(dv), dim, out.ptr, _dt(dtype)))
    return out.numpy(n * dim).reshape(n, dim)


def accumulate_along_rays_backward(p: PackedSamples, weights, values, dim: int, g_out,
                                   dev: Optional[Device] = None, dtype=np.float64):
    """-> (dL/dweights, dL/dvalues or None)."""
    dev = dev or default_device()
    d, s, n = p.to_device(dev), p.n_samples, p.n_rays
    dw = _per_sample(dev, p, weights, dtype, "weight")
    dv = None if values is None else dev.upload(np.asarray(values, dtype).reshape(-1) if s else np.zeros(1, dtype))
    g = dev.upload(np.asarray(g_out, dtype).reshape(-1) if n else np.zeros(1, dtype))
    gw = dev.zeros(max(s, 1), dtype)
    gv = dev.zeros(max(s * dim, 1), dtype) if values is not None else None
    v = d.view()
    check(dev.lib.vmb_accumulate_along_rays_backward(dev.h, C.byref(v), dw.ptr, _ptr(dv), dim, g.ptr, gw.ptr,
                                                     _ptr(gv), _dt(dtype)))
    return gw.numpy(s), (gv.numpy(s * dim).reshape(s, dim) if gv is not None else None)


def ray_aabb_intersect(origins, dirs, aabbs, near_plane=-np.inf, far_plane=np.inf, miss_value=np.inf,
                       dev: Optional[Device] = None):
    """-> (t_min, t_max, hit), each [n_rays, n_aabbs]; aabbs [n_aabbs, 6] = min xyz, max xyz."""
    dev = dev or default_device()
    o = np.ascontiguousarray(origins, np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
    b = np.ascontiguousarray(aabbs, np.float64).reshape(-1, 6)
    n, m = len(o), len(b)
    do_, dd_ = dev.upload(o if n else np.zeros((1, 3))), dev.upload(d if n else np.zeros((1, 3)))
    db = dev.upload(b if m else np.zeros((1, 6)))
    rays = Rays(do_.ptr, dd_.ptr, VMB_F64, 0, n, float(near_plane), float(far_plane))
    tmin, tmax = dev.empty(max(n * m, 1), np.float64), dev.empty(max(n * m, 1), np.float64)
    hit = dev.empty(max(n * m, 1), np.uint8)
    check(dev.lib.vmb_ray_aabb_intersect(dev.h, C.byref(rays), db.ptr, m, float(miss_value), tmin.ptr, tmax.ptr,
                                         hit.ptr))
    return (tmin.numpy(n * m).reshape(n, m), tmax.numpy(n * m).reshape(n, m),
            hit.numpy(n * m).reshape(n, m).astype(bool))


# ---------------------------------------------------------------------- multi-level grid
class Cascade:
    """NerfAcc's multi-level occupancy grid (vmb_march_ext): level 0
    is an AABB OccupancyGrid over `base`, level l its box scaled by 2^l about the
    center (vmb_cascade_level_box). Each level is a full OccupancyGrid (update /
    query / bits / OGRD) with the reference's semantics; a point is decided by the
    finest level containing it. levels=1 is a plain OccupancyGrid."""

    def __init__(self, resolution: int, base: Contraction, levels: int = 4, alpha_threshold: float = 1e-2,
                 reference_step: float = 0.0, initial_density: float = 0.0, dev: Optional[Device] = None):
        self.dev = dev or default_device()
        self.grids = []
        for level in range(levels):
            con = Contraction()
            check(self.dev.lib.vmb_cascade_level_box(C.byref(base), level, C.byref(con)))
            self.grids.append(OccupancyGrid(resolution, con, alpha_threshold, reference_step, initial_density,
                                            dev=self.dev))
        self._arr = (C.c_void_p * max(levels - 1, 1))(*[g.h.value for g in self.grids[1:]])

    @property
    def levels(self):
        return len(self.grids)

    def update_field(self, field: Field, decay: float, seed=None, timestamps=(0.0,)):
        for g in self.grids:
            g.update_field(field, decay, seed, timestamps)

    def ext(self, cone_angle: Optional[float] = None, max_step: float = 1e10) -> MarchExt:
        return MarchExt(C.cast(self._arr, C.c_void_p), len(self.grids) - 1, int(cone_angle is not None),
                        float(cone_angle or 0.0), float(max_step))

    def query(self, points) -> np.ndarray:
        x = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        dx = self.dev.upload(x if len(x) else np.zeros((1, 3)))
        out = self.dev.empty(max(len(x), 1), np.uint8)
        e = self.ext()
        check(self.dev.lib.vmb_cascade_query(self.dev.h, self.grids[0].h, C.byref(e), dx.ptr, len(x), out.ptr))
        return out.numpy(len(x)).astype(bool)


def march_cascade_device(dev: Device, cascade: Cascade, rays: Rays, field: Field, cfg: MarchConfig,
                         out: DevicePacked, cone_angle: Optional[float] = None, max_step: float = 1e10,
                         stats: Optional[MarchStats] = None) -> DevicePacked:
    """vmb_march_cascade into caller buffers; grows them once on VMB_CAPACITY."""
    e = cascade.ext(cone_angle, max_step)
    n = C.c_uint64()
    for attempt in range(2):
        smp = out.samples_struct()
        rc = dev.lib.vmb_march_cascade(dev.h, cascade.grids[0].h, C.byref(e), C.byref(rays), C.byref(field),
                                       C.byref(cfg), C.byref(smp), C.byref(n),
                                       C.byref(stats) if stats is not None else None)
        if rc != VMB_CAPACITY or attempt:
            break
        grown = DevicePacked.allocate(dev, out.n_rays, int(n.value * 1.25) + 1024)
        out.t_starts, out.t_ends, out.ray_indices = grown.t_starts, grown.t_ends, grown.ray_indices
    check(rc)
    out.n_samples = int(n.value)
    return out


def march_render_cascade_device(dev: Device, cascade: Cascade, rays: Rays, field: Field, cfg: MarchConfig,
                                out: DevicePacked, rgbs: DeviceArray, sigmas: DeviceArray, color: DeviceArray,
                                opacity: DeviceArray, depth: DeviceArray, cone_angle: Optional[float] = None,
                                max_step: float = 1e10, time: float = 0.0,
                                stats: Optional[MarchStats] = None) -> DevicePacked:
    """vmb_march_render_cascade: cascade march + analytic shading + render_forward."""
    e = cascade.ext(cone_angle, max_step)
    n = C.c_uint64()
    smp = out.samples_struct()
    check(dev.lib.vmb_march_render_cascade(dev.h, cascade.grids[0].h, C.byref(e), C.byref(rays), C.byref(field),
                                           C.byref(cfg), C.byref(smp), rgbs.ptr, sigmas.ptr, color.ptr, opacity.ptr,
                                           depth.ptr, _dt(rgbs.dtype), time, C.byref(n),
                                           C.byref(stats) if stats is not None else None))
    out.n_samples = int(n.value)
    return out
