"""CPU oracle loader (TEST INFRASTRUCTURE ONLY).

Wraps the two C libraries that implement ``oracle/vm_oracle.h``:

* ``Oracle("ref")``  -> ``oracle/_ref/libvoxmarch_ref.so``: the reference's own
  sources (``/root/reference/proj/src``) compiled in place by ``oracle/Makefile``;
* ``Oracle("port")`` -> ``oracle/_build/libvm_oracle.so``: ``oracle/vm_oracle.c``,
  the plain-C restatement (pinned against "ref" by tests/test_oracle_port.py).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libvoxmarch_ref.so"),
    "port": os.path.join(HERE, "_build", "libvm_oracle.so"),
}
PREFIX = {"ref": "vmr_", "port": "vmo_"}

VMB_OK, VMB_INVALID_ARGUMENT, VMB_RUNTIME = 0, 1, 2
VALIDATE_NAMES = [None, "length mismatch", "offset mismatch", "non-positive interval",
                  "non-monotone t_starts", "overlapping intervals", "partition mismatch"]


class Contraction(C.Structure):
    """vmb_contraction (include/vmb200_types.h) <- voxmarch::Contraction."""
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("box_min", C.c_double * 3),
                ("box_max", C.c_double * 3), ("center", C.c_double * 3), ("radius", C.c_double)]

    @staticmethod
    def aabb(lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0)):
        c = Contraction()
        c.kind = 0
        c.box_min[:] = list(lo)
        c.box_max[:] = list(hi)
        return c

    @staticmethod
    def sphere(center, radius):
        c = Contraction()
        c.kind = 1
        c.center[:] = list(center)
        c.radius = float(radius)
        return c


class Field(C.Structure):
    """vmb_field (include/vmb200_types.h) <- voxmarch::AnalyticField (+ velocity)."""
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("box_min", C.c_double * 3),
                ("box_max", C.c_double * 3), ("center", C.c_double * 3), ("radius", C.c_double),
                ("sigma", C.c_double), ("rgb", C.c_double * 3), ("rgb_b", C.c_double * 3),
                ("period", C.c_double), ("velocity", C.c_double * 3),
                ("vox_density", C.c_void_p), ("vox_color", C.c_void_p), ("vox_resolution", C.c_uint32),
                ("pad2_", C.c_uint32)]

    @staticmethod
    def sphere(center=(0.5, 0.5, 0.5), radius=0.2, sigma=200.0, rgb=(0.8, 0.25, 0.25),
               velocity=(0.0, 0.0, 0.0)):
        f = Field()
        f.kind = 1
        f.center[:] = list(center)
        f.radius = radius
        f.sigma = sigma
        f.rgb[:] = list(rgb)
        f.velocity[:] = list(velocity)
        return f

    @staticmethod
    def box(lo, hi, sigma=1.0, rgb=(1.0, 1.0, 1.0), velocity=(0.0, 0.0, 0.0)):
        f = Field()
        f.kind = 0
        f.box_min[:] = list(lo)
        f.box_max[:] = list(hi)
        f.sigma = sigma
        f.rgb[:] = list(rgb)
        f.velocity[:] = list(velocity)
        return f

    @staticmethod
    def checker(period=0.125, sigma=1.0, rgb_a=(1.0, 1.0, 1.0), rgb_b=(0.0, 0.0, 0.0)):
        f = Field()
        f.kind = 2
        f.period = period
        f.sigma = sigma
        f.rgb[:] = list(rgb_a)
        f.rgb_b[:] = list(rgb_b)
        return f

    @staticmethod
    def voxel(resolution, box_min, box_max, density, color, velocity=(0.0, 0.0, 0.0)):
        """TrilinearVoxelField over host arrays (kept alive on the Field object)."""
        f = Field()
        f.kind = 3
        f.box_min[:] = list(box_min)
        f.box_max[:] = list(box_max)
        f.vox_resolution = int(resolution)
        f._dens = np.ascontiguousarray(density, dtype=np.float64).ravel()
        f._col = np.ascontiguousarray(color, dtype=np.float64).ravel()
        f.vox_density = f._dens.ctypes.data
        f.vox_color = f._col.ctypes.data
        f.velocity[:] = list(velocity)
        return f


class MarchConfig(C.Structure):
    """vmb_march_config <- voxmarch::MarchingConfig (ray_marching.hpp:11-17 defaults)."""
    _fields_ = [("step_size", C.c_double), ("early_stop_eps", C.c_double),
                ("alpha_thre", C.c_double), ("max_samples_per_ray", C.c_uint32),
                ("pad_", C.c_uint32), ("unbounded_step_growth", C.c_double)]

    def __init__(self, step_size=1.6914558667664816e-3, early_stop_eps=1e-4, alpha_thre=1e-2,
                 max_samples_per_ray=2048, unbounded_step_growth=1.0):
        super().__init__(step_size, early_stop_eps, alpha_thre, max_samples_per_ray, 0,
                         unbounded_step_growth)


class Camera(C.Structure):
    """vmb_camera <- voxmarch::PinholeCamera (scene_camera.hpp:12-19)."""
    _fields_ = [("rotation", C.c_double * 9), ("position", C.c_double * 3), ("focal", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class _Packed(C.Structure):
    _fields_ = [("n_rays", C.c_uint64), ("n_samples", C.c_uint64),
                ("offsets", C.POINTER(C.c_uint32)), ("counts", C.POINTER(C.c_uint32)),
                ("t_starts", C.POINTER(C.c_double)), ("t_ends", C.POINTER(C.c_double)),
                ("ray_indices", C.POINTER(C.c_uint32)), ("samples_emitted", C.c_uint64),
                ("samples_kept", C.c_uint64)]


@dataclass
class Packed:
    offsets: np.ndarray
    counts: np.ndarray
    t_starts: np.ndarray
    t_ends: np.ndarray
    ray_indices: np.ndarray
    samples_emitted: int = 0
    samples_kept: int = 0

    @property
    def n_rays(self):
        return len(self.counts)

    @property
    def n_samples(self):
        return len(self.t_starts)


class OracleError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
        self.msg = msg


DENSITY_CB = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.POINTER(C.c_double), C.c_uint64, C.c_double,
                         C.POINTER(C.c_double))
SIGMA_CB = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                       C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_double))


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


class Oracle:
    def __init__(self, kind: str = "ref"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.kind = kind
        self.lib = C.CDLL(path)
        pre = PREFIX[kind]
        self._f = lambda name: getattr(self.lib, pre + name)
        self._f("last_error").restype = C.c_char_p
        self._f("uniform_step_count").restype = C.c_uint64
        self._f("uniform_step_count").argtypes = [C.c_double] * 3
        self._f("packed_free").argtypes = [C.c_void_p]
        self._f("grid_destroy").argtypes = [C.c_void_p]
        for name in ("march_field", "march_callback", "march_uniform", "grid_create",
                     "grid_update_field", "grid_update_callback", "grid_seed_mask", "grid_get",
                     "grid_info", "grid_query", "grid_save", "grid_load", "pack", "validate",
                     "contract", "invert_grid_point", "shade", "transmittance", "render_forward",
                     "render_backward", "render_attribute", "train_step", "camera_look_at",
                     "generate_rays", "field_query", "voxel_field_backward"):
            self._f(name).restype = C.c_int

    # ------------------------------------------------------------ helpers
    def _check(self, rc):
        if rc != VMB_OK:
            raise OracleError(rc, self._f("last_error")().decode())

    def _take_packed(self, pp):
        p = pp.contents
        n, s = p.n_rays, p.n_samples
        out = Packed(
            offsets=np.ctypeslib.as_array(p.offsets, (max(n, 1),))[:n].copy(),
            counts=np.ctypeslib.as_array(p.counts, (max(n, 1),))[:n].copy(),
            t_starts=np.ctypeslib.as_array(p.t_starts, (max(s, 1),))[:s].copy(),
            t_ends=np.ctypeslib.as_array(p.t_ends, (max(s, 1),))[:s].copy(),
            ray_indices=np.ctypeslib.as_array(p.ray_indices, (max(s, 1),))[:s].copy(),
            samples_emitted=int(p.samples_emitted), samples_kept=int(p.samples_kept))
        self._f("packed_free")(pp)
        return out

    # ------------------------------------------------------------ core types
    def uniform_step_count(self, near, far, step):
        return int(self._f("uniform_step_count")(near, far, step))

    def pack(self, counts):
        counts = _u32(counts)
        n = len(counts)
        offsets = np.zeros(max(n, 1), np.uint32)
        total = C.c_uint64(0)
        cap = int(counts.astype(np.uint64).sum())
        idx = np.zeros(max(min(cap, 1 << 31), 1), np.uint32) if cap <= (1 << 31) else None
        rc = self._f("pack")(_p(counts, C.c_uint32), C.c_uint64(n), _p(offsets, C.c_uint32),
                             _p(idx, C.c_uint32), C.c_uint64(cap if idx is not None else 0),
                             C.byref(total))
        self._check(rc)
        return offsets[:n], (idx[:total.value] if idx is not None else None)

    def validate(self, offsets, counts, t_starts, t_ends, ray_indices):
        arrs = [_u32(offsets), _u32(counts), _f64(t_starts), _f64(t_ends), _u32(ray_indices)]
        cts = [C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint32]
        args = []
        for a, ct in zip(arrs, cts):
            args += [_p(a, ct), C.c_uint64(len(a))]
        return VALIDATE_NAMES[self._f("validate")(*args)]

    def contract(self, con, x):
        x = _f64(x, (-1, 3))
        out = np.zeros_like(x)
        self._check(self._f("contract")(C.byref(con), _p(x, C.c_double), C.c_uint64(len(x)),
                                        _p(out, C.c_double)))
        return out

    def invert_grid_point(self, con, g):
        g = _f64(g, (-1, 3))
        out = np.zeros_like(g)
        valid = np.zeros(len(g), np.uint8)
        self._check(self._f("invert_grid_point")(C.byref(con), _p(g, C.c_double),
                                                 C.c_uint64(len(g)), _p(out, C.c_double),
                                                 _p(valid, C.c_uint8)))
        return out, valid.astype(bool)

    # ------------------------------------------------------------ grid
    def grid(self, resolution, con, alpha_threshold=1e-2, reference_step=0.0,
             initial_density=0.0):
        return OracleGrid(self, resolution, con, alpha_threshold, reference_step,
                          initial_density)

    def grid_load(self, path):
        h = C.c_void_p()
        self._check(self._f("grid_load")(path.encode(), C.byref(h)))
        g = OracleGrid.__new__(OracleGrid)
        g.o, g.h = self, h
        return g

    # ------------------------------------------------------------ marching
    def march_field(self, origins, dirs, near, far, grid, field, cfg, n_threads=1):
        o, d = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3))
        pp = C.POINTER(_Packed)()
        self._check(self._f("march_field")(_p(o, C.c_double), _p(d, C.c_double),
                                           C.c_uint64(len(o)), C.c_double(near),
                                           C.c_double(far), grid.h, C.byref(field),
                                           C.byref(cfg), C.c_int(n_threads), C.byref(pp)))
        return self._take_packed(pp)

    def march_cascade(self, origins, dirs, near, far, grid, levels, field, cfg, cone_angle=None, max_step=1e10):
        """port only: vmo_march_cascade (levels = OracleGrids above `grid`, finest first)"""
        assert self.kind == "port"
        o, d = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3))
        arr = (C.c_void_p * max(len(levels), 1))(*[g.h.value for g in levels])
        pp = C.POINTER(_Packed)()
        f = self.lib.vmo_march_cascade
        f.restype = C.c_int
        self._check(f(_p(o, C.c_double), _p(d, C.c_double), C.c_uint64(len(o)), C.c_double(near), C.c_double(far),
                      grid.h, arr, C.c_uint32(len(levels)), C.c_int(cone_angle is not None),
                      C.c_double(cone_angle or 0.0), C.c_double(max_step), C.byref(field), C.byref(cfg),
                      C.byref(pp)))
        return self._take_packed(pp)

    def cascade_query(self, grid, levels, points):
        assert self.kind == "port"
        x = _f64(points, (-1, 3))
        out = np.zeros(len(x), np.uint8)
        arr = (C.c_void_p * max(len(levels), 1))(*[g.h.value for g in levels])
        f = self.lib.vmo_cascade_query
        f.restype = C.c_int
        self._check(f(grid.h, arr, C.c_uint32(len(levels)), _p(x, C.c_double), C.c_uint64(len(x)),
                      _p(out, C.c_uint8)))
        return out.astype(bool)

    def march_callback(self, origins, dirs, near, far, grid, sigma_fn, cfg, n_threads=1):
        """sigma_fn(ts, te, idx) -> array of sigmas (any length; mismatch is an error)."""
        o, d = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3))

        def cb(_user, ts, te, idx, n, out):
            a = np.ctypeslib.as_array(ts, (n,)) if n else np.zeros(0)
            b = np.ctypeslib.as_array(te, (n,)) if n else np.zeros(0)
            c = np.ctypeslib.as_array(idx, (n,)) if n else np.zeros(0, np.uint32)
            vals = np.asarray(sigma_fn(a.copy(), b.copy(), c.copy()), dtype=np.float64)
            m = min(len(vals), n + 16)
            for i in range(m):
                out[i] = float(vals[i])
            return len(vals)

        cbf = SIGMA_CB(cb)
        pp = C.POINTER(_Packed)()
        self._check(self._f("march_callback")(_p(o, C.c_double), _p(d, C.c_double),
                                              C.c_uint64(len(o)), C.c_double(near),
                                              C.c_double(far), grid.h, cbf, None, C.byref(cfg),
                                              C.c_int(n_threads), C.byref(pp)))
        return self._take_packed(pp)

    def march_uniform(self, origins, dirs, near, far, cfg):
        o, d = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3))
        pp = C.POINTER(_Packed)()
        self._check(self._f("march_uniform")(_p(o, C.c_double), _p(d, C.c_double),
                                             C.c_uint64(len(o)), C.c_double(near),
                                             C.c_double(far), C.byref(cfg), C.byref(pp)))
        return self._take_packed(pp)

    def shade(self, origins, dirs, packed, field):
        o, d = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3))
        s = packed.n_samples
        rgbs = np.zeros((s, 3))
        sig = np.zeros(s)
        self._check(self._f("shade")(_p(o, C.c_double), _p(d, C.c_double),
                                     _p(_u32(packed.ray_indices), C.c_uint32),
                                     _p(_f64(packed.t_starts), C.c_double),
                                     _p(_f64(packed.t_ends), C.c_double), C.c_uint64(s),
                                     C.byref(field), _p(rgbs, C.c_double), _p(sig, C.c_double)))
        return rgbs, sig

    # ------------------------------------------------------------ cameras
    def look_at(self, eye, target, up, focal, width, height) -> Camera:
        cam = Camera()
        self._check(self._f("camera_look_at")(_p(_f64(eye), C.c_double), _p(_f64(target), C.c_double),
                                              _p(_f64(up), C.c_double), C.c_double(focal),
                                              C.c_int32(width), C.c_int32(height), C.byref(cam)))
        return cam

    def generate_rays(self, cam: Camera, near_, far_):
        n = max(cam.width, 0) * max(cam.height, 0)
        o, d = np.zeros((n, 3)), np.zeros((n, 3))
        self._check(self._f("generate_rays")(C.byref(cam), C.c_double(near_), C.c_double(far_),
                                             _p(o, C.c_double), _p(d, C.c_double)))
        return o, d

    # ------------------------------------------------------------ fields
    def field_query(self, field, points, time=0.0, rgb=True):
        p = _f64(points, (-1, 3))
        n = len(p)
        sig = np.zeros(n)
        col = np.zeros((n, 3)) if rgb else None
        self._check(self._f("field_query")(C.byref(field), _p(p, C.c_double), C.c_uint64(n), C.c_double(time),
                                           _p(sig, C.c_double), _p(col, C.c_double)))
        return (sig, col) if rgb else sig

    def voxel_field_backward(self, field, points, d_rgbs, d_sigmas, accum_density=None, accum_color=None):
        """TrilinearVoxelField::backward; returns the accumulated (d_density, d_color)."""
        p = _f64(points, (-1, 3))
        n = len(p)
        nv = int(field.vox_resolution) ** 3
        acc_d = np.zeros(nv) if accum_density is None else _f64(accum_density).copy()
        acc_c = np.zeros(3 * nv) if accum_color is None else _f64(accum_color).copy().ravel()
        self._check(self._f("voxel_field_backward")(C.byref(field), _p(p, C.c_double), C.c_uint64(n),
                                                    _p(_f64(d_rgbs, (-1, 3)), C.c_double),
                                                    _p(_f64(d_sigmas), C.c_double), _p(acc_d, C.c_double),
                                                    _p(acc_c, C.c_double)))
        return acc_d, acc_c

    # ------------------------------------------------------------ rendering
    def _pk(self, packed):
        off, cnt = _u32(packed.offsets), _u32(packed.counts)
        ts, te = _f64(packed.t_starts), _f64(packed.t_ends)
        self._keep = (off, cnt, ts, te)
        return [_p(off, C.c_uint32), _p(cnt, C.c_uint32), C.c_uint64(len(cnt)),
                _p(ts, C.c_double), _p(te, C.c_double), C.c_uint64(len(ts))]

    def transmittance(self, packed, sigmas):
        sig = _f64(sigmas)
        out = np.zeros(packed.n_samples)
        self._check(self._f("transmittance")(*self._pk(packed), _p(sig, C.c_double),
                                             _p(out, C.c_double)))
        return out

    def render_forward(self, packed, rgbs, sigmas, n_threads=1):
        rgb, sig = _f64(rgbs, (-1, 3)), _f64(sigmas)
        n = packed.n_rays
        color, op, dep = np.zeros((n, 3)), np.zeros(n), np.zeros(n)
        self._check(self._f("render_forward")(*self._pk(packed), _p(rgb, C.c_double),
                                              _p(sig, C.c_double), C.c_int(n_threads),
                                              _p(color, C.c_double), _p(op, C.c_double),
                                              _p(dep, C.c_double)))
        return color, op, dep

    def render_backward(self, packed, rgbs, sigmas, d_color, d_opacity, d_depth, n_threads=1):
        rgb, sig = _f64(rgbs, (-1, 3)), _f64(sigmas)
        dc, do, dd = _f64(d_color, (-1, 3)), _f64(d_opacity), _f64(d_depth)
        s = packed.n_samples
        d_rgb, d_sig = np.zeros((s, 3)), np.zeros(s)
        self._check(self._f("render_backward")(*self._pk(packed), _p(rgb, C.c_double),
                                               _p(sig, C.c_double), _p(dc, C.c_double),
                                               _p(do, C.c_double), _p(dd, C.c_double),
                                               C.c_int(n_threads), _p(d_rgb, C.c_double),
                                               _p(d_sig, C.c_double)))
        return d_rgb, d_sig

    def render_attribute(self, packed, sigmas, values, dim):
        sig, val = _f64(sigmas), _f64(values).ravel()
        out = np.zeros(packed.n_rays * dim)
        self._check(self._f("render_attribute")(*self._pk(packed), _p(sig, C.c_double),
                                                _p(val, C.c_double), C.c_uint64(len(val)),
                                                C.c_uint64(dim), _p(out, C.c_double)))
        return out

    def train_step(self, origins, dirs, near, far, grid, field, cfg, d_color, d_opacity,
                   d_depth, n_threads=1):
        o, d = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3))
        dc, do, dd = _f64(d_color, (-1, 3)), _f64(d_opacity), _f64(d_depth)
        phase = np.zeros(4)
        ns = C.c_uint64(0)
        cs = C.c_double(0)
        self._check(self._f("train_step")(_p(o, C.c_double), _p(d, C.c_double),
                                          C.c_uint64(len(o)), C.c_double(near), C.c_double(far),
                                          grid.h, C.byref(field), C.byref(cfg),
                                          _p(dc, C.c_double), _p(do, C.c_double),
                                          _p(dd, C.c_double), C.c_int(n_threads),
                                          _p(phase, C.c_double), C.byref(ns), C.byref(cs)))
        return phase, int(ns.value), float(cs.value)


class OracleGrid:
    def __init__(self, o, resolution, con, thr, ref_step, init):
        self.o = o
        self.h = C.c_void_p()
        o._check(o._f("grid_create")(C.c_uint32(resolution), C.byref(con), C.c_double(thr),
                                     C.c_double(ref_step), C.c_double(init), C.byref(self.h)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.o._f("grid_destroy")(h)
            self.h = None

    def info(self):
        res = C.c_uint32()
        thr, ref, thd, frac = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        self.o._f("grid_info")(self.h, C.byref(res), C.byref(thr), C.byref(ref), C.byref(thd),
                               C.byref(frac))
        return dict(resolution=res.value, alpha_threshold=thr.value, reference_step=ref.value,
                    threshold_density=thd.value, occupied_fraction=frac.value)

    @property
    def resolution(self):
        return self.info()["resolution"]

    def bits(self):
        n = self.resolution ** 3
        b = np.zeros(n, np.uint8)
        self.o._f("grid_get")(self.h, _p(b, C.c_uint8), None)
        return b

    def cache(self):
        n = self.resolution ** 3
        c = np.zeros(n)
        self.o._f("grid_get")(self.h, None, _p(c, C.c_double))
        return c

    def update_field(self, field, decay, seed=None, timestamps=(0.0,)):
        ts = _f64(timestamps)
        self.o._check(self.o._f("grid_update_field")(
            self.h, C.byref(field), _p(ts, C.c_double), C.c_uint64(len(ts)), C.c_double(decay),
            C.c_int(seed is not None), C.c_uint64(0 if seed is None else int(seed))))

    def update_callback(self, fn, decay, seed=None, timestamps=(0.0,)):
        """fn(points[n,3], t) -> densities (length mismatch reproduces the reference error)."""
        ts = _f64(timestamps)

        def cb(_user, pts, n, t, out):
            p = np.ctypeslib.as_array(pts, (n * 3,)).reshape(n, 3).copy() if n else np.zeros((0, 3))
            vals = np.asarray(fn(p, t), dtype=np.float64)
            m = min(len(vals), n + 16)
            if m:
                np.ctypeslib.as_array(out, (m,))[:] = vals[:m]
            return len(vals)

        cbf = DENSITY_CB(cb)
        self.o._check(self.o._f("grid_update_callback")(
            self.h, cbf, None, _p(ts, C.c_double), C.c_uint64(len(ts)), C.c_double(decay),
            C.c_int(seed is not None), C.c_uint64(0 if seed is None else int(seed))))

    def probe_range(self, field, c0, c1, seed=None, timestamps=(0.0,)):
        """Port only: probes of cells [c0, c1) (0 elsewhere) — one rank's share."""
        ts = _f64(timestamps)
        out = np.zeros(self.resolution ** 3)
        self.o._check(self.o.lib.vmo_grid_probe_range(
            self.h, C.byref(field), _p(ts, C.c_double), C.c_uint64(len(ts)),
            C.c_int(seed is not None), C.c_uint64(0 if seed is None else int(seed)),
            C.c_uint64(c0), C.c_uint64(c1), _p(out, C.c_double)))
        return out

    def apply(self, probed, decay):
        """Port only: cache = max(cache*decay, probed); refresh bits."""
        p = _f64(probed)
        self.o._check(self.o.lib.vmo_grid_apply(self.h, _p(p, C.c_double), C.c_double(decay)))

    def seed_mask(self, mask):
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        self.o._check(self.o._f("grid_seed_mask")(self.h, _p(m, C.c_uint8)))

    def query(self, points):
        p = _f64(points, (-1, 3))
        out = np.zeros(len(p), np.uint8)
        self.o._check(self.o._f("grid_query")(self.h, _p(p, C.c_double), C.c_uint64(len(p)),
                                              _p(out, C.c_uint8)))
        return out.astype(bool)

    def save(self, path):
        self.o._check(self.o._f("grid_save")(self.h, path.encode()))


class NerfaccOracle:
    """The port's sequential restatement of NerfAcc's standalone operators
    (vm_oracle.h: vmo_weight_from_density ... vmo_ray_aabb_intersect). The
    reference has no such functions; tests pin these against its render_forward /
    render_backward / transmittance by decomposition and by finite differences."""

    def __init__(self):
        self.lib = C.CDLL(LIBS["port"])
        for name in ("weight_from_density", "weight_from_density_backward", "weight_from_alpha",
                     "weight_from_alpha_backward", "accumulate_along_rays",
                     "accumulate_along_rays_backward", "ray_aabb_intersect"):
            getattr(self.lib, "vmo_" + name).restype = C.c_int

    def _pk(self, packed):
        off, cnt = _u32(packed.offsets), _u32(packed.counts)
        self._keep = (off, cnt)
        return [_p(off, C.c_uint32), _p(cnt, C.c_uint32), C.c_uint64(len(cnt))]

    @staticmethod
    def _opt(a, shape=None):
        return None if a is None else _f64(a, shape)

    def weight_from_density(self, packed, sigmas):
        s = packed.n_samples
        ts, te, sig = _f64(packed.t_starts), _f64(packed.t_ends), _f64(sigmas)
        w, t, a = np.zeros(s), np.zeros(s), np.zeros(s)
        assert self.lib.vmo_weight_from_density(*self._pk(packed), _p(ts, C.c_double), _p(te, C.c_double),
                                                _p(sig, C.c_double), _p(w, C.c_double), _p(t, C.c_double),
                                                _p(a, C.c_double)) == 0
        return w, t, a

    def weight_from_density_backward(self, packed, sigmas, g_weights, g_trans=None, g_alphas=None):
        s = packed.n_samples
        ts, te, sig = _f64(packed.t_starts), _f64(packed.t_ends), _f64(sigmas)
        gw, gt, ga = self._opt(g_weights), self._opt(g_trans), self._opt(g_alphas)
        out = np.zeros(s)
        assert self.lib.vmo_weight_from_density_backward(
            *self._pk(packed), _p(ts, C.c_double), _p(te, C.c_double), _p(sig, C.c_double), _p(gw, C.c_double),
            _p(gt, C.c_double), _p(ga, C.c_double), _p(out, C.c_double)) == 0
        return out

    def weight_from_alpha(self, packed, alphas):
        s = packed.n_samples
        al = _f64(alphas)
        w, t = np.zeros(s), np.zeros(s)
        assert self.lib.vmo_weight_from_alpha(*self._pk(packed), _p(al, C.c_double), _p(w, C.c_double),
                                              _p(t, C.c_double)) == 0
        return w, t

    def weight_from_alpha_backward(self, packed, alphas, g_weights=None, g_trans=None):
        al, gw, gt = _f64(alphas), self._opt(g_weights), self._opt(g_trans)
        out = np.zeros(packed.n_samples)
        assert self.lib.vmo_weight_from_alpha_backward(*self._pk(packed), _p(al, C.c_double), _p(gw, C.c_double),
                                                       _p(gt, C.c_double), _p(out, C.c_double)) == 0
        return out

    def accumulate_along_rays(self, packed, weights, values=None, dim=1):
        w, v = _f64(weights), self._opt(values)
        out = np.zeros(packed.n_rays * dim)
        assert self.lib.vmo_accumulate_along_rays(*self._pk(packed), _p(w, C.c_double), _p(v, C.c_double),
                                                  C.c_uint64(dim), _p(out, C.c_double)) == 0
        return out.reshape(packed.n_rays, dim)

    def accumulate_along_rays_backward(self, packed, weights, values, dim, g_out):
        w, v, g = _f64(weights), self._opt(values), _f64(g_out)
        s = packed.n_samples
        gw, gv = np.zeros(s), np.zeros(s * dim)
        assert self.lib.vmo_accumulate_along_rays_backward(
            *self._pk(packed), _p(w, C.c_double), _p(v, C.c_double), C.c_uint64(dim), _p(g, C.c_double),
            _p(gw, C.c_double), _p(gv, C.c_double)) == 0
        return gw, gv.reshape(s, dim)

    def ray_aabb_intersect(self, origins, dirs, aabbs, near=-np.inf, far=np.inf, miss=np.inf):
        o, d, b = _f64(origins, (-1, 3)), _f64(dirs, (-1, 3)), _f64(aabbs, (-1, 6))
        n, m = len(o), len(b)
        tmin, tmax, hit = np.zeros(n * m), np.zeros(n * m), np.zeros(n * m, np.uint8)
        assert self.lib.vmo_ray_aabb_intersect(_p(o, C.c_double), _p(d, C.c_double), C.c_uint64(n),
                                               _p(b, C.c_double), C.c_uint64(m), C.c_double(near), C.c_double(far),
                                               C.c_double(miss), _p(tmin, C.c_double), _p(tmax, C.c_double),
                                               _p(hit, C.c_uint8)) == 0
        return tmin.reshape(n, m), tmax.reshape(n, m), hit.reshape(n, m).astype(bool)
