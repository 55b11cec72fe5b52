"""Data-parallel training of a TrilinearVoxelField through the B200 path — the
reference CLI's `voxmarch train` (tools/voxmarch.cpp:385-562), SURVEY §8(f) rank 4.

One iteration (cmd_train:460-508), every array resident in HBM:

    minibatch gather (vmb_gather_rays, indices from the reference's Rng stream)
    -> march + voxel shading + render_forward fused (vmb_march_render_field)
    -> MSE-vs-white-background loss and upstream grads (vmb_loss_mse_background)
    -> render_backward -> voxel-field backward at the sample midpoints
       (vmb_voxel_field_backward_samples; deterministic sample-order folds)
    -> [N > 1: ncclAllReduce(sum) of the parameter gradients]
    -> Adam on density and colour (vmb_adam_step), exponential lr decay
    -> every grid_update_every iterations: occupancy update from the field.

With one rank the minibatches are the reference's (Rng(seed).uniform_below over the
ray pool), so a run follows the reference's training trajectory up to the ulp-level
differences of CUDA's exp/log1p. With N ranks each rank draws from Rng(seed + rank)
and the gradients are summed (weak scaling of the batch).

    python -m paper_2210_04847_b200.train --iterations 200 --batch-size 4096
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import time
from dataclasses import dataclass, field as dc_field
from typing import Optional

import numpy as np

from . import api, workload
from ._lib import (VMB_CAPACITY, VMB_F32, VMB_F64, VMB_GRAD_ATOMIC, VMB_GRAD_DETERMINISTIC, Contraction,
                   Field, MarchConfig, MarchStats, Rays, Samples, check)

MASK = (1 << 64) - 1


@dataclass
class TrainOptions:
    # TrainOptions (voxmarch.cpp:385-398)
    n_views: int = 20
    eval_views: int = 4
    iterations: int = 2000
    width: int = 64
    height: int = 64
    field_resolution: int = 32
    batch_size: int = 1024
    lr: float = 0.1
    lr_density: float = 8.0
    lr_final_fraction: float = 0.1
    grid_update_every: int = 16
    # CommonOptions used by train (voxmarch.cpp:39-75; alpha_thre defaults to 0 for train)
    seed: int = 0
    aabb: tuple = (0.0, 0.0, 0.0, 1.0, 1.0, 1.0)
    scene_center: Optional[tuple] = None
    scene_radius: float = 0.2
    scene_sigma: float = 200.0
    scene_rgb: tuple = (0.8, 0.25, 0.25)
    grid_resolution: int = 128
    ema_decay: float = 0.95
    grid_alpha_threshold: float = 1e-2
    near_plane: float = 0.2
    far_plane: float = 1.0
    early_stop_eps: float = 1e-4
    alpha_thre: float = 0.0
    step_size: float = 0.0  # 0: domain diagonal / 1024
    max_samples_per_ray: int = 2048
    grad_mode: int = VMB_GRAD_DETERMINISTIC
    out_checkpoint: str = ""


def _rng_block(state: int, n: int):
    """n consecutive splitmix64 outputs of a Rng in `state` (vectorised rng.hpp:10-15);
    returns (new_state, uint64[n])."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state) + k * np.uint64(workload.GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (state + n * workload.GOLDEN) & MASK, z


def uniform_below_batch(rng: workload.Rng, bound: int, n: int) -> np.ndarray:
    """n draws of Rng::uniform_below(bound) (rng.hpp:41-47), in order."""
    limit = MASK + 1 - ((MASK + 1) % bound)
    state, v = _rng_block(rng.state, n)
    if limit <= MASK and bool((v >= np.uint64(limit)).any()):  # a rejection: replay exactly
        return np.array([_uniform_below(rng, bound) for _ in range(n)], dtype=np.uint64)
    rng.state = state
    return v % np.uint64(bound)


def _uniform_below(rng, bound):
    limit = MASK + 1 - ((MASK + 1) % bound)
    v = rng.next_u64()
    while v >= limit:
        v = rng.next_u64()
    return v % bound


def uniform_batch(rng: workload.Rng, lo: float, hi: float, n: int) -> np.ndarray:
    """n draws of Rng::uniform(lo, hi) = lo + (hi - lo) * unit_double(next)."""
    state, v = _rng_block(rng.state, n)
    rng.state = state
    u = (v >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + (hi - lo) * u


class _Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.pg = dist

    def bcast_bytes(self, b: bytes) -> bytes:
        if not self.pg:
            return b
        obj = [b]
        self.pg.broadcast_object_list(obj, src=0)
        return obj[0]


class Trainer:
    def __init__(self, opts: TrainOptions, dev: Optional[api.Device] = None, rank: int = 0, world: int = 1):
        self.o = opts
        self.dev = dev or api.default_device()
        self.rank, self.world = rank, world
        L = self.dev.lib
        o = opts
        lo, hi = np.array(o.aabb[:3], float), np.array(o.aabb[3:], float)
        self.lo, self.hi = lo, hi
        center = tuple(o.scene_center) if o.scene_center else tuple((lo + hi) * 0.5)
        self.target = Field.sphere(center=center, radius=o.scene_radius, sigma=o.scene_sigma, rgb=o.scene_rgb)
        diag = float(np.sqrt(((hi - lo) ** 2).sum()))
        step = o.step_size if o.step_size > 0 else diag / 1024.0  # default_step_size
        self.cfg = MarchConfig(step, o.early_stop_eps, o.alpha_thre, o.max_samples_per_ray, 1.0)
        rng = workload.Rng(o.seed)
        # cameras (orbit_camera, voxmarch.cpp:278-286)
        self.train_cams = [self._orbit(2.0 * math.pi * v / o.n_views) for v in range(o.n_views)]
        self.eval_cams = [self._orbit(2.0 * math.pi * (v + 0.5) / max(1, o.eval_views))
                          for v in range(o.eval_views)]
        # ground truth and the flat (ray, colour) pool, all on the device
        self.gt_train = [self._render(c, self.target, None, uniform=True) for c in self.train_cams]
        self.gt_eval = [self._render(c, self.target, None, uniform=True) for c in self.eval_cams]
        n_pix = o.width * o.height
        self.pool = o.n_views * n_pix
        self.pool_o = self.dev.empty(3 * self.pool, np.float64)
        self.pool_d = self.dev.empty(3 * self.pool, np.float64)
        self.pool_c = self.dev.empty(3 * self.pool, np.float64)
        for v, cam in enumerate(self.train_cams):
            rays, ro, rd = api.generate_rays_device(self.dev, cam, o.near_plane, o.far_plane, np.float64)
            for dst, src in ((self.pool_o, ro), (self.pool_d, rd), (self.pool_c, self.gt_train[v])):
                check(L.vmb_memcpy_d2d(self.dev.h, dst.ptr + v * n_pix * 24, src.ptr, n_pix * 24))
        # model: near-zero random init from the same Rng stream as the reference
        self.field = api.VoxelField(o.field_resolution, lo, hi, self.dev)
        nv = self.field.n_vertices
        self.field.set_params(uniform_batch(rng, -1e-4, 1e-4, nv), uniform_batch(rng, -1e-4, 1e-4, 3 * nv))
        self.adam = {k: (self.dev.zeros(n, np.float64), self.dev.zeros(n, np.float64))
                     for k, n in (("density", nv), ("color", 3 * nv))}
        self.t = 0
        # occupancy grid: starts fully occupied at 4x the threshold density
        probe = api.OccupancyGrid(o.grid_resolution, Contraction.aabb(lo, hi), o.grid_alpha_threshold, dev=self.dev)
        self.grid = api.OccupancyGrid(o.grid_resolution, Contraction.aabb(lo, hi), o.grid_alpha_threshold, 0.0,
                                      4.0 * probe.threshold_density(), dev=self.dev)
        self.jitter_root = rng.next_u64()
        self.rng = rng if rank == 0 else workload.Rng(o.seed + rank)
        # per-iteration device buffers
        B = o.batch_size
        self.idx = self.dev.empty(B, np.uint32)
        self.bo, self.bd, self.bt = (self.dev.empty(3 * B, np.float64) for _ in range(3))
        self.color, self.opacity, self.depth = (self.dev.empty(3 * B, np.float64), self.dev.empty(B, np.float64),
                                                self.dev.empty(B, np.float64))
        self.dcol, self.dop, self.ddep = (self.dev.empty(3 * B, np.float64), self.dev.empty(B, np.float64),
                                          self.dev.empty(B, np.float64))
        self.grad_d, self.grad_c = self.field.zero_gradients()
        self._alloc_samples(B * 64)
        self.loss_curve, self.last_stats = [], MarchStats()

    # ------------------------------------------------------------------ helpers
    def _orbit(self, angle, elevation=0.4):
        o = self.o
        center = (self.lo + self.hi) * 0.5
        radius = 0.6 * float(np.sqrt(((self.hi - self.lo) ** 2).sum())) / math.sqrt(3.0)
        eye = center + np.array([radius * math.cos(angle) * math.cos(elevation),
                                 radius * math.sin(angle) * math.cos(elevation), radius * math.sin(elevation)])
        return api.look_at(eye, center, (0, 0, 1), 1.1 * o.width, o.width, o.height)

    def _alloc_samples(self, cap):
        d = self.dev
        B = self.o.batch_size
        self.packed = api.DevicePacked.allocate(d, B, cap)
        self.rgb, self.sig = d.empty(3 * cap, np.float64), d.empty(cap, np.float64)
        self.g_rgb, self.g_sig = d.empty(3 * cap, np.float64), d.empty(cap, np.float64)

    def _render(self, cam, fld: Field, grid, uniform: bool):
        """Image = color + (1 - opacity) (composite_to_image, voxmarch.cpp:253-260), f64 [n][3] on device."""
        d, L, o = self.dev, self.dev.lib, self.o
        rays, ro, rd = api.generate_rays_device(d, cam, o.near_plane, o.far_plane, np.float64)
        n = cam.width * cam.height
        if uniform:
            guess = n * api.uniform_step_count(o.near_plane, o.far_plane, self.cfg.step_size)
            packed = api._packed_call(d, lambda smp, k: L.vmb_march_uniform(d.h, C.byref(rays), C.byref(self.cfg),
                                                                              C.byref(smp), C.byref(k)), n, guess)
        else:
            packed = api.march_device(d, grid, rays, fld, self.cfg, api.DevicePacked.allocate(d, n, 64 * n))
        cap = packed.capacity
        rgb, sig = d.empty(3 * cap, np.float64), d.empty(cap, np.float64)
        api.shade_device(d, rays, fld, packed, rgb, sig)
        col, op, dep = d.empty(3 * n, np.float64), d.empty(n, np.float64), d.empty(n, np.float64)
        api.render_forward_device(d, packed, rgb, sig, col, op, dep)
        img = d.empty(3 * n, np.float64)
        h = col.numpy().reshape(n, 3) + (1.0 - op.numpy())[:, None]
        img.copy_from(h)
        return img

    # ------------------------------------------------------------------ one iteration
    def step(self, it: int) -> float:
        o, d, L = self.o, self.dev, self.dev.lib
        B = o.batch_size
        decay = o.lr_final_fraction ** ((it - 1) / max(1, o.iterations - 1))
        lr_density = (o.lr_density if o.lr_density > 0 else o.lr) * decay
        lr_color = o.lr * decay
        pick = uniform_below_batch(self.rng, self.pool, B).astype(np.uint32)
        self.idx.copy_from(pick)
        check(L.vmb_gather_rays(d.h, self.pool_o.ptr, self.pool_d.ptr, self.pool_c.ptr, self.idx.ptr, B, VMB_F64,
                                self.bo.ptr, self.bd.ptr, self.bt.ptr))
        rays = Rays(self.bo.ptr, self.bd.ptr, VMB_F64, 0, B, o.near_plane, o.far_plane)
        f = self.field.field
        while True:
            n = C.c_uint64()
            smp = self.packed.samples_struct()
            rc = L.vmb_march_render_field(d.h, self.grid.h, C.byref(rays), C.byref(f), C.byref(self.cfg),
                                          C.byref(smp), self.rgb.ptr, self.sig.ptr, self.color.ptr,
                                          self.opacity.ptr, self.depth.ptr, VMB_F64, 0.0, C.byref(n),
                                          C.byref(self.last_stats) if it == o.iterations else None)
            if rc == VMB_CAPACITY:
                self._alloc_samples(int(n.value * 1.25) + 1024)
                continue
            check(rc)
            break
        self.packed.n_samples = S = int(n.value)
        loss = C.c_double()
        check(L.vmb_loss_mse_background(d.h, self.color.ptr, self.opacity.ptr, self.bt.ptr, B, VMB_F64,
                                        self.dcol.ptr, self.dop.ptr, self.ddep.ptr, C.byref(loss)))
        api.render_backward_device(d, self.packed, self.rgb, self.sig, self.dcol, self.dop, self.ddep,
                                   self.g_rgb, self.g_sig)
        nv = self.field.n_vertices
        check(L.vmb_memset(d.h, self.grad_d.ptr, 0, nv * 8))
        check(L.vmb_memset(d.h, self.grad_c.ptr, 0, 3 * nv * 8))
        check(L.vmb_voxel_field_backward_samples(d.h, C.byref(f), C.byref(rays), self.packed.ray_indices.ptr,
                                                 self.packed.t_starts.ptr, self.packed.t_ends.ptr, S, 0.0,
                                                 self.g_rgb.ptr, self.g_sig.ptr, VMB_F64, self.grad_d.ptr,
                                                 self.grad_c.ptr, int(o.grad_mode)))
        if self.world > 1:
            check(L.vmb_comm_allreduce_sum_f64(d.h, self.grad_d.ptr, nv))
            check(L.vmb_comm_allreduce_sum_f64(d.h, self.grad_c.ptr, 3 * nv))
        self.t += 1
        for (m, v), p, g, n_, lr in ((self.adam["density"], self.field.d_density, self.grad_d, nv, lr_density),
                                     (self.adam["color"], self.field.d_color, self.grad_c, 3 * nv, lr_color)):
            check(L.vmb_adam_step(d.h, n_, p.ptr, g.ptr, m.ptr, v.ptr, lr, 0.9, 0.999, 1e-8, self.t))
        if it % o.grid_update_every == 0:
            self.grid.update_field(f, o.ema_decay, workload.mix_seed(self.jitter_root, it))
        self.loss_curve.append(loss.value)
        if not math.isfinite(loss.value):
            raise RuntimeError(f"train: loss diverged at iteration {it}")
        return loss.value

    def psnr(self, cam, gt, use_grid=True) -> float:
        img = self._render(cam, self.field.field, self.grid if use_grid else None, uniform=not use_grid)
        a, b = img.numpy(), gt.numpy()
        mse = float(((a - b) ** 2).sum()) / (3.0 * (len(a) // 3))
        return math.inf if mse <= 0 else 10.0 * math.log10(1.0 / mse)

    def report(self, wall_ms: float) -> dict:
        o = self.o
        pt = sum(self.psnr(c, g) for c, g in zip(self.train_cams, self.gt_train)) / max(1, o.n_views)
        pe = sum(self.psnr(c, g) for c, g in zip(self.eval_cams, self.gt_eval)) / max(1, o.eval_views)
        pn = sum(self.psnr(c, g, False) for c, g in zip(self.eval_cams, self.gt_eval)) / max(1, o.eval_views)
        if o.out_checkpoint:
            self.field.save(o.out_checkpoint)
        return {"schema": 1, "command": "train", "seed": o.seed, "iterations": o.iterations,
                "n_views": o.n_views, "eval_views": o.eval_views, "field_resolution": o.field_resolution,
                "batch_size": o.batch_size, "lr": o.lr, "loss_curve": self.loss_curve,
                "final_loss": self.loss_curve[-1] if self.loss_curve else 0.0, "psnr_train": pt,
                "psnr_eval": pe, "psnr_eval_nogrid": pn, "occupied_fraction": self.grid.occupied_fraction(),
                "samples_emitted": int(self.last_stats.samples_emitted),
                "samples_after_filter": int(self.last_stats.samples_kept),
                "checkpoint": o.out_checkpoint, "wall_time_ms": wall_ms, "world_size": self.world}


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    d = TrainOptions()
    for name in ("n_views", "eval_views", "iterations", "width", "height", "field_resolution", "batch_size",
                 "grid_update_every", "seed", "grid_resolution", "max_samples_per_ray", "grad_mode"):
        ap.add_argument("--" + name.replace("_", "-"), type=int, default=getattr(d, name))
    for name in ("lr", "lr_density", "lr_final_fraction", "scene_radius", "scene_sigma", "ema_decay",
                 "grid_alpha_threshold", "near_plane", "far_plane", "early_stop_eps", "alpha_thre", "step_size"):
        ap.add_argument("--" + name.replace("_", "-"), type=float, default=getattr(d, name))
    ap.add_argument("--out-checkpoint", default="")
    a = ap.parse_args(argv)
    opts = TrainOptions(**{k: v for k, v in vars(a).items()})
    dist = _Dist()
    dev = api.Device(dist.local)
    if dist.world > 1:
        uid = (C.c_char * 128)()
        if dist.rank == 0:
            check(dev.lib.vmb_comm_unique_id(uid))
        uid = (C.c_char * 128).from_buffer_copy(dist.bcast_bytes(bytes(uid)))
        check(dev.lib.vmb_comm_init(dev.h, uid, dist.world, dist.rank))
    tr = Trainer(opts, dev, dist.rank, dist.world)
    t0 = time.perf_counter()
    for it in range(1, opts.iterations + 1):
        tr.step(it)
    dev.sync()
    wall = 1e3 * (time.perf_counter() - t0)
    rep = tr.report(wall)
    if dist.rank == 0:
        print(json.dumps(rep, indent=2))
    if dist.world > 1:
        dev.lib.vmb_comm_destroy(dev.h)
    return rep


if __name__ == "__main__":
    main()
