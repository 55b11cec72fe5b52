#!/usr/bin/env python
"""Benchmark of the B200 hot path: march + render forward + render backward.

One STEP = one training-step pass of the path over one batch of synthetic rays
(BASELINE.json config 5: 2^22 rays of the reference CLI's bench camera, 128^3
occupancy grid warmed by 16 jittered updates, SolidSphere r=0.2 sigma=200,
step 5e-3, alpha_thre 1e-2, early_stop_eps 1e-4):

    march (fused traversal + density + alpha floor + T cut + packing)
    -> shade (analytic field rgb/sigma at each sample; harness)
    -> render_forward -> render_backward (upstream grads U(-1,1))

The timed resident step (fusion=forward) runs the batch as `--chunks` contiguous
ray sub-batches served by `--streams` contexts (default 2 x 2): the same C-ABI
calls per sub-batch, overlapping on the device; its outputs are checked equal,
bit for bit, to the single-call step's. `--streams 1 --chunks 1` times the single
call sequence.

Multi-GPU (torchrun): each rank marches its own 2^22-ray batch (weak scaling, its
own camera angle) against a replicated grid; rank 0 prints one JSON line with the
max-over-ranks device time. The grid warm-up runs the sharded probe +
ncclAllReduce(max) path. `--impl reference` times the reference's own CPU code
(oracle/_ref) on a bounded sample on the host cores.
"""
import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2210_04847_b200.pipeline import ResidentPipeline  # noqa: E402

BASELINE_METRIC = "rays/sec & samples/sec (march+render fwd+bwd) at 1/2/4/8 B200; % HBM roofline"
SCENE = dict(center=(0.5, 0.5, 0.5), radius=0.2, sigma=200.0, rgb=(0.8, 0.25, 0.25))
# march = k_zero_words + k_march_walk + k_scan_onepass + k_march_expand + k_march_fixup; then k_shade,
# k_forward (not launched when fused), k_zero_words + k_backward_hy + k_backward_long
KERNELS_PER_STEP = 10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--width", type=int, default=2048, help="rays per side (2048 -> 2^22 rays)")
    ap.add_argument("--resolution", type=int, default=128)
    ap.add_argument("--step-size", type=float, default=5e-3)
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--config2", type=int, default=1,
                    help="N=1: also time BASELINE config 2 (2^18 rays, step sqrt(3)/1024) in a sub-run "
                         "and report it under `config2`")
    ap.add_argument("--config3", type=int, default=1,
                    help="N=1: also time BASELINE config 3 (4-level cascaded grid, cone stepping, 2^20 rays) "
                         "in a sub-run and report it under `config3`")
    ap.add_argument("--workload", default="config5", choices=["config5", "config3", "config1"],
                    help="config3: the multi-level grid + cone-step workload alone; config1: the 4096-ray "
                         "batch as a CUDA graph (one JSON line each)")
    ap.add_argument("--res256", type=int, default=1,
                    help="N=1: also time config 5 over a 256^3 grid in a sub-run -> `grid256`")
    ap.add_argument("--config4", type=int, default=1,
                    help="N=1: also time BASELINE config 4 (2^20 rays, grid update every 16 steps) -> `config4`")
    ap.add_argument("--config1", type=int, default=1,
                    help="N=1: also time BASELINE config 1 (4096 rays, CUDA graph) in a sub-run -> `config1`")
    ap.add_argument("--field", default="sphere", choices=["sphere", "checker", "voxel"],
                    help="density field of the config 5 step: the SolidSphere scene (default), a Checker "
                         "(per-sample colour, dense everywhere) or a 128^3 TrilinearVoxelField holding the "
                         "sphere (stored density: trilinear + softplus/sigmoid per sample)")
    ap.add_argument("--fields", type=int, default=1,
                    help="N=1, sphere: also time the checker and voxel fields in sub-runs -> `fields`")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank marches its own 2^22-ray batch (its own camera angle); strong: the "
                         "ranks split ONE 2^22-ray batch by vmb_shard_range (BASELINE config 5's sweep)")
    ap.add_argument("--cpu-sample-rays", type=int, default=1 << 20)
    ap.add_argument("--ref-sample-rays", type=int, default=1 << 18)
    ap.add_argument("--phases", type=int, default=1, help="per-phase event timing pass")
    ap.add_argument("--fusion", default="forward", choices=["forward", "shade", "none"],
                    help="forward: march+shade+render_forward fused; shade: march+shade fused; none: separate")
    ap.add_argument("--grid-update-every", type=int, default=0,
                    help="config 4: an occupancy-grid EMA update (sharded probe + NCCL all-reduce(max) when N > 1) "
                         "inside the timed loop every K steps (0: none)")
    ap.add_argument("--streams", type=int, default=2,
                    help="resident step: sub-batches served round-robin by this many contexts (streams)")
    ap.add_argument("--chunks", type=int, default=2,
                    help="resident step: the batch is marched as this many sub-batches (2x2 measured best, r1)")
    ap.add_argument("--e2e-streams", type=int, default=2)
    ap.add_argument("--e2e-chunks", type=int, default=8)  # 2x8 best in the r2 sweep (profiles/r2/ab/e2e_*)
    ap.add_argument("--e2e-async", type=int, default=1, help="async march (no per-chunk host sync)")
    # device-generated rays leave PCIe to the gradients: more, smaller chunks pay (4x8 best on B200, r1)
    ap.add_argument("--e2e-camera-streams", type=int, default=4)
    ap.add_argument("--e2e-camera-chunks", type=int, default=8)
    return ap.parse_args()


# ---------------------------------------------------------------------- plumbing
class Dist:
    """torch.distributed (gloo) used only as host plumbing: id exchange, barrier, max."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo")
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, v: float) -> float:
        if not self.dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.dist:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def bcast_bytes(self, b: bytes) -> bytes:
        if not self.dist:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]


class Clocks:
    """nvidia-smi sampler (every 200 ms) around the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.rows = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].lower().startswith("active")})
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


PHASE_KERNELS = {"march": ["k_march_walk", "k_scan_onepass", "k_march_expand", "k_march_fixup"],
                 "shade": ["k_shade"], "render_forward": ["k_forward"],
                 "render_backward": ["k_backward_hy", "k_backward_long"]}


def traffic_of(phase):
    """DRAM bytes (read + write) per launch of a phase's kernels, from the committed
    ncu --set full summary of the same workload (profiles/ncu_traffic.json), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return sum(t["kernels"][k] for k in PHASE_KERNELS[phase] if k in t["kernels"]) or None
    except Exception:
        return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------- CPU legs
def reference_grid(orc, res):
    from oracle import oracle as O
    from paper_2210_04847_b200 import workload
    g = orc.grid(res, O.Contraction.aabb())
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(O.Field.sphere(**SCENE), 0.95, s)
    return g


def cpu_step(orc, grid, o, d, step_size, threads, seed=113):
    from oracle import oracle as O
    from paper_2210_04847_b200 import workload
    dc, do, dd = workload.upstream_grads(len(o), seed)
    cfg = O.MarchConfig(step_size, 1e-4, 1e-2)
    t0 = time.perf_counter()
    phase, ns, _ = orc.train_step(o, d, 0.2, 1.0, grid, O.Field.sphere(**SCENE), cfg, dc, do, dd, threads)
    return time.perf_counter() - t0, ns, phase


def cpu_baseline(args, o, d):
    """Reference CPU path (oracle/_ref, else the C port) on a strided sample of the batch."""
    from oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    threads = (os.cpu_count() or 1) if kind == "reference" else 1
    grid = reference_grid(orc, args.resolution)
    stride = max(1, len(o) // args.cpu_sample_rays)
    so, sd = o[::stride], d[::stride]
    times = []
    for _ in range(3):
        dt, ns, _ = cpu_step(orc, grid, so, sd, args.step_size, threads)
        times.append(dt)
    dt = statistics.median(times)
    return {"value": len(so) / dt, "unit": "rays/s", "cores": threads, "kind": kind,
            "samples_per_s": ns / dt,
            "sample": f"every {stride}th ray of the {len(o)}-ray batch ({len(so)} rays), median of 3 "
                      f"train steps (march+shade+fwd+bwd), {threads} threads, {cpu_model()}"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation, rank 0 only."""
    dist = Dist()
    if dist.rank != 0:
        return
    from oracle import Oracle, available
    from paper_2210_04847_b200 import workload
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "port")
    threads = (os.cpu_count() or 1) if kind == "reference" else 1
    o, d = workload.orbit_rays(args.width)
    grid = reference_grid(orc, args.resolution)
    n_sample = min(args.ref_sample_rays, len(o))
    stride = max(1, len(o) // n_sample)
    for i in range(args.warmup):
        cpu_step(orc, grid, o[i % stride::stride], d[i % stride::stride], args.step_size, threads)
    tot_t, tot_rays, tot_s = 0.0, 0, 0
    for i in range(args.steps):
        k = (args.warmup + i) % stride
        dt, ns, _ = cpu_step(orc, grid, o[k::stride], d[k::stride], args.step_size, threads)
        tot_t += dt
        tot_rays += len(o[k::stride])
        tot_s += ns
    v = tot_rays / tot_t
    line = {"impl": "reference", "metric": BASELINE_METRIC, "value": v, "unit": "rays/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "samples_per_s": tot_s / tot_t,
            "config": {"workload": f"config 5 sample: {n_sample} of {len(o)} orbit-camera rays per step, "
                                   f"{args.resolution}^3 grid, step {args.step_size}",
                       "global_batch": n_sample, "parallelism": "cpu threads"},
            "cpu_baseline": {"value": v, "unit": "rays/s", "cores": threads, "kind": kind,
                             "sample": f"every {stride}th ray per step, {threads} threads, {cpu_model()}"},
            "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- e2e
def e2e_pipeline(args, dist, api, dev, grid, field, cfg, o32, d32, ups, cap, dev_out, total_rays, cam=None,
                 pixel0=0):
    """The same step through the C ABI from HOST memory: every step copies its rays and
    upstream gradients host->device and reads the rendered color/opacity/depth back.

    The batch is cut into `--e2e-chunks` ray chunks served round-robin by
    `--e2e-streams` contexts (one CUDA stream each, one host thread each; the ctypes
    calls release the GIL), so one chunk's PCIe copies overlap another chunk's
    kernels. Timed with CUDA events on context 0, which waits for every other
    context at the end (vmb_ctx_wait); the others wait for its start event.

    With `cam` (a vmb_camera) the rays are not copied: each chunk generates its own
    pixels' rays on the device (vmb_generate_rays_range, scene_camera.cpp:46-63), so
    only the upstream gradients cross PCIe."""
    import ctypes as C
    from paper_2210_04847_b200._lib import VMB_F32, Rays, check
    L = dev.lib
    N = len(o32)
    n_ctx, n_chunk = max(1, args.e2e_streams), max(1, args.e2e_chunks)
    if cam is not None:
        n_ctx, n_chunk = max(1, args.e2e_camera_streams), max(1, args.e2e_camera_chunks)
    bounds = [(N * i // n_chunk, N * (i + 1) // n_chunk) for i in range(n_chunk)]
    cmax = max(e - b for b, e in bounds)
    host_in = [o32, d32] + list(ups)            # per-ray: 12, 12, 12, 4, 4 bytes
    widths = [3, 3, 3, 1, 1]
    first_in = 2 if cam is not None else 0      # camera mode: rays made on the device
    # The host keeps each chunk's inputs as one block [origins | directions | d_color |
    # d_opacity | d_depth] (camera mode: the three gradients only) and receives its
    # outputs as one block [color | opacity | depth]: one H2D and one D2H copy per
    # chunk instead of five and three (the layout of the user's buffers; filled before
    # the timed region).
    in_w, out_w = widths[first_in:], [3, 1, 1]
    win, wout = sum(in_w), sum(out_w)           # floats per ray
    p_in, p_out = C.c_void_p(), C.c_void_p()
    check(L.vmb_host_alloc(N * win * 4, C.byref(p_in)))
    check(L.vmb_host_alloc(N * wout * 4, C.byref(p_out)))
    h_in = np.ctypeslib.as_array((C.c_float * (N * win)).from_address(p_in.value))
    for b, e in bounds:
        at = b * win
        for arr, w in zip(host_in[first_in:], in_w):
            h_in[at:at + (e - b) * w] = arr.reshape(-1)[b * w:e * w]
            at += (e - b) * w
    ctxs = [dev] + [api.Device(dist.local) for _ in range(n_ctx - 1)]
    ccap = cap  # the full batch's capacity bounds any chunk's sample count
    bufs = []
    for cx in ctxs:
        d_in = cx.empty(cmax * win, np.float32)
        d_out = cx.empty(cmax * wout, np.float32)
        bufs.append(dict(d_in=d_in, d_out=d_out, o=cx.empty(cmax * 3, np.float32), d=cx.empty(cmax * 3, np.float32),
                         packed=api.DevicePacked.allocate(cx, cmax, ccap),
                         n_dev=cx.zeros(n_chunk, np.uint64),
                         rgb=cx.empty(ccap * 3, np.float32), sig=cx.empty(ccap, np.float32),
                         grgb=cx.empty(ccap * 3, np.float32), gsig=cx.empty(ccap, np.float32)))

    class Ptr:  # a device pointer with the DeviceArray interface the api needs
        def __init__(self, ptr):
            self.ptr = ptr

    def run_chunk(ci, b, e):
        cx, bf = ctxs[ci], bufs[ci]
        n = e - b
        check(L.vmb_memcpy_h2d(cx.h, bf["d_in"].ptr, p_in.value + b * win * 4, n * win * 4))
        views, at = [], bf["d_in"].ptr
        for w in in_w:  # the block's arrays on the device
            views.append(Ptr(at))
            at += n * w * 4
        if cam is None:
            o_ptr, d_ptr, ups_dev = views[0].ptr, views[1].ptr, views[2:]
        else:
            o_ptr, d_ptr, ups_dev = bf["o"].ptr, bf["d"].ptr, views
        outs, at = [], bf["d_out"].ptr
        for w in out_w:
            outs.append(Ptr(at))
            at += n * w * 4
        rays = Rays(o_ptr, d_ptr, VMB_F32, 0, n, 0.2, 1.0)
        if cam is not None:
            check(L.vmb_generate_rays_range(cx.h, C.byref(cam), 0.2, 1.0, VMB_F32, pixel0 + b, n, o_ptr, d_ptr,
                                            C.byref(rays)))
        pk = bf["packed"]
        if args.e2e_async:  # no host round trip: the sample total stays on the device
            smp = pk.samples_struct()
            check(L.vmb_march_render_field_async(cx.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                                 C.byref(smp), bf["rgb"].ptr, bf["sig"].ptr, outs[0].ptr,
                                                 outs[1].ptr, outs[2].ptr, VMB_F32, 0.0,
                                                 bf["n_dev"].ptr + 8 * chunk_id[0]))
            pk.n_samples = pk.capacity
        else:
            api.march_render_device(cx, grid, rays, field, cfg, pk, bf["rgb"], bf["sig"], *outs)
        api.render_backward_device(cx, pk, bf["rgb"], bf["sig"], *ups_dev, bf["grgb"], bf["gsig"])
        d2h = L.vmb_memcpy_d2h_async if args.e2e_async else L.vmb_memcpy_d2h  # async: synced at the end
        check(d2h(cx.h, p_out.value + b * wout * 4, bf["d_out"].ptr, n * wout * 4))

    def worker(ci, steps, err):
        try:
            for _ in range(steps):
                for k in range(ci, n_chunk, n_ctx):
                    run_chunk(ci, *bounds[k])
        except Exception as ex:  # pragma: no cover
            err.append(ex)

    chunk_id = [0]

    def run(steps):
        if args.e2e_async:  # one host thread enqueues everything; the streams overlap
            for _ in range(steps):
                for k in range(n_chunk):
                    chunk_id[0] = k
                    run_chunk(k % n_ctx, *bounds[k])
            return
        err = []
        ts = [threading.Thread(target=worker, args=(i, steps, err)) for i in range(n_ctx)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if err:
            raise err[0]

    run(2)  # warm-up (also grows each context's packed buffers to the chunk's need)
    for cx in ctxs:
        cx.sync()
    dist.barrier()
    dev.record(7)
    for cx in ctxs[1:]:
        check(L.vmb_ctx_wait(cx.h, dev.h, 9))
    run(args.steps)
    for i, cx in enumerate(ctxs[1:]):
        check(L.vmb_ctx_wait(dev.h, cx.h, 9 + (i % 8)))
    dev.record(8)
    for cx in ctxs:
        cx.sync()
    e2e_ms = dist.max(dev.elapsed_ms(7, 8) / args.steps)
    if args.e2e_async:  # deferred error report + every chunk's samples fitted the buffers
        for cx, bf in zip(ctxs, bufs):
            check(L.vmb_march_check(cx.h))
            assert int(bf["n_dev"].numpy().max()) <= ccap, "e2e chunk exceeded its sample capacity"
    # the pipelined result must equal the resident single-stream step's
    same = True
    h_out = np.ctypeslib.as_array((C.c_float * (N * wout)).from_address(p_out.value)).copy()
    got = [[], [], []]
    for b, e in bounds:
        at = b * wout
        for j, w in enumerate(out_w):
            got[j].append(h_out[at:at + (e - b) * w])
            at += (e - b) * w
    for parts, w, darr in zip(got, out_w, dev_out):
        same &= bool(np.array_equal(np.concatenate(parts), darr.numpy(N * w)))
    for p in (p_in, p_out):
        L.vmb_host_free(p)
    for cx in ctxs[1:]:
        cx.sync()
    if cam is not None:
        return {"value": total_rays / (e2e_ms * 1e-3), "unit": "rays/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": int(sum(a.nbytes for a in host_in[2:])), "d2h_bytes_per_step": N * 20,
                "streams": n_ctx, "chunks": n_chunk, "matches_resident_outputs": same,
                "path": f"C ABI: camera in, rays generated per chunk on the device (vmb_generate_rays_range), "
                        f"vmb_march_render_field{'_async' if args.e2e_async else ''} + vmb_render_backward, "
                        "pinned host upstream grads in, color/opacity/depth out"}
    return {"value": total_rays / (e2e_ms * 1e-3), "unit": "rays/s", "ms_per_step": e2e_ms,
            "h2d_bytes_per_step": int(sum(a.nbytes for a in host_in)), "d2h_bytes_per_step": N * 20,
            "streams": n_ctx, "chunks": n_chunk, "matches_resident_outputs": same,
            "path": f"C ABI (vmb_memcpy_h2d, vmb_march_render_field{'_async' if args.e2e_async else ''}, "
                    "vmb_render_backward, vmb_memcpy_d2h): "
                    "pinned host rays + upstream grads in, color/opacity/depth out, "
                    f"{n_chunk} chunks pipelined over {n_ctx} streams"}



# ---------------------------------------------------------------------- config 1
def run_config1(args):
    """BASELINE config 1: the reference CLI's bench batch, 4096 orbit-camera rays
    (W=64), 128^3 grid, step 5e-3 — launch-bound. The step (async march + shading +
    forward, then backward: ~10 kernel/memset nodes) is captured once as a CUDA
    graph (vmb_graph_begin/end) and replayed; the same step launched call by call
    is timed beside it."""
    from paper_2210_04847_b200 import api, workload
    from paper_2210_04847_b200._lib import VMB_F32, Contraction, Field, MarchConfig, Rays, check
    dev = api.Device(0)
    L = dev.lib
    field = Field.sphere(**SCENE)
    cfg = MarchConfig(5e-3, 1e-4, 1e-2)
    R, W = 128, 64
    grid = api.OccupancyGrid(R, Contraction.aabb(), dev=dev)
    for s in workload.grid_warmup_seeds(16, 5):
        grid.update_field(field, 0.95, s)
    o64, d64 = workload.orbit_rays(W)
    N = len(o64)
    o32, d32 = o64.astype(np.float32), d64.astype(np.float32)
    dc, do, dd = (x.astype(np.float32) for x in workload.upstream_grads(N, 113))
    do_, dd_ = dev.upload(o32), dev.upload(d32)
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.2, 1.0)
    packed = api.march_device(dev, grid, rays, field, cfg, api.DevicePacked.allocate(dev, N, 16 * N))
    S = packed.n_samples
    cap = packed.capacity
    rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    gr, gs = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
    ups = [dev.upload(x) for x in (dc, do, dd)]
    n_dev = dev.zeros(1, np.uint64)
    smp = packed.samples_struct()
    packed.n_samples = cap  # the backward reads the exact ranges from offsets/counts

    def step():
        check(L.vmb_march_render_field_async(dev.h, grid.h, C.byref(rays), C.byref(field), C.byref(cfg),
                                             C.byref(smp), rgb.ptr, sig.ptr, outs[0].ptr, outs[1].ptr, outs[2].ptr,
                                             VMB_F32, 0.0, n_dev.ptr))
        api.render_backward_device(dev, packed, rgb, sig, *ups, gr, gs)

    def timed(fn, k):
        dev.sync()
        dev.record(0)
        for _ in range(k):
            fn()
        dev.record(1)
        dev.sync()
        return dev.elapsed_ms(0, 1) / k

    for _ in range(max(args.warmup, 3)):
        step()
    dev.sync()
    check(L.vmb_march_check(dev.h))
    assert int(n_dev.numpy()[0]) == S
    graph = C.c_void_p()
    check(L.vmb_graph_begin(dev.h))
    step()
    check(L.vmb_graph_end(dev.h, C.byref(graph)))
    launch = lambda: check(L.vmb_graph_launch(dev.h, graph))  # noqa: E731
    steps = max(args.steps, 200)
    clocks = Clocks(0)
    for _ in range(max(args.warmup, 3)):
        launch()
    ms_graph = timed(launch, steps)
    ms_calls = timed(step, steps)
    t_end = time.time() + 1.0
    while time.time() < t_end:
        for _ in range(50):
            launch()
        dev.sync()
    clk = clocks.stop()
    check(L.vmb_march_check(dev.h))
    assert int(n_dev.numpy()[0]) == S
    check(L.vmb_graph_destroy(graph))
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    step_bytes = 80 * N + 84 * S + R ** 3 / 8
    line = {"metric": BASELINE_METRIC, "value": N / (ms_graph * 1e-3), "unit": "rays/s", "n_gpus": 1,
            "steps": steps, "warmup": args.warmup, "ms_per_step": ms_graph, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "samples_per_s": S / (ms_graph * 1e-3), "samples": S,
            "calls_ms_per_step": ms_calls, "graph": "one CUDA graph per step (vmb_graph_begin/end/launch)",
            "config": {"workload": f"config 1: {N} orbit-camera rays (W={W}), {R}^3 grid, SolidSphere r=0.2 "
                                   "sigma=200, step 5e-3 (launch-bound)",
                       "l2": "working set ~1 MB (L2-resident; the batch is launch-bound, not HBM-bound)"},
            "roofline": {"bound": "hbm", "kernel": "step", "algorithmic_bytes": step_bytes,
                         "achieved": step_bytes / (ms_graph * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": step_bytes / (ms_graph * 1e-3) / 1e9 / peak, "traffic": None},
            "clocks": clk}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- config 3
def run_config3(args):
    """BASELINE config 3 (Mip-NeRF-360-shaped, unbounded): a 4-level cascaded
    occupancy grid (128^3 per level, level l = the unit box scaled by 2^l about its
    center, up to [-3.5, 4.5]^3) and NerfAcc cone stepping (cone_angle 1/256), 2^20
    rays of the orbit camera from inside level 1 (near 0.01, far 100), SolidSphere
    r=0.3 sigma=40: central rays end in the sphere (T cut), the others cross every
    level until they leave the outermost box. Step = vmb_march_render_cascade (walk
    count -> scan -> fill, shading + forward) -> vmb_render_backward."""
    from paper_2210_04847_b200 import api, workload
    from paper_2210_04847_b200._lib import VMB_F32, Contraction, Field, MarchConfig, MarchStats, Rays, check
    dev = api.Device(0)
    L = dev.lib
    field = Field.sphere(radius=0.3, sigma=40.0)
    cfg = MarchConfig(math.sqrt(3.0) / 1024, 1e-4, 1e-2, 4096, 1.0)
    cone = 1.0 / 256
    R, levels, W = 128, 4, 1024
    cas = api.Cascade(R, Contraction.aabb((0, 0, 0), (1, 1, 1)), levels, dev=dev)
    dev.record(10)
    for s in workload.grid_warmup_seeds(16, 5):
        cas.update_field(field, 0.95, s)
    dev.record(11)
    upd_ms = dev.elapsed_ms(10, 11) / 16
    o64, d64 = workload.orbit_rays(W, near=0.01, far=100.0)
    N = len(o64)
    o32, d32 = o64.astype(np.float32), d64.astype(np.float32)
    dc, do, dd = (x.astype(np.float32) for x in workload.upstream_grads(N, 31))
    do_, dd_ = dev.upload(o32), dev.upload(d32)
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.01, 100.0)
    st = MarchStats()
    packed = api.march_cascade_device(dev, cas, rays, field, cfg, api.DevicePacked.allocate(dev, N, 64 * N), cone,
                                      1e10, st)
    S, cap = packed.n_samples, packed.capacity
    rgb, sig = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    gr, gs = dev.empty(3 * cap, np.float32), dev.empty(cap, np.float32)
    outs = [dev.empty(3 * N, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)]
    ups = [dev.upload(x) for x in (dc, do, dd)]

    def step():
        api.march_render_cascade_device(dev, cas, rays, field, cfg, packed, rgb, sig, *outs, cone_angle=cone)
        api.render_backward_device(dev, packed, rgb, sig, *ups, gr, gs)

    clocks = Clocks(0)
    for _ in range(max(args.warmup, 3)):
        step()
    dev.sync()
    dev.record(0)
    for _ in range(args.steps):
        step()
    dev.record(1)
    dev.sync()
    ms = dev.elapsed_ms(0, 1) / args.steps
    t_end = time.time() + 1.0
    while time.time() < t_end:
        step()
    dev.sync()
    clk = clocks.stop()
    assert packed.n_samples == S
    # e2e through the C ABI: pinned host rays + upstream grads in, outputs out
    host = [o32, d32, dc, do, dd]
    pins = []
    for a in host:
        pp = C.c_void_p()
        check(L.vmb_host_alloc(a.nbytes, C.byref(pp)))
        C.memmove(pp.value, a.ctypes.data, a.nbytes)
        pins.append(pp)
    outp = []
    for w in (3, 1, 1):
        pp = C.c_void_p()
        check(L.vmb_host_alloc(4 * w * N, C.byref(pp)))
        outp.append(pp)
    dst = [do_, dd_] + ups

    def e2e_step():
        for pp, a, dv in zip(pins, host, dst):
            check(L.vmb_memcpy_h2d(dev.h, dv.ptr, pp.value, a.nbytes))
        step()
        for pp, o, w in zip(outp, outs, (3, 1, 1)):
            check(L.vmb_memcpy_d2h(dev.h, pp.value, o.ptr, 4 * w * N))

    e2e_step()
    dev.sync()
    dev.record(2)
    for _ in range(args.steps):
        e2e_step()
    dev.record(3)
    dev.sync()
    e2e_ms = dev.elapsed_ms(2, 3) / args.steps
    for pp in pins + outp:
        L.vmb_host_free(pp)
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    # fused march + shade + forward, then backward: 80 N + 84 S + the levels' bits
    step_bytes = 80 * N + 84 * S + levels * R ** 3 / 8
    line = {"metric": BASELINE_METRIC, "value": N / (ms * 1e-3), "unit": "rays/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "samples_per_s": S / (ms * 1e-3), "samples": S, "samples_emitted": st.samples_emitted,
            "grid_update_ms": upd_ms,
            "config": {"workload": f"config 3: {N} orbit-camera rays from inside level 1 (W={W}, near 0.01, far 100), "
                                   f"{levels}-level cascaded {R}^3 grid over [0,1]^3 (to [-3.5,4.5]^3), cone "
                                   f"stepping cone_angle 1/256, step sqrt(3)/1024, SolidSphere r=0.3 sigma=40",
                       "l2": "inputs larger than L2 (~0.4 GB working set per step)"},
            "roofline": {"bound": "hbm", "kernel": "step (vmb_march_render_cascade + vmb_render_backward)",
                         "algorithmic_bytes": step_bytes, "achieved": step_bytes / (ms * 1e-3) / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                         "traffic": None},
            "e2e": {"value": N / (e2e_ms * 1e-3), "unit": "rays/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(sum(a.nbytes for a in host)), "d2h_bytes_per_step": 20 * N},
            "clocks": clk}
    print(json.dumps(line), flush=True)


def make_field(kind, api, dev):
    """(field descriptor, keep-alive, label) of the config 5 step's density field."""
    from paper_2210_04847_b200._lib import Field
    if kind == "checker":
        f = Field.checker(period=0.125, sigma=200.0, rgb_a=(0.8, 0.25, 0.25), rgb_b=(0.2, 0.3, 0.9))
        return f, None, "Checker period 0.125 sigma=200 (dense everywhere, two colours)"
    if kind == "voxel":
        res = 128
        vf = api.VoxelField(res, (0.0, 0.0, 0.0), (1.0, 1.0, 1.0), dev=dev)
        g = (np.arange(res) + 0.0) / (res - 1)
        x, y, z = np.meshgrid(g, g, g, indexing="ij")
        inside = ((x - 0.5) ** 2 + (y - 0.5) ** 2 + (z - 0.5) ** 2) <= 0.2 ** 2
        dens = np.where(inside, 200.0, -30.0).transpose(2, 1, 0).ravel()  # x fastest
        col = np.tile(np.log(np.array([0.8, 0.25, 0.25]) / (1 - np.array([0.8, 0.25, 0.25]))), (res ** 3, 1))
        vf.set_params(dens, col)
        return vf.field, vf, "TrilinearVoxelField 128^3 over [0,1]^3 holding the sphere (raw density 200 / -30)"
    return Field.sphere(**SCENE), None, "SolidSphere r=0.2 sigma=200"


# ---------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "config3":
        return run_config3(args)
    if args.workload == "config1":
        return run_config1(args)
    from paper_2210_04847_b200 import api, workload
    from paper_2210_04847_b200._lib import VMB_F32, Contraction, Field, MarchConfig, Rays, check

    dist = Dist()
    dev = api.Device(dist.local)
    L = dev.lib
    if dist.world > 1:
        uid = (C.c_char * 128)()
        if dist.rank == 0:
            check(L.vmb_comm_unique_id(uid))
        raw = dist.bcast_bytes(bytes(uid))
        uid = (C.c_char * 128).from_buffer_copy(raw)
        check(L.vmb_comm_init(dev.h, uid, dist.world, dist.rank))

    field, field_keep, field_label = make_field(args.field, api, dev)
    cfg = MarchConfig(args.step_size, 1e-4, 1e-2)
    R = args.resolution
    grid = api.OccupancyGrid(R, Contraction.aabb(), dev=dev)
    seeds = workload.grid_warmup_seeds(16, 5)
    dev.record(10)
    for s in seeds:
        grid.update_field(field, 0.95, s)  # sharded probes + ncclAllReduce(max) when N > 1
    dev.record(11)
    grid_update_ms = dev.elapsed_ms(10, 11) / len(seeds)

    strong = args.scaling == "strong"
    angle = 0.0 if strong else 2.0 * math.pi * dist.rank / max(dist.world, 1)
    o64, d64 = workload.orbit_rays(args.width, angle=angle)
    shard = (0, len(o64))
    if strong:  # this rank's contiguous slice of the one batch (parallel_for's static split)
        b_, e_ = C.c_uint64(), C.c_uint64()
        check(L.vmb_shard_range(len(o64), dist.world, dist.rank, C.byref(b_), C.byref(e_)))
        shard = (b_.value, e_.value)
        o64, d64 = o64[shard[0]:shard[1]], d64[shard[0]:shard[1]]
    N = len(o64)
    o32, d32 = o64.astype(np.float32), d64.astype(np.float32)
    if strong:
        dc, do, dd = (x[shard[0]:shard[1]] for x in workload.upstream_grads(args.width ** 2, 113))
    else:
        dc, do, dd = workload.upstream_grads(N, 113 + dist.rank)
    do_, dd_ = dev.upload(o32), dev.upload(d32)
    rays = Rays(do_.ptr, dd_.ptr, VMB_F32, 0, N, 0.2, 1.0)
    check(L.vmb_rays_validate(dev.h, C.byref(rays)))
    up_c, up_o, up_d = dev.upload(dc.astype(np.float32)), dev.upload(do.astype(np.float32)), \
        dev.upload(dd.astype(np.float32))
    packed = api.DevicePacked.allocate(dev, N, 8 * N)
    packed = api.march_device(dev, grid, rays, field, cfg, packed)
    S0 = packed.n_samples
    cap = packed.capacity
    rgb, sig = dev.empty(cap * 3, np.float32), dev.empty(cap, np.float32)
    g_rgb, g_sig = dev.empty(cap * 3, np.float32), dev.empty(cap, np.float32)
    col, op, dep = dev.empty(N * 3, np.float32), dev.empty(N, np.float32), dev.empty(N, np.float32)

    # The step, phase by phase (record(k) brackets the phases for the timing pass):
    #   fusion=none    march | shade | render_forward | render_backward
    #   fusion=shade   march+shade (vmb_march_field_shaded) | render_forward | render_backward
    #   fusion=forward march+shade+render_forward (vmb_march_render_field) | render_backward
    step_no = [0]
    update_seeds = workload.grid_warmup_seeds(4096, 11)

    def step(record=None):
        rec = record or (lambda k: None)
        step_no[0] += 1
        if args.grid_update_every and step_no[0] % args.grid_update_every == 0:
            # config 4's training loop (voxmarch.cpp:514-515): EMA update of the grid
            grid.update_field(field, 0.95, update_seeds[(step_no[0] // args.grid_update_every) % 4096])
        rec(2)
        if args.fusion == "forward":
            api.march_render_device(dev, grid, rays, field, cfg, packed, rgb, sig, col, op, dep)
            rec(3), rec(4), rec(5)
        else:
            if args.fusion == "shade":
                api.march_shaded_device(dev, grid, rays, field, cfg, packed, rgb, sig)
                rec(3)
            else:
                api.march_device(dev, grid, rays, field, cfg, packed)
                rec(3)
                api.shade_device(dev, rays, field, packed, rgb, sig)
            rec(4)
            api.render_forward_device(dev, packed, rgb, sig, col, op, dep)
            rec(5)
        api.render_backward_device(dev, packed, rgb, sig, up_c, up_o, up_d, g_rgb, g_sig)
        rec(6)

    # The timed step: the resident pipeline (sub-batches over several streams) when
    # the forward is fused and no grid update sits inside the loop; else the
    # single-call step above.
    pipe = None
    pipe_step = [0]

    def pipe_update(dry=False):
        """config 4: the grid update due before pipelined step pipe_step (dry: is one due?)"""
        if not args.grid_update_every:
            return False
        due = (pipe_step[0] + 1) % args.grid_update_every == 0
        if dry:
            return due
        pipe_step[0] += 1
        grid.update_field(field, 0.95, update_seeds[(pipe_step[0] // args.grid_update_every) % 4096])
        return True

    def pipe_run(steps):
        for _ in range(steps):
            if not pipe_update(dry=True):
                pipe_step[0] += 1
                pipe.run(1)
            else:
                pipe.run(1, pre_step=pipe_update)

    if args.fusion == "forward" and args.streams * args.chunks > 1:
        pipe = ResidentPipeline(args.streams, args.chunks, api, dev, grid, field, cfg, (do_, dd_), (up_c, up_o, up_d), N, S0)
    clocks = Clocks(dist.local)
    for _ in range(max(args.warmup, 3)):
        step()
        if pipe:
            pipe_run(1)
    dev.sync()
    if pipe:
        pipe.sync()
    dist.barrier()
    if pipe:
        pipe.begin(0)
        pipe_run(args.steps)
        pipe.end(1)
        pipe.sync()
    else:
        dev.record(0)
        for _ in range(args.steps):
            step()
        dev.record(1)
        dev.sync()
    dist.barrier()
    ms_total = dev.elapsed_ms(0, 1)
    # keep the GPU loaded ~1 s more so the clock sampler sees the steady state
    t_end = time.time() + 1.2
    while time.time() < t_end:
        pipe_run(1) if pipe else step()
    dev.sync()
    if pipe:
        pipe.sync()
    clk = clocks.stop()

    S = packed.n_samples
    pipe_info = None
    if pipe:  # the pipelined step's outputs == the single-call step's, bit for bit
        s_pipe = pipe.check()
        pipe_info = {"streams": pipe.S, "sub_batches": pipe.K, "samples": s_pipe}
        if args.grid_update_every:  # the grid moves between the runs: no common state to compare
            pipe_info["matches_single_call_outputs"] = None
        else:
            same = s_pipe == S and all(np.array_equal(a.numpy(), b.numpy(N * w))
                                       for a, b, w in zip(pipe.outs, (col, op, dep), (3, 1, 1)))
            pipe_info["matches_single_call_outputs"] = bool(same)
            assert same, "pipelined step differs from the single-call step"
    ms_step = dist.max(ms_total / args.steps)
    total_rays = dist.sum(float(N))
    total_samples = dist.sum(float(S))
    value = total_rays / (ms_step * 1e-3)

    # per-phase device timing (one more pass, events between phases)
    phase = {}
    if args.phases:
        acc = np.zeros(4)
        for _ in range(args.steps):
            step(dev.record)
            acc += [dev.elapsed_ms(2 + i, 3 + i) for i in range(4)]
        acc /= args.steps
        phase = dict(zip(["march", "shade", "render_forward", "render_backward"], acc.tolist()))

    # roofline (HBM). Algorithmic bytes per SURVEY §8(d): rays f32 (24 B), packed_info
    # 8 B/ray, t's f64 + ray index (20 B/sample), rgb+sigma f32 (16 B), outputs f32.
    pk = peaks()
    peak = pk.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in pk else "fallback"
    # The march phase's compulsory bytes grow with what is fused into it: shading
    # writes rgb+sigma (16 B/sample); the fused forward writes color/opacity/depth
    # (20 B/ray) and does not re-read the samples.
    bytes_march = 24 * N + 8 * N + 20 * S + R ** 3 / 8
    if args.fusion in ("shade", "forward"):
        bytes_march += 16 * S
    if args.fusion == "forward":
        bytes_march += 20 * N
    bytes_fwd = 8 * N + 32 * S + 20 * N
    bytes_bwd = 8 * N + 20 * N + 32 * S + 16 * S
    # step bytes: each API call reads its inputs and writes its outputs
    # once, 88 N + 100 S + R^3/8 for march | forward | backward (shading excluded).
    # With the forward fused into the march, the forward's re-read (8 N + 32 S) is
    # gone, while the fused call must write rgb/sigma (16 S) for the backward, so it
    # is credited only its compulsory traffic: 80 N + 84 S + R^3/8.
    bytes_step = (80 * N + 84 * S if args.fusion == "forward" else 88 * N + 100 * S) + R ** 3 / 8
    dom = max(phase, key=phase.get) if phase else "march"
    dom_bytes = {"march": bytes_march, "shade": 20 * S + 24 * S + 16 * S,
                 "render_forward": bytes_fwd, "render_backward": bytes_bwd}[dom]
    achieved = dom_bytes / (phase.get(dom, ms_step) * 1e-3) / 1e9
    api_name = {"march": {"forward": "vmb_march_render_field", "shade": "vmb_march_field_shaded",
                     "none": "vmb_march_field"}[args.fusion],
           "shade": "vmb_shade_field", "render_forward": "vmb_render_forward",
           "render_backward": "vmb_render_backward"}[dom]
    roof = {"bound": "hbm", "kernel": f"{dom} ({api_name}: {' + '.join(PHASE_KERNELS[dom])})",
            "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic_of(dom), "peak_source": peak_src,
            "algorithmic_bytes": dom_bytes,
            "step": {"algorithmic_bytes": bytes_step,
                     "achieved": bytes_step / (ms_step * 1e-3) / 1e9,
                     "frac": bytes_step / (ms_step * 1e-3) / 1e9 / peak}}

    # e2e: host buffers in, result out, through the C ABI (pinned host staging)
    try:
        e2e = e2e_pipeline(args, dist, api, dev, grid, field, cfg, o32, d32,
                           [x.astype(np.float32) for x in (dc, do, dd)], cap, (col, op, dep), total_rays)
    except Exception as ex:  # pragma: no cover
        e2e = {"error": repr(ex)}
    try:  # the same step with the benchmark camera's rays generated on the device
        ang = 0.0 if strong else 2.0 * math.pi * dist.rank / max(dist.world, 1)
        rad = 0.6 * math.sqrt(3.0) / math.sqrt(3.0)  # orbit_camera's radius, as workload.orbit_rays
        eye = [0.5 + rad * math.cos(ang) * math.cos(0.4), 0.5 + rad * math.sin(ang) * math.cos(0.4),
               0.5 + rad * math.sin(0.4)]
        cam = api.look_at(eye, (0.5, 0.5, 0.5), (0, 0, 1), 1.1 * args.width, args.width, args.width)
        e2e_cam = e2e_pipeline(args, dist, api, dev, grid, field, cfg, o32, d32,
                               [x.astype(np.float32) for x in (dc, do, dd)], cap, (col, op, dep), total_rays, cam,
                               shard[0])
    except Exception as ex:  # pragma: no cover
        e2e_cam = {"error": repr(ex)}

    cfg2 = None
    if dist.rank == 0 and dist.world == 1 and args.config2 and args.width == 2048:
        try:  # BASELINE config 2 (NeRF-Synthetic-shaped batch), same step, its own process
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--width", "512", "--step-size",
                                  repr(math.sqrt(3.0) / 1024), "--steps", str(max(args.steps, 20)), "--warmup",
                                  str(args.warmup), "--cpu-baseline", "0", "--config2", "0", "--phases", "0"],
                                 capture_output=True, text=True, timeout=600)
            c2 = json.loads(out.stdout.strip().splitlines()[-1])
            cfg2 = {k: c2[k] for k in ("value", "unit", "ms_per_step", "samples_per_s")}
            cfg2["workload"] = ("config 2: 262144 orbit-camera rays (W=512), 128^3 grid, step sqrt(3)/1024, "
                                "alpha 1e-2, eps 1e-4, SolidSphere field")
            cfg2["samples"] = c2["config"]["samples_per_gpu"]
            cfg2["roofline_step_frac"] = c2["roofline"]["step"]["frac"]
            cfg2["e2e"] = {k: c2["e2e"].get(k) for k in ("value", "unit", "ms_per_step")}
            cfg2["clocks"] = c2.get("clocks")
        except Exception as ex:  # pragma: no cover
            cfg2 = {"error": repr(ex)}

    res256 = None
    if dist.rank == 0 and dist.world == 1 and args.res256 and args.width == 2048 and args.resolution == 128:
        try:  # BASELINE config 5's second grid size: the same step over a 256^3 grid
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--resolution", "256", "--steps",
                                  str(args.steps), "--warmup", str(args.warmup), "--cpu-baseline", "0",
                                  "--config1", "0", "--config2", "0", "--config3", "0", "--config4", "0",
                                  "--fields", "0", "--res256", "0"],
                                 capture_output=True, text=True, timeout=900)
            c5 = json.loads(out.stdout.strip().splitlines()[-1])
            res256 = {k: c5[k] for k in ("value", "unit", "ms_per_step", "samples_per_s", "phases_ms", "clocks")}
            res256["workload"] = c5["config"]["workload"]
            res256["samples"] = c5["config"]["samples_per_gpu"]
            res256["roofline_step_frac"] = c5["roofline"]["step"]["frac"]
            res256["roofline_march_frac"] = c5["roofline"]["frac"]
        except Exception as ex:  # pragma: no cover
            res256 = {"error": repr(ex)}

    cfg4 = None
    if dist.rank == 0 and dist.world == 1 and args.config4 and args.width == 2048:
        try:  # BASELINE config 4 (training loop shape): 2^20 rays per step, a grid EMA update every 16 steps
            steps4 = max(args.steps, 32)
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--width", "1024", "--grid-update-every",
                                  "16", "--steps", str(steps4), "--warmup", str(args.warmup), "--cpu-baseline", "0",
                                  "--config1", "0", "--config2", "0", "--config3", "0", "--config4", "0",
                                  "--fields", "0", "--phases", "0", "--res256", "0"],
                                 capture_output=True, text=True, timeout=600)
            c4 = json.loads(out.stdout.strip().splitlines()[-1])
            cfg4 = {k: c4[k] for k in ("value", "unit", "ms_per_step", "samples_per_s", "clocks", "grid_update_ms")}
            cfg4["workload"] = (f"config 4: 1048576 orbit-camera rays per step (W=1024), 128^3 grid, an occupancy-grid "
                                f"EMA update (probe + EMA + threshold + distance map) every 16 steps inside the timed "
                                f"loop ({steps4} steps), SolidSphere field")
            cfg4["samples"] = c4["config"]["samples_per_gpu"]
            cfg4["roofline_step_frac"] = c4["roofline"]["step"]["frac"]
        except Exception as ex:  # pragma: no cover
            cfg4 = {"error": repr(ex)}

    fields = None
    if dist.rank == 0 and dist.world == 1 and args.fields and args.field == "sphere" and args.width == 2048:
        fields = {}
        for kind in ("checker", "voxel"):
            try:  # the same step with a general field: no constant-density shortcuts
                out = subprocess.run([sys.executable, os.path.abspath(__file__), "--field", kind, "--steps",
                                      str(args.steps), "--warmup", str(args.warmup), "--cpu-baseline", "0",
                                      "--config1", "0", "--config2", "0", "--config3", "0", "--config4", "0",
                                      "--fields", "0", "--res256", "0"],
                                     capture_output=True, text=True, timeout=900)
                fl = json.loads(out.stdout.strip().splitlines()[-1])
                fields[kind] = {k: fl[k] for k in ("value", "unit", "ms_per_step", "samples_per_s", "phases_ms",
                                                   "clocks")}
                fields[kind]["workload"] = fl["config"]["workload"]
                fields[kind]["samples"] = fl["config"]["samples_per_gpu"]
                fields[kind]["roofline_step_frac"] = fl["roofline"]["step"]["frac"]
                fields[kind]["roofline_march_frac"] = fl["roofline"]["frac"]
            except Exception as ex:  # pragma: no cover
                fields[kind] = {"error": repr(ex)}

    cfg1 = None
    if dist.rank == 0 and dist.world == 1 and args.config1 and args.width == 2048:
        try:  # BASELINE config 1 (4096 rays, launch-bound): CUDA graph, its own process
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--workload", "config1", "--steps",
                                  "200", "--warmup", str(args.warmup)], capture_output=True, text=True, timeout=600)
            c1 = json.loads(out.stdout.strip().splitlines()[-1])
            cfg1 = {k: c1[k] for k in ("value", "unit", "ms_per_step", "calls_ms_per_step", "samples_per_s",
                                       "samples", "clocks")}
            cfg1["workload"] = c1["config"]["workload"]
        except Exception as ex:  # pragma: no cover
            cfg1 = {"error": repr(ex)}

    cfg3 = None
    if dist.rank == 0 and dist.world == 1 and args.config3 and args.width == 2048:
        try:  # BASELINE config 3 (cascaded grid + cone stepping), its own process
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "--workload", "config3", "--steps",
                                  str(max(min(args.steps, 20), 5)), "--warmup", str(args.warmup)],
                                 capture_output=True, text=True, timeout=900)
            c3 = json.loads(out.stdout.strip().splitlines()[-1])
            cfg3 = {k: c3[k] for k in ("value", "unit", "ms_per_step", "samples_per_s", "samples", "e2e",
                                       "clocks", "grid_update_ms")}
            cfg3["workload"] = c3["config"]["workload"]
            cfg3["roofline_step_frac"] = c3["roofline"]["frac"]
        except Exception as ex:  # pragma: no cover
            cfg3 = {"error": repr(ex)}

    cpu = None
    if dist.rank == 0 and dist.world == 1 and args.cpu_baseline:
        try:
            cpu = cpu_baseline(args, o64, d64)
        except Exception as ex:  # pragma: no cover
            cpu = {"error": str(ex)}

    if dist.rank == 0:
        line = {"metric": BASELINE_METRIC, "value": value, "unit": "rays/s", "n_gpus": dist.world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "samples_per_s": total_samples / (ms_step * 1e-3),
                "config": {"workload": (f"config 4: grid update every {args.grid_update_every} steps, "
                                        if args.grid_update_every else "config 5: ") +
                                       f"{N} orbit-camera rays/GPU (W={args.width}), "
                                       f"{R}^3 grid (16 jittered warm-up updates), {field_label}, "
                                       f"step {args.step_size}, alpha 1e-2, eps 1e-4",
                           "rays_per_gpu": N, "samples_per_gpu": S, "resolution": R,
                           "fusion": args.fusion + " (the field's rgb/sigma shaded at sample midpoints)",
                           "storage": "rays/rgb/sigma/outputs f32, t f64, compute f64",
                           "l2": "inputs larger than L2 (~1 GB working set per step)",
                           "parallelism": f"dp{dist.world} (rays sharded, grid replicated)",
                           "sharding": ("one batch of " + str(args.width ** 2) + " rays split by vmb_shard_range "
                                        f"(rank 0: rays [{shard[0]}, {shard[1]}))" if strong else
                                        "each rank its own batch (camera angle 2 pi rank / N)"),
                           "step_schedule": (f"{pipe.K} contiguous sub-batches over {pipe.S} streams "
                                             "(vmb_march_render_field_async + vmb_render_backward each)"
                                             if pipe else "single call sequence on one stream")},
                "pipeline": pipe_info,
                "phases_ms": phase, "grid_update_ms": grid_update_ms,
                "roofline": roof, "e2e": e2e, "e2e_camera": e2e_cam, "cpu_baseline": cpu, "clocks": clk,
                "config1": cfg1, "config2": cfg2, "config3": cfg3, "config4": cfg4, "grid256": res256, "fields": fields,
                "gpu_launches": (KERNELS_PER_STEP - {"none": 0, "shade": 1, "forward": 2}[args.fusion])
                * args.steps * (pipe.K if pipe else 1)}
        print(json.dumps(line), flush=True)
    if dist.world > 1:
        L.vmb_comm_destroy(dev.h)


if __name__ == "__main__":
    main()
