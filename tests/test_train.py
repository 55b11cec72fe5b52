"""Data-parallel voxel-field training (paper_2210_04847_b200/train.py; the reference
CLI's cmd_train, tools/voxmarch.cpp:400-562).

CPU: the vectorised Rng streams equal the reference's scalar Rng; the DP
decomposition (per-rank gradients, all-reduce(sum), identical Adam on every rank)
over gloo with world size 2, the gradients computed by the C oracle.
GPU: one full iteration (gather, march with the voxel field, shading, forward,
loss, backward, field backward, Adam) against the same iteration assembled from
the oracle's pieces; a short run lowers the loss.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_2210_04847_b200 import train, workload


def test_vectorised_rng_matches_reference_stream():
    a, b = workload.Rng(42), workload.Rng(42)
    got = train.uniform_below_batch(a, 1000003, 500)
    want = [train._uniform_below(b, 1000003) for _ in range(500)]
    assert [int(x) for x in got] == want and a.state == b.state
    u = train.uniform_batch(a, -1e-4, 1e-4, 300)
    assert np.array_equal(u, [b.uniform(-1e-4, 1e-4) for _ in range(300)]) and a.state == b.state


def _adam(p, g, m, v, lr, t, b1=0.9, b2=0.999, eps=1e-8):
    """AdamOptimizer::step (fields.cpp:282-291), element-wise in numpy (IEEE f64)."""
    m[:] = b1 * m + (1.0 - b1) * g
    v[:] = b2 * v + (1.0 - b2) * g * g
    bias1, bias2 = 1.0 - b1 ** float(t), 1.0 - b2 ** float(t)
    p -= lr * (m / bias1) / (np.sqrt(v / bias2) + eps)


def oracle_iteration(orc, o, d, tgt, dens, col, res, box, grid, cfg, near, far):
    """One cmd_train iteration from the oracle's pieces; returns loss and grads."""
    f = O.Field.voxel(res, box[0], box[1], dens, col)
    q = orc.march_field(o, d, near, far, grid, f, cfg)
    rgb, sig = orc.shade(o, d, q, f)
    color, op, _ = orc.render_forward(q, rgb, sig)
    n = len(o)
    inv = 1.0 / (3.0 * n)
    err = color + (1.0 - op)[:, None] - tgt
    loss = 0.0
    for r in range(n):
        loss += float(err[r] @ err[r]) * inv
    dcol = err * (2.0 * inv)
    dop = (-2.0 * inv) * ((err[:, 0] + err[:, 1]) + err[:, 2])
    drgb, dsig = orc.render_backward(q, rgb, sig, dcol, dop, np.zeros(n))
    ri = q.ray_indices.astype(np.int64)
    pos = o[ri] + d[ri] * (0.5 * (q.t_starts + q.t_ends))[:, None]
    gd, gc = orc.voxel_field_backward(f, pos, drgb, dsig)
    return loss, gd, gc, q


# ------------------------------------------------------------------ DP decomposition (gloo, CPU)
_WORKER = r"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
from oracle import Oracle, oracle as O
from paper_2210_04847_b200 import train, workload
sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
from test_train import oracle_iteration, _adam
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
orc = Oracle("port")
res, box = 5, ((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
rng = np.random.default_rng(0)
dens, col = rng.normal(size=res ** 3), rng.normal(size=3 * res ** 3)
o, d = workload.orbit_rays(12)
tgt = np.random.default_rng(1).uniform(size=(len(o), 3))
g = orc.grid(16, O.Contraction.aabb(), 1e-2, 0.0, 10.0)
cfg = O.MarchConfig(1.6914558667664816e-3, 1e-4, 0.0)
pick = train.uniform_below_batch(workload.Rng(7 + rank), len(o), 40).astype(np.int64)
loss, gd, gc, _ = oracle_iteration(orc, o[pick], d[pick], tgt[pick], dens, col, res, box, g, cfg, 0.2, 1.0)
t = torch.from_numpy(np.concatenate([gd, gc]))
dist.all_reduce(t, op=dist.ReduceOp.SUM)  # the NCCL sum of the device path, here over gloo
gsum = t.numpy()
p = np.concatenate([dens, col]); m = np.zeros_like(p); v = np.zeros_like(p)
_adam(p, gsum, m, v, 0.1, 1)
out = [None] * world
dist.all_gather_object(out, (p, gd, gc))
if rank == 0:
    # parameters identical on every rank, and equal to the single-process update
    # with the sum of both ranks' gradients
    assert all(np.array_equal(out[0][0], x[0]) for x in out)
    ref = np.concatenate([out[0][1] + out[1][1], out[0][2] + out[1][2]])
    q = np.concatenate([dens, col]); m2 = np.zeros_like(q); v2 = np.zeros_like(q)
    _adam(q, ref, m2, v2, 0.1, 1)
    assert np.array_equal(q, out[0][0])
    assert not np.array_equal(out[0][1], out[1][1])  # different minibatches per rank
    print("DP_OK")
"""


def test_data_parallel_gradient_sum_gloo(tmp_path):
    from conftest import ROOT
    script = tmp_path / "dp_worker.py"
    script.write_text(_WORKER)
    env = dict(os.environ, ROOT=ROOT)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29641", str(script)],
                       capture_output=True, text=True, env=env, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "DP_OK" in p.stdout


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_one_iteration_matches_oracle(port):
    from paper_2210_04847_b200 import api
    dev = api.Device(0)
    opts = train.TrainOptions(n_views=2, eval_views=1, iterations=3, width=12, height=12, field_resolution=6,
                              batch_size=96, grid_resolution=16, grid_update_every=2)
    tr = train.Trainer(opts, dev)
    dens, col = tr.field.raw_density(), tr.field.raw_color()
    rng = workload.Rng(0)
    rng.state = tr.rng.state
    pick = train.uniform_below_batch(rng, tr.pool, opts.batch_size).astype(np.int64)
    po, pd, pc = (a.numpy().reshape(-1, 3) for a in (tr.pool_o, tr.pool_d, tr.pool_c))
    o, d, tgt = po[pick], pd[pick], pc[pick]
    og = port.grid(16, O.Contraction.aabb(), 1e-2, 0.0, 4.0 * tr.grid.threshold_density())
    assert np.array_equal(og.bits(), tr.grid.bits())
    cfg = O.MarchConfig(tr.cfg.step_size, 1e-4, 0.0)
    box = (tuple(tr.lo), tuple(tr.hi))
    loss_o, gd_o, gc_o, q = oracle_iteration(port, o, d, tgt, dens, col, 6, box, og, cfg, 0.2, 1.0)

    loss = tr.step(1)
    p = tr.packed.to_host()
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), getattr(q, k)), k
    assert q.n_samples > 1000
    assert abs(loss - loss_o) <= 1e-12 * abs(loss_o)
    scale = max(np.abs(gd_o).max(), np.abs(gc_o).max())
    np.testing.assert_allclose(tr.grad_d.numpy(), gd_o, rtol=1e-9, atol=1e-12 * scale)
    np.testing.assert_allclose(tr.grad_c.numpy(), gc_o, rtol=1e-9, atol=1e-12 * scale)
    # Adam (t = 1, lr_density 8, lr 0.1) on the oracle's gradients
    pd_ = dens.copy()
    _adam(pd_, gd_o, np.zeros_like(pd_), np.zeros_like(pd_), 8.0, 1)
    pc_ = col.copy()
    _adam(pc_, gc_o, np.zeros_like(pc_), np.zeros_like(pc_), 0.1, 1)
    np.testing.assert_allclose(tr.field.raw_density(), pd_, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(tr.field.raw_color(), pc_, rtol=1e-9, atol=1e-9)


@pytest.mark.gpu
def test_short_run_learns():
    from paper_2210_04847_b200 import api
    opts = train.TrainOptions(n_views=8, eval_views=2, iterations=120, width=32, height=32, field_resolution=16,
                              batch_size=1024, grid_resolution=64)
    tr = train.Trainer(opts, api.Device(0))
    for it in range(1, opts.iterations + 1):
        tr.step(it)
    first, last = np.mean(tr.loss_curve[:10]), np.mean(tr.loss_curve[-10:])
    assert last < 0.5 * first, (first, last)
    rep = tr.report(0.0)
    assert rep["psnr_train"] > 15.0 and np.isfinite(rep["psnr_eval"])
    assert 0.0 < rep["occupied_fraction"] <= 1.0  # the grid starts at 4x threshold and decays 0.95 per update
