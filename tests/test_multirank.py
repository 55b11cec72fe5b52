"""Multi-rank decomposition of the path, on CPU with torch.distributed (gloo,
world size 2): exactly the host logic the multi-GPU run uses.

* grid update: each rank probes one equal block of cells (B = ceil(n / world),
  as vmb_grid_update_field does under NCCL) -> in-place all_gather of the blocks
  -> EMA/binarise; the grid must be bit-identical to a single-process update and
  to the reference;
* marching: each rank marches its contiguous ray shard; the global packing is
  the concatenation with offsets shifted by the exclusive scan of the per-rank
  sample totals (all_gather) and must equal the single-process packing.
The compute inside each rank is the C oracle (this container has no GPU); the
GPU kernels of the same decomposition are checked in test_gpu_parity.py.
"""
import ctypes as C
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import Oracle
    from oracle import oracle as O
    from paper_2210_04847_b200 import _lib, workload
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _lib.lib()
    port_o = Oracle("port")
    field = O.Field.sphere(**workload.SPHERE)
    R = 32
    g = port_o.grid(R, O.Contraction.aabb())
    seeds = workload.grid_warmup_seeds(4, 5)
    n = R ** 3
    B = (n + world - 1) // world
    for s in seeds:
        c0, c1 = B * rank, min(n, B * (rank + 1))
        mine = np.zeros(B)
        mine[:c1 - c0] = g.probe_range(field, c0, c1, seed=s)[c0:c1]
        blocks = [torch.zeros(B, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(blocks, torch.from_numpy(mine))
        g.apply(torch.cat(blocks).numpy()[:n], 0.95)
    bits, cache = g.bits(), g.cache()
    # ray sharding + global packing
    o, d = workload.orbit_rays(24)
    b, e = C.c_uint64(), C.c_uint64()
    lib.vmb_shard_range(len(o), world, rank, C.byref(b), C.byref(e))
    p = port_o.march_field(o[b.value:e.value], d[b.value:e.value], 0.2, 1.0, g, field,
                           O.MarchConfig(5e-3, 1e-4, 1e-2))
    totals = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(totals, torch.tensor([p.n_samples], dtype=torch.int64))
    base = int(sum(t.item() for t in totals[:rank]))
    parts = [None] * world
    dist.all_gather_object(parts, (p.offsets + base, p.counts, p.t_starts, p.t_ends,
                                   p.ray_indices + b.value))
    if rank == 0:
        q.put(dict(bits=bits, cache=cache, parts=parts))
    dist.destroy_process_group()


def test_two_rank_grid_update_and_ray_sharding():
    import torch.multiprocessing as mp
    from oracle import Oracle
    from oracle import oracle as O
    from paper_2210_04847_b200 import workload
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    orc = Oracle("port")
    field = O.Field.sphere(**workload.SPHERE)
    g = orc.grid(32, O.Contraction.aabb())
    for s in workload.grid_warmup_seeds(4, 5):
        g.update_field(field, 0.95, s)
    assert np.array_equal(res["bits"], g.bits())
    assert np.array_equal(res["cache"], g.cache())
    o, d = workload.orbit_rays(24)
    full = orc.march_field(o, d, 0.2, 1.0, g, field, O.MarchConfig(5e-3, 1e-4, 1e-2))
    cat = [np.concatenate([part[i] for part in res["parts"]]) for i in range(5)]
    for got, k in zip(cat, ("offsets", "counts", "t_starts", "t_ends", "ray_indices")):
        assert np.array_equal(got, getattr(full, k)), k
