"""The device side of the multi-GPU grid update, on one GPU.

Each rank of a multi-GPU update runs vmb_grid_probe_field_range on its
vmb_shard_range slice of cells, the buffers are combined by ncclAllReduce(max)
(u64 bit patterns of non-negative doubles) and vmb_grid_apply folds them into the
cache. Here the ranks' probes run one after the other on the same device and the
max is taken on the host, so the kernels of the sharded path are checked without
running kernels that wait on each other. The grid must be bit-identical to the
single-GPU fused update and to the oracle, for 1..8 "ranks".
"""
import ctypes as C

import numpy as np
import pytest

from oracle import Oracle, available
from oracle import oracle as O
from paper_2210_04847_b200 import api, workload
from paper_2210_04847_b200._lib import Contraction, Field, check

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_probe_allreduce_apply_matches_fused(world):
    dev = api.Device(0)
    L = dev.lib
    R = 64
    field = Field.sphere(center=(0.45, 0.5, 0.55), radius=0.27, sigma=90.0, velocity=(0.05, 0, 0))
    fused = api.OccupancyGrid(R, Contraction.aabb(), dev=dev)
    sharded = api.OccupancyGrid(R, Contraction.aabb(), dev=dev)
    n = R ** 3
    ts = np.array([0.0, 0.7])
    probe = dev.empty(n, np.float64)
    for s in workload.grid_warmup_seeds(5, 9):
        fused.update_field(field, 0.9, s, ts)
        combined = np.zeros(n)
        for rank in range(world):
            c0, c1 = api.shard_range(n, world, rank)
            check(L.vmb_grid_probe_field_range(dev.h, sharded.h, C.byref(field),
                                               ts.ctypes.data_as(C.POINTER(C.c_double)), len(ts),
                                               1, s, c0, c1, probe.ptr))
            part = probe.numpy()
            assert not part[:c0].any() and not part[c1:].any()
            # max of the u64 bit patterns == max of the doubles (all >= 0)
            combined = np.maximum(combined.view(np.uint64), part.view(np.uint64)).view(np.float64)
        dev_combined = dev.upload(combined)
        check(L.vmb_grid_apply(dev.h, sharded.h, dev_combined.ptr, 0.9))
    assert np.array_equal(sharded.bits(), fused.bits())
    assert np.array_equal(sharded.density_cache(), fused.density_cache())
    orc = Oracle("ref") if available("ref") else Oracle("port")
    of = O.Field.sphere(center=(0.45, 0.5, 0.55), radius=0.27, sigma=90.0, velocity=(0.05, 0, 0))
    og = orc.grid(R, O.Contraction.aabb())
    for s in workload.grid_warmup_seeds(5, 9):
        og.update_field(of, 0.9, s, ts)
    assert np.array_equal(fused.bits(), og.bits())


def test_nccl_single_rank_communicator_runs_the_collective_path():
    """With a communicator attached (here 1 rank on cuda:0) the grid update takes the
    sharded probe + ncclAllReduce(max) + apply path through the real NCCL library, and
    the grid equals the plain fused update bit for bit; the training all-reduce(sum)
    of a 1-rank communicator is the identity."""
    import ctypes as C
    import os
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    from paper_2210_04847_b200 import api, workload
    from paper_2210_04847_b200._lib import Contraction, Field, check
    dev, plain = api.Device(0), api.Device(0)
    L = dev.lib
    uid = (C.c_char * 128)()
    check(L.vmb_comm_unique_id(uid))
    check(L.vmb_comm_init(dev.h, uid, 1, 0))
    try:
        field = Field.sphere(**workload.SPHERE)
        g1 = api.OccupancyGrid(128, Contraction.aabb(), dev=dev)
        g2 = api.OccupancyGrid(128, Contraction.aabb(), dev=plain)
        for s in workload.grid_warmup_seeds(4, 5):
            g1.update_field(field, 0.95, s)
            g2.update_field(field, 0.95, s)
        assert np.array_equal(g1.bits(), g2.bits())
        assert np.array_equal(g1.density_cache(), g2.density_cache())
        x = np.random.default_rng(0).normal(size=1000)
        buf = dev.upload(x)
        check(L.vmb_comm_allreduce_sum_f64(dev.h, buf.ptr, 1000))
        assert np.array_equal(buf.numpy(), x)
    finally:
        check(L.vmb_comm_destroy(dev.h))
