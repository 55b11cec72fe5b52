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
