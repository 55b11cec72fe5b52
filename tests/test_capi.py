"""C-ABI library checks that need no GPU: it loads, exports every symbol declared in
include/vmb200.h, its host-only helpers agree with the reference, and compute
entry points fail loudly (no CPU fallback) when no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import HAS_GPU, ROOT
from paper_2210_04847_b200 import _lib

HEADER = os.path.join(ROOT, "include", "vmb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(vmb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared_symbols()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes signature table covers the whole header
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_struct_layouts_match_oracle():
    from oracle import oracle as o
    for a, b in [(_lib.Contraction, o.Contraction), (_lib.Field, o.Field),
                 (_lib.MarchConfig, o.MarchConfig)]:
        assert C.sizeof(a) == C.sizeof(b)
        assert [f[0] for f in a._fields_] == [f[0] for f in b._fields_]
    assert C.sizeof(_lib.Field) == 8 + 3 * 8 * 3 + 8 + 8 + 24 + 24 + 8 + 24 + 8 + 8 + 8
    assert C.sizeof(_lib.Rays) == 48 and C.sizeof(_lib.Samples) == 48


def test_uniform_step_count_matches_reference(port):
    lib = _lib.lib()
    rng = np.random.default_rng(0)
    for _ in range(3000):
        near = rng.uniform(0, 2)
        far = near + rng.choice([0.0, rng.uniform(0, 5)])
        step = rng.choice([5e-3, 1.6914558667664816e-3, rng.uniform(1e-4, 0.3)])
        assert lib.vmb_uniform_step_count(near, far, step) == port.uniform_step_count(near, far, step)


def test_shard_range_is_parallel_for_split():
    lib = _lib.lib()
    for n in (0, 1, 7, 4096, 4194304, 2 ** 21 + 3):
        for g in (1, 2, 3, 4, 8):
            spans = []
            for r in range(g):
                b, e = C.c_uint64(), C.c_uint64()
                assert lib.vmb_shard_range(n, g, r, C.byref(b), C.byref(e)) == 0
                spans.append((b.value, e.value))
            # contiguous, ordered, covering [0, n)
            covered = [i for b, e in spans for i in ((b, e),)]
            assert covered[0][0] == 0 and covered[-1][1] == n
            for (b0, e0), (b1, e1) in zip(covered, covered[1:]):
                assert e0 == b1 or (e0 == n and b1 == n)
    b, e = C.c_uint64(), C.c_uint64()
    assert lib.vmb_shard_range(10, 2, 2, C.byref(b), C.byref(e)) == _lib.VMB_INVALID_ARGUMENT


@pytest.mark.skipif(HAS_GPU, reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device():
    lib = _lib.lib()
    h = C.c_void_p()
    rc = lib.vmb_ctx_create(0, C.byref(h))
    assert rc == _lib.VMB_CUDA
    assert "no CUDA device" in lib.vmb_last_error().decode()
    from paper_2210_04847_b200 import api
    with pytest.raises(_lib.VmbError):
        api.Device(0)
