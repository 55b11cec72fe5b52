"""The C restatement (oracle/vm_oracle.c) reproduces the reference-generated golden
fixtures bit for bit. Runs anywhere (no /root/reference needed)."""
import os

import numpy as np
import pytest

from oracle import Contraction, Field, MarchConfig, Packed
from paper_2210_04847_b200 import workload

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_config1_golden(port):
    z = np.load(os.path.join(G, "c1.npz"))
    field = Field.sphere(**workload.SPHERE)
    g = port.grid(128, Contraction.aabb())
    for s in workload.grid_warmup_seeds(16, 5):
        g.update_field(field, 0.95, s)
    assert np.array_equal(np.packbits(g.bits(), bitorder="little"), z["bits"])
    assert np.array_equal(g.cache().astype(np.float32), z["cache"])
    o, d = workload.orbit_rays(64)
    p = port.march_field(o, d, 0.2, 1.0, g, field, MarchConfig(5e-3, 1e-4, 1e-2))
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), z[k]), k
    assert p.samples_emitted == z["emitted"] == 107555
    assert p.samples_kept == z["kept"] == 19362
    rgb, sig = port.shade(o, d, p, field)
    assert np.array_equal(rgb, z["rgbs"]) and np.array_equal(sig, z["sigmas"])
    for a, k in zip(port.render_forward(p, rgb, sig), ("color", "opacity", "depth")):
        assert np.array_equal(a, z[k]), k
    d_rgb, d_sig = port.render_backward(p, rgb, sig, z["d_color"], z["d_opacity"], z["d_depth"])
    assert np.array_equal(d_rgb, z["d_rgbs"]) and np.array_equal(d_sig, z["d_sigmas"])


def test_growth_golden(port):
    z = np.load(os.path.join(G, "growth.npz"))
    con = Contraction.sphere((0.5, 0.5, 0.5), 0.5)
    field = Field.sphere(radius=0.3, sigma=40.0)
    g = port.grid(64, con)
    for s in (1, 2, 3):
        g.update_field(field, 0.95, s)
    assert np.array_equal(np.packbits(g.bits(), bitorder="little"), z["bits"])
    cfg = MarchConfig(1.6914558667664816e-3, 1e-4, 1e-2, 2048, 1.01)
    p = port.march_field(z["origins"], z["dirs"], 0.01, 100.0, g, field, cfg)
    for k in ("offsets", "counts", "t_starts", "t_ends", "ray_indices"):
        assert np.array_equal(getattr(p, k), z[k]), k
    assert p.samples_emitted == z["emitted"]


def test_render_golden(port):
    z = np.load(os.path.join(G, "render.npz"))
    for i in range(60):
        k = lambda n: z[f"{i}_{n}"]  # noqa: E731
        p = Packed(k("offsets"), k("counts"), k("t_starts"), k("t_ends"),
                   np.repeat(np.arange(len(k("counts")), dtype=np.uint32), k("counts")))
        assert np.array_equal(port.transmittance(p, k("sigmas")), k("trans"))
        c, o, d = port.render_forward(p, k("rgbs"), k("sigmas"))
        assert np.array_equal(c, k("color")) and np.array_equal(o, k("opacity"))
        assert np.array_equal(d, k("depth"))
        dr, ds = port.render_backward(p, k("rgbs"), k("sigmas"), k("d_color"), k("d_opacity"),
                                      k("d_depth"))
        assert np.array_equal(dr, k("d_rgbs")) and np.array_equal(ds, k("d_sigmas"))
        assert np.array_equal(port.render_attribute(p, k("sigmas"), k("values"), 2), k("attr"))
