"""Pinhole cameras and ray generation (scene_camera.cpp:10-63).

CPU: the C restatement (port) against the reference's own look_at/generate_rays
(ref), bit for bit, including the validation messages; the bench's Python ray
source (workload.orbit_rays) against the reference. GPU: vmb_generate_rays
against the port, bit for bit in f64 and as the once-rounded f32 values.
"""
import math

import numpy as np
import pytest

from oracle import OracleError
from oracle.oracle import Camera as OCamera
from paper_2210_04847_b200 import workload


def _orbit_eye(angle, elevation=0.4):
    radius = 0.6 * math.sqrt(3.0) / math.sqrt(3.0)
    return [0.5 + radius * math.cos(angle) * math.cos(elevation),
            0.5 + radius * math.sin(angle) * math.cos(elevation),
            0.5 + radius * math.sin(elevation)]


CAMS = [  # (eye, target, up, focal, width, height)
    (_orbit_eye(0.0), [0.5, 0.5, 0.5], [0, 0, 1], 1.1 * 64, 64, 64),
    (_orbit_eye(1.3), [0.5, 0.5, 0.5], [0, 0, 1], 1.1 * 48, 48, 30),
    ([0.1, -2.0, 0.7], [0.3, 0.2, 0.1], [0.2, 0.1, 1.0], 37.5, 17, 23),
    ([3.0, 1.0, -2.0], [0.0, 0.0, 0.0], [0, 1, 0], 1000.0, 5, 1),
]


@pytest.mark.parametrize("k", range(len(CAMS)))
def test_look_at_and_generate_rays_match_reference(ref, port, k):
    eye, tgt, up, f, w, h = CAMS[k]
    ca, cb = ref.look_at(eye, tgt, up, f, w, h), port.look_at(eye, tgt, up, f, w, h)
    assert bytes(ca) == bytes(cb)
    oa, da = ref.generate_rays(ca, 0.2, 1.0)
    ob, db = port.generate_rays(cb, 0.2, 1.0)
    assert np.array_equal(oa, ob) and np.array_equal(da, db)
    assert len(oa) == w * h


def test_bench_rays_are_the_reference_orbit_camera(ref):
    o, d = workload.orbit_rays(40, angle=0.7)
    cam = ref.look_at(_orbit_eye(0.7), [0.5, 0.5, 0.5], [0, 0, 1], 1.1 * 40, 40, 40)
    oa, da = ref.generate_rays(cam, 0.2, 1.0)
    assert np.array_equal(o, oa) and np.array_equal(d, da)


def _bad_cameras():
    good = (_orbit_eye(0.0), [0.5, 0.5, 0.5], [0, 0, 1], 64.0, 8, 8)
    yield "look_at", (good[0], good[0], [0, 0, 1], 64.0, 8, 8), "look_at: eye and target coincide"
    yield "look_at", ([0.5, 0.5, 2.0], [0.5, 0.5, 0.5], [0, 0, 1], 64.0, 8, 8), \
        "look_at: up is parallel to view direction"
    yield "look_at", good[:3] + (0.0, 8, 8), "camera: focal must be > 0"
    yield "look_at", good[:3] + (64.0, 0, 8), "camera: image dimensions must be positive"


@pytest.mark.parametrize("case", list(_bad_cameras()), ids=lambda c: c[2])
def test_camera_errors_match_reference(oracle_impl, case):
    _, args, msg = case
    with pytest.raises(OracleError) as e:
        oracle_impl.look_at(*args)
    assert e.value.msg == msg


def test_rotation_checks_match_reference(ref, port):
    cam = ref.look_at(_orbit_eye(0.0), [0.5, 0.5, 0.5], [0, 0, 1], 64.0, 4, 4)
    skew = OCamera.from_buffer_copy(bytes(cam))
    skew.rotation[0] += 1e-3
    flip = OCamera.from_buffer_copy(bytes(cam))
    for i in (0, 3, 6):  # negate column 0: orthonormal, determinant -1
        flip.rotation[i] = -flip.rotation[i]
    for o in (ref, port):
        with pytest.raises(OracleError) as e:
            o.generate_rays(skew, 0.2, 1.0)
        assert e.value.msg == "camera: rotation is not orthonormal"
        with pytest.raises(OracleError) as e:
            o.generate_rays(flip, 0.2, 1.0)
        assert e.value.msg == "camera: rotation determinant must be +1"
        with pytest.raises(OracleError) as e:
            o.generate_rays(cam, 1.0, 1.0)
        assert e.value.msg == "ray batch: requires far > near >= 0"


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CAMS)))
def test_device_generate_rays_bit_exact(port, k):
    from paper_2210_04847_b200 import api
    from paper_2210_04847_b200._lib import Camera
    eye, tgt, up, f, w, h = CAMS[k]
    cam_o = port.look_at(eye, tgt, up, f, w, h)
    cam = api.look_at(eye, tgt, up, f, w, h)
    assert bytes(cam) == bytes(cam_o)  # host look_at == the reference's expressions
    o_ref, d_ref = port.generate_rays(cam_o, 0.2, 1.0)
    dev = api.Device(0)
    rays, o, d = api.generate_rays_device(dev, Camera.from_buffer_copy(bytes(cam)), 0.2, 1.0, np.float64)
    assert rays.n_rays == w * h and rays.near_plane == 0.2 and rays.far_plane == 1.0
    assert np.array_equal(o.numpy().reshape(-1, 3), o_ref)
    assert np.array_equal(d.numpy().reshape(-1, 3), d_ref)
    rays32, o32, d32 = api.generate_rays_device(dev, cam, 0.2, 1.0, np.float32)
    assert np.array_equal(d32.numpy().reshape(-1, 3), d_ref.astype(np.float32))
    assert np.array_equal(o32.numpy().reshape(-1, 3), o_ref.astype(np.float32))


@pytest.mark.gpu
def test_device_generate_rays_errors():
    from paper_2210_04847_b200 import api
    dev = api.Device(0)
    cam = api.look_at(_orbit_eye(0.0), [0.5, 0.5, 0.5], [0, 0, 1], 64.0, 4, 4)
    with pytest.raises(ValueError, match="requires far > near >= 0"):
        api.generate_rays_device(dev, cam, 0.5, 0.5)
    cam.position[1] = float("nan")
    with pytest.raises(ValueError, match="non-finite ray at index 0"):
        api.generate_rays_device(dev, cam, 0.2, 1.0)
