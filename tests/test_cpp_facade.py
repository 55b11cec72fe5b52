"""The C++ drop-in facade (namespace voxmarch over the C ABI).

* CPU: libvoxmarch_cpp.so exports the reference API surface.
* GPU: build/vm_cpp_tests (this repo's C++ tests of the facade) and
  build/ref_unit_tests — the REFERENCE's own hot-path unit tests
  (proj/tests/unit/test_{core_types,contraction,occupancy_grid,ray_marching,
  rendering,fields,scene_camera}.cpp, compiled unchanged against include/voxmarch/ by
  tests/ref_unit/Makefile) — must pass on the B200.
"""
import os
import subprocess

import pytest

from conftest import ROOT

LIB = os.path.join(ROOT, "paper_2210_04847_b200", "lib", "libvoxmarch_cpp.so")

API = ["voxmarch::march(voxmarch::RayBatch const&, voxmarch::OccupancyGrid const&, std::function",
       "voxmarch::march_uniform(", "voxmarch::uniform_step_count(", "voxmarch::pack(",
       "voxmarch::validate[abi:cxx11](", "voxmarch::transmittance(", "voxmarch::render_forward(",
       "voxmarch::render_backward(", "voxmarch::render_attribute(", "voxmarch::contract(",
       "voxmarch::invert_grid_point(", "voxmarch::RayBatch::create(",
       "voxmarch::OccupancyGrid::OccupancyGrid(unsigned int", "voxmarch::OccupancyGrid::query(",
       "voxmarch::OccupancyGrid::update(", "voxmarch::OccupancyGrid::update_over_time(",
       "voxmarch::OccupancyGrid::seed_occupancy(", "voxmarch::OccupancyGrid::save(",
       "voxmarch::OccupancyGrid::load(", "voxmarch::OccupancyGrid::occupied_fraction(",
       "voxmarch::OccupancyGrid::threshold_density(", "voxmarch::TrilinearVoxelField::backward(",
       "voxmarch::TrilinearVoxelField::query_rgb_sigma(", "voxmarch::TrilinearVoxelField::load(",
       "voxmarch::AdamOptimizer::step(", "voxmarch::generate_rays(", "voxmarch::look_at(",
       "voxmarch::load_camera_json("]


def test_facade_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", LIB], capture_output=True, text=True,
                         check=True).stdout
    missing = [a for a in API if a not in out]
    assert not missing, missing


def _run(binary):
    path = os.path.join(ROOT, "build", binary)
    if not os.path.exists(path):
        pytest.skip(f"{binary} not built")
    p = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(p.stdout[-4000:])
    print(p.stderr[-4000:])
    return p


@pytest.mark.gpu
def test_cpp_facade_tests_on_gpu():
    p = _run("vm_cpp_tests")
    assert p.returncode == 0, p.stderr[-2000:]


@pytest.mark.gpu
def test_reference_unit_tests_against_facade_on_gpu():
    p = _run("ref_unit_tests")
    assert p.returncode == 0, p.stderr[-2000:]
    assert "0 failed" in p.stdout
