"""C-ABI checks that need no GPU: the library builds/loads, exports every
symbol include/gsr.h declares, and validates arguments on the host."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import scenegen as sg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def gsr():
    from paper_2503_11731_b200 import gsr as g
    g.load()
    return g


def test_exports_every_declared_symbol(gsr):
    hdr = open(os.path.join(ROOT, "include", "gsr.h")).read()
    declared = set(re.findall(r"\b(gs_[a-z_0-9]+)\s*\(", hdr))
    assert {"gs_project", "gs_bin_sort", "gs_render_camera", "gs_render_lidar"} <= declared
    lib = C.CDLL(gsr.load()._name)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared <= set(gsr.EXPORTS)


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2503_11731_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.SO],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_opts_are_north_star(gsr):
    o = gsr.default_opts()
    assert (o.tile_w, o.tile_h) == (16, 8) and o.split_len == 0
    assert o.alpha_max == pytest.approx(0.99) and o.alpha_min == pytest.approx(1 / 255)
    assert o.t_min == pytest.approx(1e-4) and o.support_rho == 9.0
    assert o.lowpass_sigma_px == pytest.approx(2 ** -0.5) and o.near_plane == pytest.approx(0.2)
    assert o.bg_raydrop == 1.0
    assert o.grid_share == 0.0   # 0 = the compositor's grid fills the GPU


@pytest.mark.parametrize("share,ok", [(0.0, True), (0.25, True), (1.0, True), (-0.1, False), (1.5, False),
                                      (float("nan"), False)])
def test_grid_share_validation(gsr, share, ok):
    cam = gsr.Sensor(sg.tiny().sensors[0])
    o = gsr.default_opts(grid_share=share)
    assert (gsr.gs_num_tiles(cam, o) > 0) == ok
    if not ok:
        assert "grid_share" in gsr.load().gs_last_error().decode()


def _call_project(gsr, sensor, opts=None, n=0):
    opts = opts or gsr.default_opts()
    s = gsr.gs_surfels()
    s.n = n
    buf = (C.c_uint8 * 512)()
    return gsr.load().gs_project(C.byref(s), sensor.ref, C.byref(opts),
                                 C.cast(buf, C.c_void_p), 512, None, None)


def test_host_validation_errors(gsr):
    lib = gsr.load()
    opts = gsr.default_opts()
    cam = gsr.Sensor(sg.tiny().sensors[0])
    # wrong modality for the call -> configuration error
    li = gsr.Sensor(sg.lidar64(sg.lidar_pose([0, 0, 0]), height=8, width=64))
    dummy = C.c_void_p(1)
    assert lib.gs_render_camera(dummy, 0, dummy, dummy, None, li.ref, C.byref(opts), dummy, 1 << 20,
                                None, None, None, dummy, None, None) == gsr.GS_ERR_CONFIG
    assert lib.gs_render_lidar(dummy, 0, dummy, dummy, None, cam.ref, C.byref(opts), dummy, 1 << 20,
                               None, None, None, dummy, None, None) == gsr.GS_ERR_CONFIG
    # render workspace too small
    assert lib.gs_render_camera(dummy, 0, dummy, dummy, None, cam.ref, C.byref(opts), dummy, 16,
                                None, None, None, dummy, None, None) == gsr.GS_ERR_CONFIG
    # non-monotone beam table -> range error
    bad = sg.lidar64(sg.lidar_pose([0, 0, 0]), height=8, width=64)
    bad.beam_elevation = bad.beam_elevation[::-1].copy()
    assert _call_project(gsr, gsr.Sensor(bad)) == gsr.GS_ERR_RANGE
    # focal <= 0, tile too large, theta_max out of range
    z = sg.pinhole(10, 10, 0.0, 5, 5, sg.identity_pose())
    assert _call_project(gsr, gsr.Sensor(z)) == gsr.GS_ERR_RANGE
    assert _call_project(gsr, cam, gsr.default_opts(tile_w=64, tile_h=32)) == gsr.GS_ERR_RANGE
    fe = sg.fisheye(10, 10, 3.5, np.zeros(4, np.float32), 5, 5, sg.identity_pose())
    assert _call_project(gsr, gsr.Sensor(fe)) == gsr.GS_ERR_RANGE
    # buffer too small, null pointers
    assert _call_project(gsr, cam, n=1000) == gsr.GS_ERR_CONFIG
    assert lib.gs_project(None, cam.ref, C.byref(opts), dummy, 0, None, None) == gsr.GS_ERR_CONFIG
    assert b"NULL" in lib.gs_last_error() or len(lib.gs_last_error()) > 0
    assert lib.gs_status_string(gsr.GS_ERR_RANGE) == b"argument out of range"


def test_sizes(gsr):
    cam = gsr.Sensor(sg.mid(n=10).sensors[0])
    o = gsr.default_opts()
    assert gsr.gs_num_tiles(cam, o) == 120 * 135
    assert gsr.gs_render_workspace_bytes(10_000_000, cam, o) > gsr.gs_render_workspace_bytes(0, cam, o)
    assert gsr.gs_record_bytes(0) == 96 and gsr.gs_record_bytes(1) == 144 and gsr.gs_record_bytes(2) == 96
    offs = gsr.gs_projected_offsets(1000, 0)
    assert offs["total"] == gsr.gs_projected_bytes(1000, 0)
    assert offs["rec"] == 256 and offs["rect"] >= 256 + 96 * 1000
    assert gsr.gs_sort_workspace_bytes(1000, 10_000, cam, o) > 10_000 * 12
