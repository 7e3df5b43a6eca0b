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


def test_host_validation_round2(gsr):
    """Checks added in round 2: a non-monotone or non-finite fisheye lens,
    oversized images (u16 pixel boxes), a non-finite azimuth0 (GS_ERR_RANGE)."""
    th = float(np.float32(np.deg2rad(95)))
    good = sg.fisheye(64, 48, th, np.zeros(4, np.float32), 32, 24, sg.identity_pose())
    assert _call_project(gsr, gsr.Sensor(good)) != gsr.GS_ERR_RANGE
    bad = sg.fisheye(64, 48, th, np.array([-0.45, 0.08, 0.0, 0.0], np.float32), 32, 24, sg.identity_pose())
    k = bad.k.astype(np.float64)
    t = np.linspace(0, th, 10001)
    td = t * (1 + k[0] * t ** 2 + k[1] * t ** 4 + k[2] * t ** 6 + k[3] * t ** 8)
    assert not np.all(np.diff(td) > 0)            # indeed not monotone on [0, theta_max]
    assert _call_project(gsr, gsr.Sensor(bad)) == gsr.GS_ERR_RANGE
    assert b"monotone" in gsr.load().gs_last_error()
    nan = sg.fisheye(64, 48, th, np.array([np.nan, 0, 0, 0], np.float32), 32, 24, sg.identity_pose())
    assert _call_project(gsr, gsr.Sensor(nan)) == gsr.GS_ERR_RANGE
    big = sg.pinhole(70000, 10, 100.0, 5, 5, sg.identity_pose())
    assert _call_project(gsr, gsr.Sensor(big)) == gsr.GS_ERR_RANGE
    wide = sg.lidar64(sg.lidar_pose([0, 0, 0]), height=8, width=40000)
    assert _call_project(gsr, gsr.Sensor(wide)) == gsr.GS_ERR_RANGE
    az = sg.lidar64(sg.lidar_pose([0, 0, 0]), height=8, width=64)
    az.azimuth0 = float("nan")
    assert _call_project(gsr, gsr.Sensor(az)) == gsr.GS_ERR_RANGE


def test_decode_anchors_validation(gsr):
    """gs_decode_anchors host checks: NULL structs, unknown modality, NULL
    weights or outputs, misaligned features; n = 0 launches nothing."""
    lib = gsr.load()
    an = gsr.gs_anchors()
    de = gsr.gs_decoder()
    o3 = (C.c_float * 3)(0, 0, 0)
    d = C.c_void_p(16)
    assert lib.gs_decode_anchors(None, C.byref(de), o3, d, d, d, d, d, None, None, None) == gsr.GS_ERR_CONFIG
    an.n = 0
    assert lib.gs_decode_anchors(C.byref(an), C.byref(de), o3, None, None, None, None, None, None, None,
                                 None) == gsr.GS_OK
    de.modality = 7
    assert lib.gs_decode_anchors(C.byref(an), C.byref(de), o3, d, d, d, d, d, None, None, None) == gsr.GS_ERR_CONFIG
    de.modality = gsr.GS_DECODE_CAMERA
    an.n, an.position, an.feature, an.base_scale = 10, 16, 16, 16
    assert lib.gs_decode_anchors(C.byref(an), C.byref(de), o3, d, d, d, d, d, None, None, None) == gsr.GS_ERR_CONFIG
    assert b"weight" in lib.gs_last_error()
    for h in range(6):
        m = de.head[h]
        m.w1 = m.b1 = m.w2 = m.b2 = m.w3 = m.b3 = 16
    an.feature = 18   # misaligned
    assert lib.gs_decode_anchors(C.byref(an), C.byref(de), o3, d, d, d, d, d, None, None, None) == gsr.GS_ERR_CONFIG
    an.feature = 16
    assert lib.gs_decode_anchors(C.byref(an), C.byref(de), o3, d, d, d, d, None, None, None, None) == gsr.GS_ERR_CONFIG
    de.modality = gsr.GS_DECODE_LIDAR
    assert lib.gs_decode_anchors(C.byref(an), C.byref(de), o3, d, d, d, d, None, d, None, None) == gsr.GS_ERR_CONFIG


def test_decode_kernel_uses_tcgen05():
    """The decode kernel's SASS issues 5th-gen tensor-core MMAs (UTCHMMA) and
    reads tensor memory (LDTM)."""
    import subprocess
    from paper_2503_11731_b200 import build
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build.SO],
                          capture_output=True, text=True).stdout
    funcs = sass.split("Function : ")
    dec = [f for f in funcs if f.startswith("_ZN3gsr3dec8k_decode")]
    assert len(dec) == 2   # camera and LiDAR instantiations
    assert all("UTCHMMA" in f and "LDTM" in f for f in dec)


def test_cull_bounds_validation():
    """gs_cull_bounds / gs_cull_blocks (hierarchical cull): argument
    checks run before any launch, and the binding refuses block bounds that
    cannot describe the surfel arrays they travel with."""
    import torch
    from paper_2503_11731_b200 import gsr
    lib = gsr.load()
    assert gsr.gs_cull_blocks(0) == 0 and gsr.gs_cull_blocks(1) == 1
    assert gsr.gs_cull_blocks(2048) == 1 and gsr.gs_cull_blocks(2049) == 2
    sf = gsr.gs_surfels()
    assert lib.gs_cull_bounds(None, None, None) == gsr.GS_ERR_CONFIG
    sf.n = -1
    assert lib.gs_cull_bounds(C.byref(sf), None, None) == gsr.GS_ERR_RANGE
    sf.n = 0
    assert lib.gs_cull_bounds(C.byref(sf), None, None) == gsr.GS_OK     # nothing to do
    sf.n = 10
    assert lib.gs_cull_bounds(C.byref(sf), None, None) == gsr.GS_ERR_CONFIG
    sf.means, sf.scales = 16, 20                                          # scales misaligned
    assert lib.gs_cull_bounds(C.byref(sf), C.c_void_p(32), None) == gsr.GS_ERR_CONFIG
    sf.scales = 24
    assert lib.gs_cull_bounds(C.byref(sf), C.c_void_p(40), None) == gsr.GS_ERR_CONFIG   # bounds misaligned
    t = dict(means=torch.zeros(5000, 3), quats=torch.zeros(5000, 4), scales=torch.zeros(5000, 2),
             opacities=torch.zeros(5000), cull_bounds=torch.zeros(3, 8))
    assert gsr.surfels_struct(t).cull_bounds is not None
    for bad in (torch.zeros(2, 8), torch.zeros(3, 7), torch.zeros(24)):
        t["cull_bounds"] = bad
        with pytest.raises(ValueError):
            gsr.surfels_struct(t)
    del t["cull_bounds"]
    assert gsr.surfels_struct(t).cull_bounds is None
