"""GPU parity on the configuration dimensions the BASELINE configs leave fixed
(-m gpu): anisotropic and off-centre pinholes, partial-azimuth / yawed /
non-uniform-beam LiDARs, a narrow fisheye, exact depth-key ties, invalid
surfels, non-default low-pass and support options, an undersized render
workspace, and bit-exact binning of the full Chunked forward frame.
Sensor models: PAPER.md:96-114 (Eqs. 3-5); tolerance protocol tests/parity.py."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import scenegen as sg  # noqa: E402
from tests import parity  # noqa: E402


@pytest.fixture(scope="module")
def gsr_mod():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_11731_b200 import gsr
    gsr.load()
    return gsr


def _render(surfels, sensor, opts=None, **kw):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    r = Renderer(to_device(surfels), gsr.default_opts(**(opts or {})))
    out = r.render(sensor, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy(), r


def _check(surfels, sensor, rays=None, gpu_opts=None, oracle_opts=None, label="", oracle_surfels=None):
    img, _ = _render(surfels, sensor, gpu_opts)
    if rays is None:
        rays = np.arange(sensor.width * sensor.height)
    os_ = oracle_surfels if oracle_surfels is not None else surfels
    ref, fl, _ = oracle.render(os_, sensor, rays, **(oracle_opts or {}))
    st = parity.compare(img, ref, fl, rays, sensor, os_, oracle_opts)
    print(label, {k: v for k, v in st.items() if k not in ("worst", "per_channel_unflagged")})
    assert st["ok"], st
    return st, img


# ---------------------------------------------------------------- cameras
def test_pinhole_fx_ne_fy_off_centre_principal_point(gsr_mod):
    """fx != fy and a principal point far from the image centre (Eq. 3 with a
    general K), full frame with ragged edge tiles."""
    rng = np.random.default_rng(101)
    s = sg.street(rng, 20_000, 1.0, 50.0, 3)
    se = sg.Sensor(sg.PINHOLE, 210, 130, sg.camera_pose([0.5, 1.5, 0.0], math.radians(8.0)),
                   fx=float(np.float32(150.0)), fy=float(np.float32(95.0)),
                   cx=float(np.float32(61.3)), cy=float(np.float32(97.8)))
    _check(s, se, label="fx!=fy")


def test_fisheye_narrow_fov_below_90_degrees(gsr_mod):
    """theta_max = 70 deg (every ray has z > 0) with a monotone KB lens,
    off-centre principal point; full frame."""
    rng = np.random.default_rng(102)
    s = sg.street(rng, 30_000, 0.0, 60.0, 3)
    th = float(np.float32(np.deg2rad(70.0)))
    k, _ = sg.draw_fisheye_k(rng, th)
    se = sg.fisheye(160, 120, th, k, 75.0, 66.0, sg.camera_pose([0, 1.5, 0], math.radians(-10.0)))
    _check(s, se, label="fisheye70")


@pytest.mark.parametrize("sigma,support", [(1.5, 9.0), (0.5, 4.0), (2.0, 16.0)])
def test_non_default_lowpass_and_support(gsr_mod, sigma, support):
    """Non-default low-pass sigma (px) and support cut rho: the pre-cull margin
    and the pixel boxes must follow them (a larger low-pass disc reaches
    further outside the image)."""
    rng = np.random.default_rng(103)
    s = sg.street(rng, 20_000, 1.0, 60.0, 1)
    s.scales[:] *= np.float32(0.2)   # many sub-pixel surfels: the low-pass branch dominates
    se = sg.pinhole(160, 100, 120.0, 80.0, 50.0, sg.camera_pose([0, 1.5, 0], 0.0))
    _check(s, se, gpu_opts=dict(lowpass_sigma_px=sigma, support_rho=support),
           oracle_opts=dict(lowpass_sigma=float(np.float32(sigma)), support_rho=float(np.float32(support))),
           label=f"lowpass{sigma}")


# ---------------------------------------------------------------- LiDAR
def _lidar(pose, elev_deg, az0, width, step):
    return sg.Sensor(sg.LIDAR, width, len(elev_deg), pose,
                     beam_elevation=np.deg2rad(np.asarray(elev_deg, np.float64)).astype(np.float32),
                     azimuth0=float(np.float32(az0)), azimuth_step=float(np.float32(step)))


@pytest.mark.parametrize("az0", [-0.7, 2.9, 3 * math.pi, -5.0])
def test_lidar_partial_azimuth_yawed_nonuniform_beams(gsr_mod, az0):
    """A 200-degree partial sweep starting at various azimuth0 (including
    values outside [-pi, pi]), a yawed sensor and a non-uniform beam table
    (denser near the horizon); full frame."""
    rng = np.random.default_rng(104)
    s = sg.street(rng, 60_000, -60.0, 60.0, 0, lidar_attrs=True, with_sh=False)
    elev = [14.0, 9.0, 5.0, 2.5, 1.0, 0.2, -0.5, -1.5, -3.0, -5.5, -9.0, -14.0, -20.0, -24.5]
    W = 300
    se = _lidar(sg.lidar_pose([0.3, 1.8, 2.0], math.radians(35.0)), elev, az0, W, math.radians(200.0) / W)
    _check(s, se, label=f"lidar-partial az0={az0}")


def test_lidar_full_turn_offset_azimuth0(gsr_mod):
    """A full turn starting at azimuth0 = 2.0 (the seam is not behind the
    sensor), yawed: full frame."""
    rng = np.random.default_rng(105)
    s = sg.street(rng, 60_000, -60.0, 60.0, 0, lidar_attrs=True, with_sh=False)
    elev = np.linspace(12.0, -22.0, 24)
    W = 360
    se = _lidar(sg.lidar_pose([0, 1.8, 0], math.radians(-70.0)), elev, 2.0, W, 2 * math.pi / W)
    _check(s, se, label="lidar-full az0=2")


# ---------------------------------------------------------------- ties and invalid inputs
def test_exact_depth_key_ties(gsr_mod):
    """Groups of surfels with identical means (bit-identical depth keys) but
    different shapes, opacities and colours: ties composite in surfel-index
    order (reading R9) -- oracle parity on the full frame, and the binning
    bit-exact against the CPU stable sort."""
    rng = np.random.default_rng(106)
    s = sg.street(rng, 12_000, 1.0, 40.0, 2)
    src = rng.choice(s.n, 3000, replace=False)
    dst = rng.choice(np.setdiff1d(np.arange(s.n), src), 3000, replace=False)
    s.means[dst] = s.means[src]
    se = sg.pinhole(200, 150, 125.0, 100.0, 75.0, sg.camera_pose([0, 1.5, 0], 0.0))
    okb, _ = oracle.keys(s, se)
    assert np.sum(okb[dst] == okb[src]) == 3000
    _check(s, se, label="ties")
    img, r = _render(s, se, keys=True)
    b = r.binning_state()
    parity.check_pinhole_binning(b, s, se, r.cam_opts.tile_w, r.cam_opts.tile_h)


@pytest.mark.parametrize("kind", ["pinhole", "lidar"])
def test_invalid_surfels_are_culled(gsr_mod, kind):
    """NaN / Inf means, NaN / zero quaternions, zero / negative / Inf / NaN
    scales and zero opacities (gsr.h: culled, not an error): the frame equals
    the oracle's render of the scene without them."""
    rng = np.random.default_rng(107)
    lid = kind == "lidar"
    s = sg.street(rng, 20_000, -40.0 if lid else 1.0, 40.0, 0 if lid else 2, lidar_attrs=lid, with_sh=not lid)
    bad = rng.choice(s.n, 1400, replace=False)
    groups = np.array_split(bad, 10)
    s.means[groups[0], 0] = np.nan
    s.means[groups[1], 2] = np.inf
    s.quats[groups[2]] = np.nan
    s.quats[groups[3]] = 0.0
    s.scales[groups[4], 0] = 0.0
    s.scales[groups[5], 1] = -0.1
    s.scales[groups[6], 0] = np.inf
    s.scales[groups[7], 1] = np.nan
    s.opacities[groups[8]] = 0.0
    s.means[groups[9]] = np.array([np.nan, np.inf, -np.inf], np.float32)
    good = np.setdiff1d(np.arange(s.n), bad)
    se = (sg.lidar64(sg.lidar_pose([0, 1.8, 0]), height=32, width=360) if lid else
          sg.pinhole(200, 150, 125.0, 100.0, 75.0, sg.camera_pose([0, 1.5, 0], 0.0)))
    _check(s, se, label=f"invalid-{kind}", oracle_surfels=s.subset(good))


# ---------------------------------------------------------------- boundary: undersized render workspace
def test_render_workspace_too_small_gives_background(gsr_mod):
    """gsr.h: the pair capacity is the largest whose workspace fits; a frame
    with more pairs renders as background (device-side check) instead of
    writing past the workspace."""
    from paper_2503_11731_b200 import gsr
    c = sg.mid(seed=11, n=20_000, width=200, height=150, f=125.0)
    se = gsr.Sensor(c.sensors[0])
    img, r = _render(c.surfels, c.sensors[0], opts=dict(split_len=256))
    assert img[7].max() > 0
    L = r._last
    P = L["cap"]
    nb = gsr.gs_render_workspace_bytes(P // 8, se, r.opts)
    buf = torch.full((nb + (1 << 20),), 7, dtype=torch.uint8, device="cuda")   # workspace + a guard band
    out = torch.full((8, se.height, se.width), -1.0, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    gsr.gs_render_camera(L["proj"], r.n, L["values"], L["ranges"], None, se, r.opts, buf[:nb],
                         out[0:3], out[3], out[4:7], out[7], st)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert np.all(o[7] == 0) and np.all(o[3] == 0) and np.all(o[:3] == 0)
    assert bool(torch.all(buf[nb:] == 7))


# ---------------------------------------------------------------- bench scale binning
@pytest.mark.slow
def test_binning_bit_exact_full_chunked_forward_frame(gsr_mod):
    """The Chunked forward camera of timestep 32 (12 M surfels, ~20 M pairs
    over 16,200 tiles with exact tile rows): the sorted pairs are a valid
    stable binning of the emitted set (tests/parity.check_sorted_pairs, tile
    ranges bit-exact), every required fp64 pair of 300 K sampled surfels is
    emitted; GPU keys equal the oracle's pinned keys."""
    from paper_2503_11731_b200.render import Renderer, to_device
    s = sg.chunked_surfels()
    se = sg.chunked_timestep_sensors(32)[0]
    r = Renderer(to_device(s))
    r.render(se, keys=True)
    torch.cuda.synchronize()
    b = r.binning_state()
    assert b["P"] > 10_000_000
    # sort validity over all pairs; conservativeness on a sample of 300 K surfels
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(s.n, 300_000, replace=False))
    st = parity.check_pinhole_binning(b, s, se, r.cam_opts.tile_w, r.cam_opts.tile_h, idx=idx)
    print("binning chunked forward", st)
    okb, cul = oracle.keys(s, se)
    vis = b["count"] > 0
    np.testing.assert_array_equal(b["key"][vis], okb[vis])
    assert not np.any(cul[vis])


# ---------------------------------------------------------------- hierarchical cull (gs_cull_bounds)
def _project_state(r, se):
    """Candidate list and per-surfel outputs of gs_project, as numpy."""
    proj, d_np = r.project(se)
    torch.cuda.synchronize()
    hdr = proj[:16].view(torch.int32).cpu().tolist()
    n_vis, n_cand = hdr[0], hdr[1]
    from paper_2503_11731_b200 import gsr
    import ctypes as C
    offs = (C.c_size_t * 5)()
    gsr.load().gs_projected_offsets(r.n, int(se.kind), offs)
    cnt = proj[offs[3]: offs[3] + 4 * r.n].view(torch.int32).cpu().numpy()
    key = proj[offs[2]: offs[2] + 4 * r.n].view(torch.int32).cpu().numpy()
    return n_vis, n_cand, int(d_np.item()), cnt, key


@pytest.mark.parametrize("case", ["street", "invalid"])
def test_block_bounds_cull_is_bitwise_the_per_surfel_cull(gsr_mod, case):
    """gs_project with gs_cull_bounds' block bounds (zone-wise
    resident sets) gives exactly the candidates, counts, keys, pair total and
    image of gs_project without them: six surround pinholes over a street of
    four 50 m zones stored zone by zone (whole blocks fall outside each
    frustum), with NaN / Inf centres and invalid scales mixed in."""
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    parts = [sg.street(np.random.default_rng(40 + c), 30_000, 50.0 * c, 50.0 * c + 50.0, 1) for c in range(4)]
    s = sg.Surfels.concat(parts)
    if case == "invalid":
        rng = np.random.default_rng(9)
        idx = rng.choice(s.n, 600, replace=False)
        s.means[idx[:100], 0] = np.nan
        s.means[idx[100:200], 2] = np.inf
        s.means[idx[200:300], 1] = -np.inf
        s.scales[idx[300:400], 0] = np.inf
        s.scales[idx[400:500], 1] = np.nan
        s.scales[idx[500:600]] = 0.0
    with_b, without = to_device(s), to_device(s, bounds=False)
    assert with_b["cull_bounds"].shape == (gsr.gs_cull_blocks(s.n), 8) and "cull_bounds" not in without
    ra, rb = Renderer(with_b), Renderer(without)
    skipped = 0
    for z in (20.0, 75.0, 130.0, 199.0):
        for yaw in sg.CHUNKED_CAM_YAWS:
            se = gsr.Sensor(sg.pinhole(320, 180, 200.0, 160.0, 90.0, sg.camera_pose([0.0, 1.5, z], math.radians(yaw))))
            a, b = _project_state(ra, se), _project_state(rb, se)
            assert a[:3] == b[:3], (z, yaw, a[:3], b[:3])
            np.testing.assert_array_equal(a[3], b[3])
            vis = b[3] > 0
            np.testing.assert_array_equal(a[4][vis], b[4][vis])
            skipped += int(b[1] < s.n // 2)
    assert skipped > 0
    se = sg.pinhole(320, 180, 200.0, 160.0, 90.0, sg.camera_pose([0.0, 1.5, 75.0], math.radians(60.0)))
    ia, ib = ra.render(se), rb.render(se)
    torch.cuda.synchronize()
    assert torch.equal(ia, ib)
    if case == "invalid":   # blocks holding an infinite centre have infinite bounds and are never skipped
        return
    # the block path is live: bounds that put every block far behind a forward camera cull everything
    fwd = gsr.Sensor(sg.pinhole(320, 180, 200.0, 160.0, 90.0, sg.camera_pose([0.0, 1.5, 75.0], 0.0)))
    assert _project_state(ra, fwd)[1] > 0
    with_b["cull_bounds"][:, 2] = -1000.0
    with_b["cull_bounds"][:, 5] = -900.0
    assert _project_state(ra, fwd)[1] == 0


# ---------------------------------------------------------------- cylindrical fisheye (Eq. 4, NEXT-4)
@pytest.mark.parametrize("hfov,yaw", [(300.0, 0.0), (200.0, 70.0), (90.0, -30.0)])
def test_cylindrical_fisheye_full_frame(gsr_mod, hfov, yaw):
    """PAPER.md Eq. 4 cylindrical camera (reading R20): full frame of a street
    scene (surfels all around the camera, behind it too) against the oracle,
    and the binning bit-exact."""
    rng = np.random.default_rng(108)
    s = sg.street(rng, 40_000, -40.0, 60.0, 2)
    se = sg.cylindrical(232, 88, np.deg2rad(hfov), np.deg2rad(100.0),
                        sg.camera_pose([0.3, 1.5, 5.0], math.radians(yaw)), cx=None, cy=40.3)
    st, img = _check(s, se, label=f"cylindrical {hfov}")
    assert img[7].mean() > 0.3
    img2, r = _render(s, se, keys=True)
    b = r.binning_state()
    ntx = (se.width + r.cam_opts.tile_w - 1) // r.cam_opts.tile_w
    vals, keys, ranges = parity.cpu_bin_sort(b["rect"], b["key"], ntx, b["ntiles"])
    np.testing.assert_array_equal(b["values"], vals)
    np.testing.assert_array_equal(b["ranges"], ranges)


def test_cylindrical_split_lists_match_unsplit(gsr_mod):
    rng = np.random.default_rng(109)
    s = sg.street(rng, 30_000, -30.0, 50.0, 1)
    se = sg.cylindrical(200, 80, np.deg2rad(270), np.deg2rad(90), sg.camera_pose([0, 1.5, 0], 0.0))
    a, _ = _render(s, se, opts=dict(split_len=2 ** 31 - 1))
    b, _ = _render(s, se, opts=dict(split_len=160))
    assert np.abs(a - b).max() < 2e-5 * max(1.0, np.abs(a).max())
