"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what pins it: a value printed in the paper (golden fixture),
a closed form, a textbook identity, a library routine, an invariant, or an
independent formulation (oracle/naive.py) on small inputs.
"""
import math

import numpy as np
import pytest

import oracle
import oracle.naive as naive
import scenegen as sg
from tests.helpers import (empty_scene, golden, random_small_scene, scene, small_lidar,
                           small_pinhole)

R_ID = np.eye(3)
R_XN = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])  # t_u=y, t_v=z, n=x


# ------------------------------------------------------------------ planes (Eqs. 3, 5)
def test_eq5_lidar_planes_paper_value():
    """PAPER value: Eq. 5 at theta = phi = 0 (golden/eq5_lidar_planes.json)."""
    g = golden("eq5_lidar_planes.json")
    se = sg.Sensor(sg.LIDAR, 4, 1, sg.identity_pose(), beam_elevation=np.array([0.0], np.float32),
                   azimuth0=0.0, azimuth_step=float(np.float32(0.5)))
    nu, nv, d, _, ok = oracle.ray(se, 0, 0)
    assert ok
    np.testing.assert_array_equal(nu, np.array(g["h_u"][:3]))
    np.testing.assert_array_equal(nv, np.array(g["h_v"][:3]))
    assert g["h_u"][3] == 0 and g["h_v"][3] == 0  # planes through the sensor origin
    np.testing.assert_allclose(d, [1, 0, 0], atol=0)


def test_eq4_cylindrical_planes_paper_value():
    """PAPER value: Eq. 4's h_u = (cos phi, 0, -sin phi, 0) at phi = 0 and
    phi = pi/2, and h_v at the principal row (golden/eq4_cylindrical_planes.json)."""
    g = golden("eq4_cylindrical_planes.json")
    se = sg.cylindrical(33, 25, np.deg2rad(120), np.deg2rad(60), sg.identity_pose(), cx=16.5, cy=12.5)
    nu, nv, d, p, ok = oracle.ray(se, 16, 12)
    assert ok and p[0] == 16.5 and p[1] == 12.5
    np.testing.assert_array_equal(nu, g["h_u_phi0"][:3])
    np.testing.assert_array_equal(nv, g["h_v_centre"][:3])
    np.testing.assert_allclose(d, [0, 0, 1], atol=0)
    # a column a quarter turn to the right: phi = pi/2
    se2 = sg.Sensor(sg.CYLINDRICAL, 33, 25, sg.identity_pose(), fx=1.0, fy=1.0,
                    cx=float(np.float32(16.5 - np.pi / 2)), cy=12.5)
    nu, nv, d, _, _ = oracle.ray(se2, 16, 12)
    np.testing.assert_allclose(nu, g["h_u_phi_half_pi"][:3], atol=1e-6)
    np.testing.assert_allclose(d, [1, 0, 0], atol=1e-6)


def test_eq3_pinhole_planes_paper_value():
    """Eq. 3 at the principal point (golden/eq3_pinhole_planes.json)."""
    g = golden("eq3_pinhole_planes.json")
    se = sg.pinhole(33, 25, 20.0, 16.5, 12.5, sg.identity_pose())
    nu, nv, d, p, ok = oracle.ray(se, 16, 12)
    assert ok and p[0] == 16.5 and p[1] == 12.5
    np.testing.assert_array_equal(nu, g["h_u"][:3])
    np.testing.assert_array_equal(nv, g["h_v"][:3])


def _sensors_for_planes():
    rng = np.random.default_rng(7)
    k, _ = sg.draw_fisheye_k(rng, float(np.float32(np.deg2rad(95))))
    return [sg.pinhole(64, 48, 40.0, 30.0, 26.0, sg.identity_pose()),
            sg.fisheye(64, 48, np.deg2rad(95), k, 32.0, 24.0, sg.identity_pose()),
            small_lidar(16, 128, 15.0, -25.0),
            sg.cylindrical(96, 40, np.deg2rad(300), np.deg2rad(100), sg.identity_pose(), cx=41.0, cy=17.0)]


@pytest.mark.parametrize("si", [0, 1, 2, 3])
def test_plane_pairs_contain_the_ray(si):
    """Closed form: both planes contain the ray (n.d = 0) and n_u x n_v || d;
    the pinhole/LiDAR direction reprojects to the sample coordinate."""
    se = _sensors_for_planes()[si]
    rng = np.random.default_rng(si)
    for _ in range(300):
        col, row = int(rng.integers(se.width)), int(rng.integers(se.height))
        nu, nv, d, p, ok = oracle.ray(se, col, row)
        if not ok:
            continue
        assert abs(nu @ d) < 1e-12 and abs(nv @ d) < 1e-12
        cr = np.cross(nu, nv)
        dn = d / np.linalg.norm(d)
        assert np.linalg.norm(np.cross(cr / np.linalg.norm(cr), dn)) < 1e-12
        if se.kind == sg.PINHOLE:  # reproject d through K
            assert abs(se.fx * d[0] / d[2] + se.cx - p[0]) < 1e-9
            assert abs(se.fy * d[1] / d[2] + se.cy - p[1]) < 1e-9
        elif se.kind == sg.CYLINDRICAL:  # Eq. 4: azimuth about y, height over the y-axis distance
            assert abs(se.cx + se.fx * math.atan2(d[0], d[2]) - p[0]) < 1e-9
            assert abs(se.cy + se.fy * d[1] / math.hypot(d[0], d[2]) - p[1]) < 1e-9
            assert abs(np.linalg.norm(d) - 1.0) < 1e-14
        elif se.kind == sg.LIDAR:  # elevation / azimuth of d (reading R5: theta = elevation)
            assert abs(math.asin(d[2]) - float(se.beam_elevation[row])) < 1e-12
            ph = se.azimuth0 + col * se.azimuth_step
            assert abs(math.remainder(math.atan2(d[1], d[0]) - ph, 2 * math.pi)) < 1e-12
        else:  # fisheye: equidistant KB forward projection of d recovers the pixel
            th = math.acos(max(-1.0, min(1.0, d[2])))
            td = oracle.kb_theta_d(se.k, th)
            rxy = math.hypot(d[0], d[1])
            if rxy > 1e-12:
                assert abs(se.cx + se.fx * td * d[0] / rxy - p[0]) < 1e-7
                assert abs(se.cy + se.fy * td * d[1] / rxy - p[1]) < 1e-7


def test_unified_scheme_plane_choice_invariance():
    """Invariant: (u,v) does not depend on which two distinct planes
    through the ray are used."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        M = rng.normal(size=(3, 3))
        M[:, 2] = rng.normal(size=3) * 5
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        a = np.cross(d, rng.normal(size=3)); a /= np.linalg.norm(a)
        b = np.cross(d, a)
        r1 = oracle.intersect(M, a, b)
        A = rng.normal(size=(2, 2))
        r2 = oracle.intersect(M, A[0, 0] * a + A[0, 1] * b, A[1, 0] * a + A[1, 1] * b)
        assert r1 is not None and r2 is not None
        assert abs(r1[0] - r2[0]) < 1e-9 * (1 + abs(r1[0])) and abs(r1[1] - r2[1]) < 1e-9 * (1 + abs(r1[1]))


# ------------------------------------------------------------------ Eq. 2 intersection
def test_intersection_closed_forms():
    """Closed form: a splat centred on the ray and
    perpendicular to it -> (0,0); shifted by s_u along t_u -> (-1,0)."""
    d = np.array([0.0, 0.0, 1.0])
    nu, nv = np.array([-1.0, 0, 0]), np.array([0.0, -1.0, 0])  # Eq. 3 at the principal point
    su, sv, z = 0.3, 0.2, 5.0
    M = np.array([[su, 0, 0.0], [0, sv, 0.0], [0, 0, z]])
    u, v, P = oracle.intersect(M, nu, nv)
    assert (u, v) == (0.0, 0.0) and np.allclose(P, [0, 0, z], atol=0)
    M2 = M.copy(); M2[0, 2] = su  # centre moved by s_u along t_u
    u, v, P = oracle.intersect(M2, nu, nv)
    assert abs(u + 1.0) < 1e-15 and abs(v) < 1e-15 and np.allclose(P, [0, 0, z], atol=1e-15)


def test_intersection_vs_dense_least_squares():
    """Independent formulation: the hit P = M(u,v,1) lies on both planes
    (relative residual <= 1e-9) and equals a dense solve of
    u a + v b - t d = -mu."""
    rng = np.random.default_rng(11)
    for _ in range(1000):
        M = rng.normal(size=(3, 3))
        M[:, 2] = rng.normal(size=3) * 10
        d = rng.normal(size=3); d /= np.linalg.norm(d)
        a = np.cross(d, [0.3, 0.5, 0.8]); a /= np.linalg.norm(a)
        b = np.cross(d, a)
        u, v, P = oracle.intersect(M, a, b)
        scale = np.linalg.norm(P) + 1e-300
        assert abs(a @ P) <= 1e-9 * scale and abs(b @ P) <= 1e-9 * scale
        sol = np.linalg.solve(np.stack([M[:, 0], M[:, 1], -d], 1), -M[:, 2])
        assert np.allclose([u, v], sol[:2], rtol=1e-6, atol=1e-9)
        assert np.allclose(P, sol[2] * d, rtol=1e-6, atol=1e-9)


# ------------------------------------------------------------------ SH
def test_sh_basis_matches_scipy_and_addition_theorem():
    """Library routine: the hand-written basis equals sqrt2*Im/Re of scipy's
    complex Y_l^m (Condon-Shortley phase); addition theorem per band."""
    rng = np.random.default_rng(0)
    dirs = rng.normal(size=(200, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    ref = naive.sh_basis_scipy(dirs, 3)
    for i, d in enumerate(dirs):
        Y = oracle.sh_basis(d)
        np.testing.assert_allclose(Y, ref[i], atol=1e-13)
        for l in range(4):
            band = Y[l * l:(l + 1) ** 2]
            assert abs(np.sum(band ** 2) - (2 * l + 1) / (4 * math.pi)) < 1e-13
    # special directions pin the signs: Y_1 = C1*(-y, z, -x)
    C1 = math.sqrt(3) / (2 * math.sqrt(math.pi))
    np.testing.assert_allclose(oracle.sh_basis([0, 1, 0])[1:4], [-C1, 0, 0], atol=1e-15)
    np.testing.assert_allclose(oracle.sh_basis([1, 0, 0])[1:4], [0, 0, -C1], atol=1e-15)
    np.testing.assert_allclose(oracle.sh_basis([0, 0, 1])[1:4], [0, C1, 0], atol=1e-15)


# ------------------------------------------------------------------ single-surfel closed forms
def _one_surfel_cam(o=0.7, s=(0.5, 0.5), rgb=(0.2, 0.6, 0.9)):
    # f = 16, c = (16,12): pixel (20,10) has xh = 4.5/16, yh = -1.5/16 (exact)
    se = sg.pinhole(32, 24, 16.0, 16.0, 12.0, sg.identity_pose())
    mu = [4.0 * 4.5 / 16.0, 4.0 * -1.5 / 16.0, 4.0]
    return se, scene([dict(mu=mu, R=R_ID, s=s, o=o, rgb=rgb)])


def test_single_surfel_centre_pixel():
    """north_star closed form: centre pixel alpha = min(0.99, o), rgb = alpha*c,
    depth = plane depth, normal faces the camera."""
    for o in (0.7, 0.999):
        se, s = _one_surfel_cam(o=o)
        out, fl, nc = oracle.render(s, se, [10 * 32 + 20])
        a = min(0.99, float(np.float32(o)))
        np.testing.assert_allclose(out[0, 7], a, atol=1e-15)
        np.testing.assert_allclose(out[0, :3], a * np.array([0.2, 0.6, 0.9], np.float32), atol=1e-7)
        np.testing.assert_allclose(out[0, 3], 4.0, rtol=1e-14)
        np.testing.assert_allclose(out[0, 4:7], [0, 0, -a], atol=1e-15)
        assert nc[0] == 1 and fl[0] == 0


def test_single_surfel_off_centre_hand_solved():
    """Closed form: one pixel right of the centre the ray hits the plane z=4
    0.25 m along t_u: u = 0.25/s_u, rho3d = u^2 < rho2d = 2."""
    se, s = _one_surfel_cam(o=0.7, s=(0.5, 0.5))
    out, _, _ = oracle.render(s, se, [10 * 32 + 21])
    o = float(np.float32(0.7))
    np.testing.assert_allclose(out[0, 7], o * math.exp(-0.5 * 0.25), rtol=1e-14)
    np.testing.assert_allclose(out[0, 3], 4.0, rtol=1e-14)


def test_lowpass_branch_for_small_surfel():
    """2DGS low-pass (sigma = 1/sqrt2 px): a 1 cm surfel at 4 m is
    sub-pixel; 1 px from the centre rho = min(rho3d=625, rho2d=2) = 2,
    2 px -> 8, 3 px -> 18 > 9 (no contribution).  Depth = centre depth."""
    se, s = _one_surfel_cam(o=0.6, s=(0.01, 0.01))
    o = float(np.float32(0.6))
    out, _, nc = oracle.render(s, se, [10 * 32 + 21, 10 * 32 + 22, 10 * 32 + 23])
    np.testing.assert_allclose(out[:, 7], [o * math.exp(-1), o * math.exp(-4), 0.0], rtol=1e-13, atol=0)
    np.testing.assert_allclose(out[:2, 3], 4.0, rtol=1e-14)
    assert out[2, 3] == 0.0


def test_fronto_parallel_surfel_exact_depth():
    """north_star: a fronto-parallel surfel gives the exact plane depth at
    every covered pixel, whichever branch wins."""
    se = small_pinhole(32, 24, 16.0)
    s = scene([dict(mu=[0.25, -0.125, 3.0], R=R_ID, s=(0.4, 0.15), o=0.9)])
    out, _, _ = oracle.render(s, se)
    cov = out[:, 7] > 0
    assert cov.sum() > 20
    np.testing.assert_allclose(out[cov, 3], 3.0, rtol=1e-14)


def test_empty_scene_background():
    """Special case: no surfels -> background (rgb 0, alpha 0, depth 0;
    LiDAR range 0, intensity 0, raydrop 1)."""
    out, fl, nc = oracle.render(empty_scene(), small_pinhole())
    assert np.all(out == 0) and np.all(nc == 0)
    out, _, _ = oracle.render(empty_scene(), small_lidar())
    assert np.all(out[:, [0, 1, 3]] == 0) and np.all(out[:, 2] == 1.0)
    out, _, _ = oracle.render(empty_scene(), small_pinhole(), bg_rgb=(0.1, 0.2, 0.3))
    np.testing.assert_allclose(out[:, :3], np.tile([0.1, 0.2, 0.3], (out.shape[0], 1)), atol=0)


def test_two_surfel_hand_composite():
    """Hand composite (golden/two_surfel_composite.json)."""
    g = golden("two_surfel_composite.json")
    se = sg.pinhole(16, 16, 16.0, 8.5, 8.5, sg.identity_pose())   # pixel (8,8) on the axis
    s = scene([dict(mu=[0, 0, g["back"]["z"]], R=R_ID, s=(1, 1), o=g["back"]["opacity"], rgb=g["back"]["rgb"]),
               dict(mu=[0, 0, g["front"]["z"]], R=R_ID, s=(1, 1), o=g["front"]["opacity"], rgb=g["front"]["rgb"])])
    out, _, nc = oracle.render(s, se, [8 * 16 + 8])
    np.testing.assert_allclose(out[0, :3], g["rgb"], atol=1e-15)
    np.testing.assert_allclose(out[0, 7], g["alpha"], atol=1e-15)
    np.testing.assert_allclose(out[0, 3], g["depth"], rtol=1e-14)
    assert nc[0] == 2


def test_compositing_recurrence_textbook_identity():
    """Textbook identity: with termination off, the T-recurrence
    equals sum_i alpha_i c_i prod_{j<i}(1-alpha_j) for a stack of
    axis-centred fronto-parallel surfels (alpha_i = min(0.99, o_i))."""
    rng = np.random.default_rng(4)
    se = sg.pinhole(16, 16, 16.0, 8.5, 8.5, sg.identity_pose())
    zs = rng.uniform(1, 9, 12)
    os_ = rng.uniform(0.05, 0.995, 12)
    cols = rng.uniform(0, 1, (12, 3))
    s = scene([dict(mu=[0, 0, z], R=R_ID, s=(1, 1), o=o, rgb=c) for z, o, c in zip(zs, os_, cols)])
    out, _, _ = oracle.render(s, se, [8 * 16 + 8], t_min=0.0)
    order = np.argsort(zs)
    a = np.minimum(0.99, os_.astype(np.float32).astype(np.float64))[order]
    c = s.sh[order, 0, :].astype(np.float64) * sg.SH_C0 + 0.5
    trans = np.concatenate([[1.0], np.cumprod(1 - a)[:-1]])
    np.testing.assert_allclose(out[0, :3], (a * trans) @ c, atol=1e-14)
    np.testing.assert_allclose(out[0, 7], 1 - np.prod(1 - a), atol=1e-14)


def test_early_termination_rule():
    """Reading R3: the surfel whose T(1-alpha) would drop below 1e-4 is not
    composited and the ray stops: 0.99, 0.98 composited (T=2e-4), 0.9 stops."""
    se = sg.pinhole(16, 16, 16.0, 8.5, 8.5, sg.identity_pose())
    s = scene([dict(mu=[0, 0, 2.0], R=R_ID, s=(1, 1), o=0.995, rgb=[1, 0, 0]),
               dict(mu=[0, 0, 3.0], R=R_ID, s=(1, 1), o=0.98, rgb=[0, 1, 0]),
               dict(mu=[0, 0, 4.0], R=R_ID, s=(1, 1), o=0.9, rgb=[0, 0, 1])])
    out, _, nc = oracle.render(s, se, [8 * 16 + 8])
    a2 = float(np.float32(0.98))
    assert nc[0] == 2
    np.testing.assert_allclose(out[0, 7], 1 - 0.01 * (1 - a2), atol=1e-15)
    assert out[0, 2] == 0.0


def test_transmittance_bounds_random_scenes():
    """Invariant (north_star): 0 <= alpha <= 1 - t_min; colour bounded by the
    largest surfel colour; with t_min = 0, adding a surfel behind every other
    one never lowers alpha.  (With t_min > 0 that last property fails: see
    test_early_termination_counterexample.)"""
    se = small_pinhole(24, 16, 14.0)
    for seed in range(4):
        s = random_small_scene(seed, 30)
        out, _, _ = oracle.render(s, se)
        assert np.all(out[:, 7] >= 0) and np.all(out[:, 7] <= 1 - 1e-4 + 1e-15)
        out0, _, _ = oracle.render(s, se, t_min=0.0)
        back = scene([dict(mu=[0, 0, 50.0], R=R_ID, s=(40, 40), o=0.5)])
        s2 = sg.Surfels.concat([s, sg.Surfels(back.means, back.quats, back.scales, back.opacities,
                                              np.zeros((1, 4, 3), np.float32), 1, back.intensity,
                                              back.raydrop_logit)])
        out1, _, _ = oracle.render(s2, se, t_min=0.0)
        assert np.all(out1[:, 7] >= out0[:, 7] - 1e-15)


def test_early_termination_counterexample():
    """with t_min = 1e-4 inserting a faint surfel can LOWER alpha:
    T=0.0101 then A (0.99) -> 0.999899; inserting 0.02 before A makes A cross the
    threshold -> 0.990102."""
    se = sg.pinhole(16, 16, 16.0, 8.5, 8.5, sg.identity_pose())
    pre = [dict(mu=[0, 0, 1.0], R=R_ID, s=(1, 1), o=0.9899, rgb=[1, 1, 1])]   # T = 0.0101
    A = dict(mu=[0, 0, 5.0], R=R_ID, s=(1, 1), o=0.99, rgb=[1, 1, 1])
    faint = dict(mu=[0, 0, 3.0], R=R_ID, s=(1, 1), o=0.02, rgb=[1, 1, 1])
    a0 = float(np.float32(0.9899))
    o1, _, _ = oracle.render(scene(pre + [A]), se, [8 * 16 + 8])
    o2, _, _ = oracle.render(scene(pre + [A, faint]), se, [8 * 16 + 8])
    T0 = 1 - a0
    assert abs(o1[0, 7] - (1 - T0 * 0.01)) < 1e-12
    assert abs(o2[0, 7] - (1 - T0 * (1 - float(np.float32(0.02))))) < 1e-12
    assert o2[0, 7] < o1[0, 7]


# ------------------------------------------------------------------ sensors
def test_lidar_single_opaque_perpendicular_surfel():
    """Closed form: range = plane distance; intensity = alpha r;
    raydrop = alpha p + (1-alpha)*1."""
    se = sg.Sensor(sg.LIDAR, 64, 3, sg.identity_pose(),
                   beam_elevation=np.array([0.1, 0.0, -0.1], np.float32), azimuth0=0.0,
                   azimuth_step=float(np.float32(2 * math.pi / 64)))
    s = scene([dict(mu=[17.25, 0, 0], R=R_XN, s=(0.5, 0.5), o=0.95, intensity=0.6, drop_logit=0.0)])
    out, _, nc = oracle.render(s, se, [1 * 64 + 0])
    a = float(np.float32(0.95))
    np.testing.assert_allclose(out[0, 0], 17.25, rtol=1e-15)
    np.testing.assert_allclose(out[0, 1], a * float(np.float32(0.6)), atol=1e-15)
    np.testing.assert_allclose(out[0, 2], a * 0.5 + (1 - a), atol=1e-15)
    np.testing.assert_allclose(out[0, 3], a, atol=1e-15)


def test_fisheye_k0_is_equidistant():
    """Closed form: k = 0 -> r_d = f theta exactly; near the axis the fisheye
    ray approaches the pinhole ray with the same f (difference O(theta^3))."""
    k0 = np.zeros(4, np.float32)
    se = sg.fisheye(200, 200, np.deg2rad(95), k0, 100.0, 100.0, sg.identity_pose())
    f = se.fx
    for col, row in [(150, 100), (100, 30), (199, 199), (101, 100)]:
        nu, nv, d, p, ok = oracle.ray(se, col, row)
        r = math.hypot(p[0] - 100, p[1] - 100)
        th = math.acos(d[2])
        if ok:
            assert abs(th - r / f) < 1e-13
    pin = sg.pinhole(200, 200, f, 100.0, 100.0, sg.identity_pose())
    _, _, d1, _, _ = oracle.ray(se, 102, 101)
    _, _, d2, _, _ = oracle.ray(pin, 102, 101)
    d2 = d2 / np.linalg.norm(d2)
    th = math.acos(d1[2])
    assert np.linalg.norm(d1 - d2) < th ** 3


def test_fisheye_roundtrip_and_fov():
    """Closed form: theta -> theta_d -> theta round trip; samples beyond
    theta_max are invalid (background, alpha 0)."""
    rng = np.random.default_rng(2)
    k, _ = sg.draw_fisheye_k(rng, float(np.float32(np.deg2rad(95))))
    tm = float(np.float32(np.deg2rad(95)))
    for th in np.linspace(0, tm, 50):
        assert abs(oracle.kb_inverse(k, tm, oracle.kb_theta_d(k, th)) - th) < 1e-12
    se = sg.fisheye(64, 48, np.deg2rad(95), k, 32.0, 24.0, sg.identity_pose())
    s = scene([dict(mu=[0, 0, 3.0], R=R_ID, s=(50, 50), o=0.9)])
    out, _, _ = oracle.render(s, se)
    valid = np.array([oracle.ray(se, i % 64, i // 64)[4] for i in range(64 * 48)])
    yy, xx = np.divmod(np.arange(64 * 48), 64)
    rd = np.hypot((xx + 0.5 - 32.0) / se.fx, (yy + 0.5 - 24.0) / se.fy)
    np.testing.assert_array_equal(~valid, rd > oracle.kb_theta_d(k, tm))
    assert (~valid).sum() > 0
    assert np.all(out[~valid, 7] == 0) and np.all(out[valid & (rd < 1.0), 7] > 0)


# ------------------------------------------------------------------ invariants
def test_rigid_invariance():
    """Invariant: moving scene and sensor jointly by an exactly
    representable rigid motion (integer translation + cyclic axis
    permutation, quaternion (1/2,1/2,1/2,1/2)) leaves the image unchanged."""
    se = small_pinhole(24, 18, 14.0)
    s = random_small_scene(9, 30)
    out0, fl0, _ = oracle.render(s, se)
    P = np.array([[0.0, 0, 1], [1, 0, 0], [0, 1, 0]])  # x->y, y->z, z->x
    tr = np.array([3.0, -2.0, 5.0])
    mu2 = (s.means.astype(np.float64) @ P.T + tr).astype(np.float32)
    qr = np.array([0.5, 0.5, 0.5, 0.5])  # quaternion of P
    q = s.quats.astype(np.float64)
    w1, x1, y1, z1 = qr
    w2, x2, y2, z2 = q.T
    q2 = np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2, w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                   w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2, w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], 1)
    W = np.asarray(se.world_to_sensor, np.float64)
    R2 = W[:, :3] @ P.T
    t2 = W[:, 3] - R2 @ tr
    se2 = sg.pinhole(24, 18, 14.0, 12.0, 9.0, np.concatenate([R2, t2[:, None]], 1).astype(np.float32))
    s2 = sg.Surfels(mu2, q2.astype(np.float32), s.scales, s.opacities, s.sh, s.sh_degree,
                    s.intensity, s.raydrop_logit)
    # SH coefficients are world-frame: rotate the view direction back by using
    # degree-0 colour only for this check
    s.sh[:, 1:, :] = 0
    s2.sh[:, 1:, :] = 0
    out0, fl0, _ = oracle.render(s, se)
    out1, fl1, _ = oracle.render(s2, se2)
    ok = (fl0 == 0) & (fl1 == 0)
    assert np.abs(out0[ok] - out1[ok]).max() < 1e-5


def test_permutation_invariance():
    """Invariant: shuffling surfels (no exact key ties) leaves the
    output bit-identical."""
    se = small_pinhole(24, 18, 14.0)
    s = random_small_scene(5, 40)
    perm = np.random.default_rng(0).permutation(s.n)
    a, _, _ = oracle.render(s, se)
    b, _, _ = oracle.render(s.subset(perm), se)
    np.testing.assert_array_equal(a, b)


def test_prefilter_is_result_neutral():
    """The bounding prefilter only skips surfels that cannot contribute."""
    c = sg.tiny()
    a, fa, _ = oracle.render(c.surfels, c.sensors[0], prefilter=1)
    b, fb, _ = oracle.render(c.surfels, c.sensors[0], prefilter=0)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(fa, fb)
    s = random_small_scene(1, 60, lo=(-5, -5, -5), hi=(5, 5, 5))
    for se in _sensors_for_planes():
        a, _, _ = oracle.render(s, se, prefilter=1)
        b, _, _ = oracle.render(s, se, prefilter=0)
        np.testing.assert_array_equal(a, b)


def test_culling_behind_near_plane():
    """Reading R18: surfels whose centre depth is below near never contribute,
    even if large."""
    se = small_pinhole(16, 16, 10.0)
    s = scene([dict(mu=[0, 0, 0.1], R=R_ID, s=(5, 5), o=0.99)])
    out, _, _ = oracle.render(s, se)
    assert np.all(out[:, 7] == 0)


# ------------------------------------------------------------------ brute force, 2 formulations
def test_tiny_matches_naive_full_frame():
    """Brute force: oracle == naive (different intersection, SH and fisheye
    formulations) on the full Tiny frame."""
    c = sg.tiny()
    rays = np.arange(0, c.sensors[0].n_rays, 3)
    a, _, _ = oracle.render(c.surfels, c.sensors[0], rays)
    b = naive.render(c.surfels, c.sensors[0], rays)
    assert np.abs(a - b).max() < 1e-10


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_small_scenes_all_sensors_match_naive(seed):
    """Brute force on random <=32-surfel scenes, 16x16-ish rays, 3 sensors."""
    rng = np.random.default_rng(100 + seed)
    s = sg.random_surfels(rng, 32, [-4, -4, -4], [4, 4, 4], 0.05, 0.9, sh_degree=3, lidar_attrs=True)
    k, _ = sg.draw_fisheye_k(rng, float(np.float32(np.deg2rad(95))))
    for se in [sg.pinhole(16, 16, 10.0, 8.0, 8.0, sg.identity_pose()),
               sg.fisheye(16, 16, np.deg2rad(95), k, 8.0, 8.0, sg.identity_pose()),
               small_lidar(16, 32, 30.0, -30.0),
               sg.cylindrical(24, 12, np.deg2rad(330), np.deg2rad(110), sg.identity_pose())]:
        a, _, _ = oracle.render(s, se)
        b = naive.render(s, se)
        assert np.abs(a - b).max() < 1e-10


def test_keys_pinned_formula_and_order():
    """Reading R9: keys are fp32(pinned fp64 expression); naive.py evaluates
    the same expression with numpy (no FMA) -> identical bits."""
    c = sg.tiny()
    kb, cul = oracle.keys(c.surfels, c.sensors[0])
    P = naive._prep(c.surfels, c.sensors[0], dict(naive.DEFAULTS))
    np.testing.assert_array_equal(kb, P["key"].view(np.uint32))
    np.testing.assert_array_equal(cul, P["culled"])
