"""Pins of the oracle's near-decision flags and variants, -m "not gpu".

The flags decide which rays leave the strict single-composite gate for the
variant gate, so they are pinned against things other than themselves:

  * cond_uv against the analytic Jacobian of (u,v) with respect to the ray
    angles for fronto-parallel and tilted on-axis surfels (closed form);
  * surfels placed at support rho = 9(1 +- k w), alpha = (1/255)(1 +- k w),
    hit depth = near(1 +- k w) and T(1-alpha) = t_min(1 +- k 1e-4) are
    flagged exactly when inside the window (k = 1/2), not outside (k = 2);
  * a well-conditioned interior scene flags nothing;
  * the variants of a flagged ray equal independently computed composites
    (the scene without the surfel in question; a hand composite).
"""
import math

import numpy as np
import pytest

import oracle
import scenegen as sg
from tests.helpers import scene

W0 = 2e-6   # OR_W_FLOOR (oracle.c)
C22 = 2.0 ** -22
R_ID = np.eye(3)


def _axis_cam(f=100.0):
    # pixel (16, 12) samples exactly the optical axis: d = (0, 0, 1)
    return sg.pinhole(33, 25, f, 16.5, 12.5, sg.identity_pose())


AXIS_RAY = 12 * 33 + 16


def _tilt(beta):
    """columns (t_u, t_v, n): the surfel plane tilted by beta about the y axis."""
    c, s = math.cos(beta), math.sin(beta)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


# ----------------------------------------------------------------------------- cond_uv
@pytest.mark.parametrize("su,sv,z", [(0.2, 0.2, 3.0), (0.1, 0.4, 2.0), (0.5, 0.05, 7.0)])
def test_cond_uv_fronto_parallel_closed_form(su, sv, z):
    """On axis, a fronto-parallel surfel at depth z maps ray angles (a, b) to
    (u, v) = (z tan a / s_u, z tan b / s_v): J = diag(z/s_u, z/s_v) at a = b = 0,
    so cond = max(s_u, s_v) / min(s_u, s_v)."""
    M = np.array([[su, 0, 0], [0, sv, 0], [0, 0, z]], np.float64)
    c = oracle.cond_uv(M, np.array([0.0, 0.0, 1.0]))
    assert c == pytest.approx(max(su, sv) / min(su, sv), rel=1e-6)


@pytest.mark.parametrize("beta_deg", [0.0, 30.0, 60.0, 80.0])
def test_cond_uv_tilted_closed_form(beta_deg):
    """A surfel centred on the axis at depth z, tilted by beta about y: the
    on-axis ray hits its centre; a small angle a in x moves the hit by
    z a / cos(beta) along t_u, an angle b in y by z b along t_v, so
    J = diag(z/(s_u cos beta), z/s_v) and cond is their ratio."""
    b = math.radians(beta_deg)
    su, sv, z = 0.3, 0.2, 4.0
    R = _tilt(b)
    M = np.column_stack([su * R[:, 0], sv * R[:, 1], [0.0, 0.0, z]])
    j1, j2 = z / (su * math.cos(b)), z / sv
    c = oracle.cond_uv(M, np.array([0.0, 0.0, 1.0]))
    assert c == pytest.approx(max(j1, j2) / min(j1, j2), rel=1e-5)


# ----------------------------------------------------------------------------- decision windows
def _flag_of(s, se, ray=AXIS_RAY):
    _, fl, _ = oracle.render(s, se, [ray])
    return int(fl[0])


def _window(s, se, i=0):
    """w = 2e-5 + 2^-22 cond for surfel i on the axis ray."""
    M = oracle.surfel(s, se, i)["M"]
    return W0 + C22 * oracle.cond_uv(M, np.array([0.0, 0.0, 1.0]))


@pytest.mark.parametrize("k", [-2.0, -0.5, 0.5, 2.0])
def test_support_window(k):
    """A fronto-parallel surfel whose centre sits 3 s sqrt(1+eps) off the axis:
    the axis ray meets it at rho3d = 9 (1+eps) (3D branch: rho2d is ~1800).
    Flagged SUPPORT exactly when |rho - 9| < 9 w."""
    se = _axis_cam()
    s_ = 0.2
    w = W0 + C22   # cond = 1 here (isotropic, fronto-parallel), refined below
    eps = k * w
    s = scene([dict(mu=[-3 * s_ * math.sqrt(1 + eps), 0.0, 2.0], R=R_ID, s=(s_, s_), o=0.9)])
    w = _window(s, se)
    rho = (float(s.means[0, 0]) / float(s.scales[0, 0])) ** 2   # exact in fp64 from the fp32 inputs
    inside = abs(rho - 9.0) < 9.0 * w
    assert inside == (abs(k) < 1)
    assert bool(_flag_of(s, se) & oracle.F_SUPPORT) == inside


@pytest.mark.parametrize("k", [-2.0, -0.5, 0.5, 2.0])
def test_alpha_window(k):
    """The axis ray through the centre of a fronto-parallel surfel: rho = 0,
    alpha = o = (1/255)(1+eps).  Flagged ALPHA exactly when
    |alpha - 1/255| < w/255."""
    se = _axis_cam()
    w = W0 + C22
    s = scene([dict(mu=[0.0, 0.0, 2.0], R=R_ID, s=(0.3, 0.3), o=(1 + k * w) / 255.0)])
    w = _window(s, se)
    a = float(s.opacities[0])
    inside = abs(a - 1 / 255) < w / 255
    assert inside == (abs(k) < 1)
    assert bool(_flag_of(s, se) & oracle.F_ALPHA) == inside


@pytest.mark.parametrize("k", [-2.0, -0.5, 0.5, 2.0])
def test_near_window(k):
    """A surfel tilted by 60 deg whose plane crosses the axis at t = near(1+eps)
    while its centre is at z = 0.5 (not culled).  Flagged NEAR exactly when
    |t - near| < near w."""
    se = _axis_cam()
    beta, z0, near = math.radians(60.0), 0.5, 0.2
    w = W0 + C22 * 2.0
    t = near * (1 + k * w)
    x0 = math.cos(beta) * (t - z0) / math.sin(beta)
    s = scene([dict(mu=[x0, 0.0, z0], R=_tilt(beta), s=(0.3, 0.3), o=0.9)])
    w = _window(s, se)
    nu, nv, _, _, _ = oracle.ray(se, 16, 12)
    hit = oracle.intersect(oracle.surfel(s, se, 0)["M"], nu, nv)
    t_act = hit[2][2]
    inside = abs(t_act - near) < near * w
    assert inside == (abs(k) < 1), (t_act, w)
    assert bool(_flag_of(s, se) & oracle.F_NEAR) == inside


@pytest.mark.parametrize("k", [-2.0, -0.5, 0.5, 2.0])
def test_tstop_window(k):
    """Three centred fronto-parallel surfels (rho = 0, alpha = o): T after two
    is (1-o1)(1-o2) = 0.0049; the third has 1 - o3 = t_min (1 + k 1e-4) / 0.0049, so T(1-alpha3) = t_min (1 + k 1e-4) up to fp32 rounding of o3.
    Flagged TSTOP exactly when |T(1-alpha3) - t_min| < 1e-4 t_min."""
    se = _axis_cam()
    o12 = float(np.float32(0.93))
    T2 = (1 - o12) ** 2
    o3 = 1.0 - 1e-4 * (1 + k * 1e-4) / T2
    s = scene([dict(mu=[0, 0, 2.0], R=R_ID, s=(0.5, 0.5), o=o12),
               dict(mu=[0, 0, 3.0], R=R_ID, s=(0.5, 0.5), o=o12),
               dict(mu=[0, 0, 4.0], R=R_ID, s=(0.5, 0.5), o=o3)])
    o = s.opacities.astype(np.float64)
    T2 = (1 - o[0]) * (1 - o[1])
    Tn = T2 * (1 - min(o[2], 0.99))
    inside = abs(Tn - 1e-4) < 1e-4 * 1e-4
    assert inside == (abs(k) < 1), Tn
    fl = _flag_of(s, se)
    assert bool(fl & oracle.F_TSTOP) == inside
    # outside the window the ray stops before the third surfel iff Tn < t_min
    out, _, nc = oracle.render(s, se, [AXIS_RAY])
    assert nc[0] == (2 if Tn < 1e-4 else 3)


def test_well_conditioned_interior_scene_flags_nothing():
    """Three large fronto-parallel surfels that cover the whole image with
    rho < 1 and alpha well above 1/255 and T far above t_min: no ray is near
    any decision and no intersection is ill-conditioned."""
    se = sg.pinhole(32, 24, 20.0, 16.0, 12.0, sg.identity_pose())
    s = scene([dict(mu=[0.1, -0.05, z], R=R_ID, s=(6.0, 5.0), o=o, rgb=(0.3, 0.5, 0.7))
               for z, o in ((4.0, 0.5), (6.0, 0.6), (8.0, 0.7))])
    out, fl, nc = oracle.render(s, se)
    assert np.all(nc == 3)
    assert np.all(fl == 0)
    # tilted by 30 deg: still well inside every window
    s = scene([dict(mu=[0.1, -0.05, z], R=_tilt(math.radians(30)), s=(6.0, 5.0), o=o)
               for z, o in ((4.0, 0.5), (6.0, 0.6), (8.0, 0.7))])
    _, fl, nc = oracle.render(s, se)
    assert np.all(nc == 3) and np.all(fl == 0)


# ----------------------------------------------------------------------------- variants
def test_unflagged_ray_has_one_variant_equal_to_the_render():
    se = sg.pinhole(32, 24, 20.0, 16.0, 12.0, sg.identity_pose())
    s = scene([dict(mu=[0.1, -0.05, 4.0], R=R_ID, s=(6.0, 5.0), o=0.5)])
    rays = np.arange(32 * 24)
    out, fl, _ = oracle.render(s, se, rays)
    var, nvar, seen = oracle.variants(s, se, rays)
    assert np.all(nvar == 1) and np.all(seen == 0)
    np.testing.assert_array_equal(var[:, 0], out)


def test_support_variants_are_with_and_without_the_surfel():
    """A flagged support decision: the two variants equal the renders of the
    scene with the surfel forced in (rho just inside 9) and with it removed."""
    se = _axis_cam()
    s_ = 0.2
    back = dict(mu=[0.0, 0.0, 5.0], R=R_ID, s=(2.0, 2.0), o=0.6, rgb=(0.1, 0.2, 0.3))
    edge = dict(mu=[-3 * s_ * math.sqrt(1 + 0.5 * W0), 0.0, 2.0], R=R_ID, s=(s_, s_), o=0.9,
                rgb=(0.9, 0.8, 0.7))
    s = scene([edge, back])
    _, fl, _ = oracle.render(s, se, [AXIS_RAY])
    assert fl[0] & oracle.F_SUPPORT
    var, nvar, seen = oracle.variants(s, se, [AXIS_RAY])
    assert nvar[0] == 2 and seen[0] & oracle.F_SUPPORT
    without, _, _ = oracle.render(scene([back]), se, [AXIS_RAY])
    # with: the same surfel a hair closer (rho = 9 (1 - 2w), unflagged, composited)
    inside = dict(edge, mu=[-3 * s_ * math.sqrt(1 - 3 * W0), 0.0, 2.0])
    with_, flw, ncw = oracle.render(scene([inside, back]), se, [AXIS_RAY])
    assert flw[0] == 0 and ncw[0] == 2
    got = sorted([var[0, 0], var[0, 1]], key=lambda v: v[7])
    np.testing.assert_allclose(got[0], without[0], atol=1e-15)
    # alpha differs by ~ e^-4.5 * 9 * 3.5 w: within the north_star tolerances
    np.testing.assert_allclose(got[1], with_[0], rtol=1e-4, atol=1e-5)


def test_tstop_variants_hand_composite():
    """A near-t_min stop: one variant composites the third surfel, the other
    stops before it (hand composites of the three centred surfels)."""
    se = _axis_cam()
    o3 = 0.99
    s = scene([dict(mu=[0, 0, 2.0], R=R_ID, s=(0.5, 0.5), o=0.9, rgb=(1, 0, 0)),
               dict(mu=[0, 0, 3.0], R=R_ID, s=(0.5, 0.5), o=0.9, rgb=(0, 1, 0)),
               dict(mu=[0, 0, 4.0], R=R_ID, s=(0.5, 0.5), o=o3, rgb=(0, 0, 1))])
    o = s.opacities.astype(np.float64)
    a3 = min(o[2], 0.99)
    Tn = (1 - o[0]) * (1 - o[1]) * (1 - a3)
    assert abs(Tn - 1e-4) < 1e-8          # 0.01 * 0.01 up to fp32 rounding of 0.9
    var, nvar, seen = oracle.variants(s, se, [AXIS_RAY])
    assert seen[0] & oracle.F_TSTOP and nvar[0] == 2
    w1, T1 = o[0], 1 - o[0]
    w2, T2 = o[1] * T1, T1 * (1 - o[1])
    w3 = a3 * T2
    stop = np.array([w1, w2, 0.0])
    go = np.array([w1, w2, w3])
    rgbs = sorted([var[0, k, :3] for k in range(2)], key=lambda v: v[2])
    np.testing.assert_allclose(rgbs[0], stop, atol=1e-12)
    np.testing.assert_allclose(rgbs[1], go, atol=1e-12)
