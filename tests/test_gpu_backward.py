"""Backward pass of the compositing (NEXT-2, gs_render_backward), -m gpu.

Oracle: central finite differences of the fp64 render oracle (the plain
definition of the derivative; SPEC S:212-213 asks for 1e-3 relative) of
    L = sum_{c, p} G[c, p] * out[c, p]
for random G, every attribute of every surfel.  With smooth options
(support 50, alpha_min 0, t_min 0: no decision has a jump above 1e-10) every
gradient entry is compared; with the north_star options only the entries
whose central difference crosses no decision (the composited count of every
ray is the same at +h and -h) are.  The depth output D / (1 - T) jumps where
a pair switches between the rho3d and rho2d branches (reading R8: hit depth
vs centre depth) and is ill-conditioned where alpha is tiny, so the depth
channel is differentiated separately: large near-fronto-parallel surfels
(the 3D branch always wins) and only samples with alpha > 0.05."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import scenegen as sg  # noqa: E402

SMOOTH = dict(support_rho=50.0, alpha_min=0.0, t_min=0.0)


@pytest.fixture(scope="module")
def gsr_mod():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_11731_b200 import gsr
    gsr.load()
    return gsr


def _gpu_grad(s, se, G, opts):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    gpu_o = dict(opts)
    if "support_rho" in gpu_o:
        gpu_o["support_rho"] = float(gpu_o["support_rho"])
    r = Renderer(to_device(s), gsr.default_opts(split_len=2 ** 31 - 1, **gpu_o))
    img = r.render(se)
    g = r.backward(torch.from_numpy(G.astype(np.float32)).cuda())
    torch.cuda.synchronize()
    return img.cpu().numpy(), {k: (v.cpu().numpy().astype(np.float64) if v is not None else None) for k, v in g.items()}


def _loss(s, se, G, opts):
    out, _, nc = oracle.render(s, se, **opts)
    C = 8 if se.kind != oracle.LIDAR else 4
    return float(np.sum(out[:, :C].T.reshape(G.shape) * G)), nc


def _fd(s, se, G, opts, fields, rel=1e-3):
    """Central differences of L for every component of the listed fields,
    at steps h and h/4.  Returns {field: (fd at h/4, valid mask)}; valid =
    no ray's composited count changes between the evaluations and the two
    steps agree to 5e-4 (a step straddling a kink of the definition, e.g.
    the rho3d / rho2d switch, gives step-dependent differences)."""
    res = {}
    for name in fields:
        arr = getattr(s, name)
        fds = []
        ok = np.ones(arr.shape, bool)
        flat = arr.reshape(-1)
        for div in (1.0, 4.0):
            fd = np.zeros(arr.shape, np.float64)
            for k in range(flat.size):
                v0 = flat[k]
                h = rel / div * max(abs(float(v0)), 0.05)
                vp, vm = np.float32(v0 + h), np.float32(v0 - h)
                flat[k] = vp
                lp, ncp = _loss(s, se, G, opts)
                flat[k] = vm
                lm, ncm = _loss(s, se, G, opts)
                flat[k] = v0
                fd.reshape(-1)[k] = (lp - lm) / (float(vp) - float(vm))
                ok.reshape(-1)[k] &= bool(np.array_equal(ncp, ncm))
            fds.append(fd)
        scale = max(np.abs(fds[1]).max(), 1e-12)
        ok &= np.abs(fds[0] - fds[1]) <= 5e-4 * np.abs(fds[1]) + 1e-4 * scale
        res[name] = (fds[1], ok)
    return res


def _compare(gpu, fd, ok, name, rtol=2e-3):
    scale = max(np.abs(fd).max(), 1e-12)
    err = np.abs(gpu - fd)
    bad = ok & (err > rtol * np.abs(fd) + 2e-4 * scale)
    assert not bad.any(), (name, int(bad.sum()), float(err[bad].max()), float(scale),
                           np.argwhere(bad)[:5].tolist(), gpu[bad][:5].tolist(), fd[bad][:5].tolist())
    return float((err[ok] / scale).max()) if ok.any() else 0.0


def _scene(seed, n=10, sh_degree=1):
    rng = np.random.default_rng(seed)
    s = sg.random_surfels(rng, n, [-1.2, -0.9, 3.0], [1.2, 0.9, 6.0], 0.15, 0.6, sh_degree=sh_degree)
    s.opacities[:] = np.clip(s.opacities, 0.2, 0.85)
    return s


@pytest.mark.parametrize("sh_degree", [0, 1, 3])
def test_pinhole_gradients_match_finite_differences(gsr_mod, sh_degree):
    s = _scene(200 + sh_degree, sh_degree=sh_degree)
    se = sg.pinhole(32, 24, 20.0, 16.0, 12.0, sg.identity_pose())
    G = np.random.default_rng(7).normal(size=(8, 24, 32))
    G[3] = 0.0   # depth: test_pinhole_depth_gradient
    img, g = _gpu_grad(s, se, G, SMOOTH)
    fd = _fd(s, se, G, SMOOTH, ["means", "quats", "scales", "opacities", "sh"])
    worst = {k: _compare(g[k].reshape(fd[k][0].shape), fd[k][0], fd[k][1], k) for k in fd}
    frac = np.mean(np.concatenate([fd[k][1].ravel() for k in fd]))
    print("pinhole", sh_degree, worst, "compared", frac)
    assert frac > 0.75   # the rest: steps that straddle a kink (rho3d / rho2d switch) or a cut


def test_pinhole_gradients_posed_camera_north_star_options(gsr_mod):
    """A yawed, translated camera and the north_star cut-offs: entries whose
    difference crosses no decision."""
    s = _scene(210, n=14, sh_degree=2)
    s.means[:, 0] += 1.0
    se = sg.pinhole(40, 28, 24.0, 19.5, 14.5, sg.camera_pose([1.0, 0.2, -0.5], np.deg2rad(8.0)))
    G = np.random.default_rng(8).normal(size=(8, 28, 40))
    G[3] = 0.0
    _, g = _gpu_grad(s, se, G, {})
    fd = _fd(s, se, G, {}, ["means", "quats", "scales", "opacities"])
    frac = np.mean(np.concatenate([fd[k][1].ravel() for k in fd]))
    assert frac > 0.5
    for k in fd:
        _compare(g[k].reshape(fd[k][0].shape), fd[k][0], fd[k][1], k)


def test_pinhole_depth_gradient(gsr_mod):
    """Depth-only loss on samples with alpha > 0.05; large surfels tilted by
    at most 30 degrees, so the 3D branch wins everywhere near them."""
    rng = np.random.default_rng(240)
    n = 8
    surfs = []
    for _ in range(n):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        ang = rng.uniform(0, np.deg2rad(30))
        K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
        R = np.eye(3) + np.sin(ang) * K + (1 - np.cos(ang)) * K @ K
        surfs.append(dict(mu=rng.uniform([-0.8, -0.6, 3.0], [0.8, 0.6, 5.0]), R=R,
                          s=tuple(rng.uniform(0.35, 0.6, 2)), o=float(rng.uniform(0.3, 0.8)),
                          rgb=rng.uniform(0, 1, 3)))
    from tests.helpers import scene
    s = scene(surfs)
    se = sg.pinhole(32, 24, 20.0, 16.0, 12.0, sg.identity_pose())
    out, _, _ = oracle.render(s, se, **SMOOTH)
    G = np.zeros((8, 24, 32))
    G[3] = np.random.default_rng(10).normal(size=(24, 32)) * (out[:, 7].reshape(24, 32) > 0.05)
    _, g = _gpu_grad(s, se, G, SMOOTH)
    fd = _fd(s, se, G, SMOOTH, ["means", "quats", "scales", "opacities"])
    for k in fd:
        _compare(g[k].reshape(fd[k][0].shape), fd[k][0], fd[k][1], k)


def test_lidar_gradients_match_finite_differences(gsr_mod):
    rng = np.random.default_rng(220)
    s = sg.random_surfels(rng, 12, [3.0, -1.5, -0.6], [6.0, 1.5, 0.6], 0.15, 0.5, sh_degree=0, lidar_attrs=True)
    s.opacities[:] = np.clip(s.opacities, 0.2, 0.85)
    se = sg.Sensor(sg.LIDAR, 48, 10, sg.identity_pose(),
                   beam_elevation=np.deg2rad(np.linspace(9.0, -9.0, 10)).astype(np.float32),
                   azimuth0=float(np.float32(-0.6)), azimuth_step=float(np.float32(1.2 / 48)))
    G = np.random.default_rng(9).normal(size=(4, 10, 48))
    out, _, _ = oracle.render(s, se, **SMOOTH)
    G[0] *= out[:, 3].reshape(10, 48) > 0.05   # range = D / (1 - T): only well-conditioned samples
    _, g = _gpu_grad(s, se, G, SMOOTH)
    fd = _fd(s, se, G, SMOOTH, ["means", "quats", "scales", "opacities", "intensity", "raydrop_logit"])
    for k in fd:
        _compare(g[k].reshape(fd[k][0].shape), fd[k][0], fd[k][1], k)


def test_backward_rejects_fisheye(gsr_mod):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    s = _scene(230)
    k, _ = sg.draw_fisheye_k(np.random.default_rng(0), float(np.float32(np.deg2rad(95))))
    se = sg.fisheye(32, 24, np.deg2rad(95), k, 16.0, 12.0, sg.identity_pose())
    r = Renderer(to_device(s))
    r.render(se)
    with pytest.raises(gsr.GsError) as e:
        r.backward(torch.zeros((8, 24, 32), device="cuda"))
    assert e.value.status == gsr.GS_ERR_UNSUPPORTED
