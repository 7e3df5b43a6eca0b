"""GPU parity of the neural-Gaussian decode (gs_decode_anchors, NEXT-1)
against the fp64 oracle (oracle/neural.py), -m gpu.

Tolerance: the oracle's first-order error bound of the fp16 activations and
fp32 accumulation, doubled, per output element.  The
decoded surfels then go through the render path, which is held to the
strict gate of tests/parity.py against the render oracle on those surfels.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import oracle.neural as on  # noqa: E402
import scenegen as sg  # noqa: E402
from tests import parity  # noqa: E402


@pytest.fixture(scope="module")
def mod():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_11731_b200 import gsr, neural
    gsr.load()
    return neural


def _quat_to_R(q):
    """columns (t_u, t_v, n) of the rotation of unit quaternions (w,x,y,z) (test-side)."""
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y + w * z), 2 * (x * z - w * y)], -1),
        np.stack([2 * (x * y - w * z), 1 - 2 * (x * x + z * z), 2 * (y * z + w * x)], -1),
        np.stack([2 * (x * z + w * y), 2 * (y * z - w * x), 1 - 2 * (x * x + y * y)], -1)], -1)


def _decode(mod, a, dec, origin, modality):
    nd = mod.NeuralDecoder(dec, modality)
    out = nd.decode(mod.anchors_to_device(a), origin)
    torch.cuda.synchronize()
    return {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in out.items()}


def _check(g, o, modality):
    def within(name, got, want, tol):
        err = np.abs(np.asarray(got, np.float64) - want)
        bad = err > 2 * tol + 1e-7 * (1 + np.abs(want))
        assert not bad.any(), (name, int(bad.sum()), float(err.max()), float(tol.max()))
        return float(err.max())
    st = {"means": within("means", g["means"], o["means"], o["means_tol"]),
          "scales": within("scales", g["scales"], o["scales"], o["scales_tol"]),
          "opacities": within("opacities", g["opacities"], o["opacities"], o["opacities_tol"])}
    R = _quat_to_R(g["quats"].astype(np.float64))
    ferr = np.linalg.norm(R - o["frame"], axis=1)          # per column
    assert np.all(ferr <= 2 * o["frame_tol"] + 1e-6), float(ferr.max())
    assert np.all(g["quats"][:, 0] >= 0)
    if modality == "camera":
        st["sh_dc"] = within("sh", g["sh"][:, 0, :], o["sh_dc"], o["sh_dc_tol"])
    else:
        st["intensity"] = within("intensity", g["intensity"], o["intensity"], o["intensity_tol"])
        st["raydrop"] = within("raydrop", g["raydrop_logit"], o["raydrop_logit"], o["raydrop_logit_tol"])
    return st


@pytest.mark.parametrize("modality", ["camera", "lidar"])
@pytest.mark.parametrize("n", [1, 127, 129, 5000, 40_000])
def test_decode_matches_oracle(mod, modality, n):
    """Random anchors and decoder; n covers one partial tile, tile edges and
    many persistent tiles with a ragged tail."""
    rng = np.random.default_rng(300 + n)
    a = sg.street_anchors(rng, n, 0.0, 60.0)
    dec = sg.neural_decoder(rng, modality)
    origin = [0.4, 1.5, 12.0]
    g = _decode(mod, a, dec, origin, modality)
    o = on.decode(a.position, a.feature, a.base_scale, dec, origin, modality)
    st = _check(g, o, modality)
    print(modality, n, st)


def test_decode_zero_feature_identity(mod):
    """Zero features / weights / biases (rotation bias = identity 6D): centres
    at the anchors, scales = base scale, alpha = 1/2, identity frames."""
    rng = np.random.default_rng(7)
    a = sg.street_anchors(rng, 300, 0.0, 20.0)
    a.feature[:] = 0
    dec = sg.neural_decoder(rng, "camera")
    for h in dec.values():
        for k in h:
            h[k] = np.zeros_like(h[k])
    dec["rotation"]["b3"] = np.tile([1, 0, 0, 0, 1, 0], 5).astype(np.float32)
    g = _decode(mod, a, dec, [0, 0, 0], "camera")
    np.testing.assert_array_equal(g["means"], np.repeat(a.position, 5, axis=0))
    np.testing.assert_array_equal(g["scales"], np.repeat(a.base_scale[:, :2], 5, axis=0))
    np.testing.assert_array_equal(g["opacities"], 0.5)
    np.testing.assert_array_equal(g["quats"], np.tile([1, 0, 0, 0], (1500, 1)).astype(np.float32))
    np.testing.assert_array_equal(g["sh"], 0.0)


def test_decode_empty(mod):
    a = sg.Anchors(np.zeros((0, 3), np.float32), np.zeros((0, 32), np.float16), np.zeros((0, 3), np.float32))
    g = _decode(mod, a, sg.neural_decoder(np.random.default_rng(0), "camera"), [0, 0, 0], "camera")
    assert g["means"].shape == (0, 3)


@pytest.mark.parametrize("modality", ["camera", "lidar"])
def test_decoded_scene_renders_at_parity(mod, modality):
    """Anchors -> gs_decode_anchors -> gs_project -> gs_bin_sort -> render,
    all on the GPU; the frame against the render oracle on the decoded
    surfels (strict gate), full frame."""
    from paper_2503_11731_b200.render import Renderer
    rng = np.random.default_rng(8)
    a = sg.street_anchors(rng, 6000, 2.0, 40.0)
    dec = sg.neural_decoder(rng, modality)
    if modality == "camera":
        se = sg.pinhole(192, 128, 140.0, 96.0, 64.0, sg.camera_pose([0, 1.5, 0], 0.0))
    else:
        se = sg.lidar64(sg.lidar_pose([0, 1.8, 0]), height=24, width=360)
    origin = -se.world_to_sensor[:, :3].T.astype(np.float64) @ se.world_to_sensor[:, 3].astype(np.float64)
    nd = mod.NeuralDecoder(dec, modality)
    surf = nd.decode(mod.anchors_to_device(a), origin)
    img = Renderer(surf).render(se).cpu().numpy()
    host = sg.Surfels(*(surf[k].cpu().numpy() if surf[k] is not None else None
                        for k in ("means", "quats", "scales", "opacities", "sh")), 0,
                      surf["intensity"].cpu().numpy() if surf["intensity"] is not None else None,
                      surf["raydrop_logit"].cpu().numpy() if surf["raydrop_logit"] is not None else None)
    rays = np.arange(se.width * se.height)
    ref, fl, _ = oracle.render(host, se, rays)
    st = parity.compare(img, ref, fl, rays, se, host)
    assert st["ok"], st
    assert img[-1].mean() > 0.05   # the decoded scene is not empty
