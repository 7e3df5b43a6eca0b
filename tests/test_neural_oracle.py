"""Pins of the neural-Gaussian decode oracle (oracle/neural.py, NEXT-1), -m "not gpu".

  * zero-feature / zero-weight identity case (SPEC decode_anchor example):
    centres at the anchor, alpha = sigmoid(0) = 1/2, scales = base scale,
    colour 1/2, the rotation bias's identity frame;
  * geometry heads ignore the view direction (opposite view origins give the
    same centres, scales and frames; colour may differ);
  * a hand-solved closed form through identity layers;
  * the numpy layers against an explicit-loop dense layer (brute force);
  * Gram-Schmidt frames are orthonormal and right-handed;
  * the error bound holds for an fp16/fp32 emulation of the GPU arithmetic.
"""
import math

import numpy as np
import pytest

import oracle.neural as nn
import scenegen as sg


def _zero_decoder(modality):
    dec = {}
    for h in nn.heads_of(modality):
        out = nn.OUT_DIM[h]
        dec[h] = {"W1": np.zeros((32, nn.in_dim(h)), np.float16), "b1": np.zeros(32, np.float32),
                  "W2": np.zeros((32, 32), np.float16), "b2": np.zeros(32, np.float32),
                  "W3": np.zeros((out, 32), np.float16), "b3": np.zeros(out, np.float32)}
    dec["rotation"]["b3"] = np.tile([1, 0, 0, 0, 1, 0], nn.K).astype(np.float32)
    return dec


@pytest.mark.parametrize("modality", ["camera", "lidar"])
def test_zero_feature_identity(modality):
    rng = np.random.default_rng(1)
    a = sg.street_anchors(rng, 7, 0.0, 20.0)
    a.feature[:] = 0
    o = nn.decode(a.position, a.feature, a.base_scale, _zero_decoder(modality), [0, 1.5, 0], modality)
    np.testing.assert_array_equal(o["means"], np.repeat(a.position.astype(np.float64), nn.K, axis=0))
    np.testing.assert_array_equal(o["scales"], np.repeat(a.base_scale[:, :2].astype(np.float64), nn.K, axis=0))
    np.testing.assert_array_equal(o["opacities"], 0.5)
    np.testing.assert_array_equal(o["frame"], np.broadcast_to(np.eye(3), (7 * nn.K, 3, 3)))
    if modality == "camera":
        np.testing.assert_array_equal(o["sh_dc"], 0.0)      # colour 1/2
    else:
        np.testing.assert_array_equal(o["intensity"], 0.5)
        np.testing.assert_array_equal(o["raydrop_logit"], 0.0)


def test_geometry_ignores_view_direction():
    rng = np.random.default_rng(2)
    a = sg.street_anchors(rng, 50, 0.0, 30.0)
    dec = sg.neural_decoder(rng, "camera")
    p = nn.decode(a.position, a.feature, a.base_scale, dec, [0, 1.5, -100.0])
    q = nn.decode(a.position, a.feature, a.base_scale, dec, [0, 1.5, 200.0])
    for k in ("means", "scales", "frame"):
        np.testing.assert_array_equal(p[k], q[k])
    assert np.abs(p["sh_dc"] - q["sh_dc"]).max() > 1e-3
    assert np.abs(p["opacities"] - q["opacities"]).max() > 1e-3


def test_closed_form_through_identity_layers():
    """W1 = W2 = I (geometry heads), W3 selecting hidden units 0..14: for
    positive features O = f[0:15], so mu_j = x + f[3j:3j+3] * l (hand solved)."""
    rng = np.random.default_rng(3)
    a = sg.street_anchors(rng, 4, 0.0, 10.0)
    a.feature[:] = np.abs(a.feature)
    dec = _zero_decoder("camera")
    eye = np.eye(32, dtype=np.float16)
    dec["offset"]["W1"], dec["offset"]["W2"] = eye, eye
    W3 = np.zeros((15, 32), np.float16)
    W3[np.arange(15), np.arange(15)] = 1
    dec["offset"]["W3"] = W3
    o = nn.decode(a.position, a.feature, a.base_scale, dec, [0, 0, 0])
    f = a.feature.astype(np.float64)
    for i in range(4):
        for j in range(nn.K):
            want = a.position[i].astype(np.float64) + f[i, 3 * j:3 * j + 3] * a.base_scale[i].astype(np.float64)
            np.testing.assert_array_equal(o["means"][nn.K * i + j], want)


def test_numpy_layers_match_explicit_loops():
    rng = np.random.default_rng(4)
    dec = sg.neural_decoder(rng, "lidar")
    x = rng.normal(0, 1, 35)
    for h in ("opacity", "raydrop"):
        p = dec[h]
        h1 = [max(v, 0.0) for v in nn.dense_loop(x, p["W1"].astype(np.float64), p["b1"])]
        h2 = [max(v, 0.0) for v in nn.dense_loop(h1, p["W2"].astype(np.float64), p["b2"])]
        z3 = nn.dense_loop(h2, p["W3"].astype(np.float64), p["b3"])
        got, _ = nn._mlp(x[None, :], np.zeros((1, 35)), p)
        np.testing.assert_allclose(got[0], z3, rtol=1e-12, atol=1e-12)


def test_frames_orthonormal_right_handed():
    rng = np.random.default_rng(5)
    a = sg.street_anchors(rng, 200, 0.0, 30.0)
    o = nn.decode(a.position, a.feature, a.base_scale, sg.neural_decoder(rng, "camera"), [0, 1.5, 0])
    R = o["frame"]
    np.testing.assert_allclose(np.einsum("nij,nik->njk", R, R), np.broadcast_to(np.eye(3), R.shape), atol=1e-12)
    np.testing.assert_allclose(np.linalg.det(R), 1.0, atol=1e-12)


def _emulate_gpu(a, dec, origin, modality):
    """fp16 view direction and hidden activations, fp32 accumulation: an
    emulation of the kernel's arithmetic (test-side, not the oracle)."""
    x = a.position.astype(np.float32)
    v = x - np.asarray(origin, np.float32)
    d = (v / np.sqrt((v * v).sum(1, keepdims=True))).astype(np.float16)
    out = {}
    for h in nn.heads_of(modality):
        p = dec[h]
        inp = a.feature if h in nn.GEOMETRY else np.concatenate([a.feature, d], 1)
        z = inp.astype(np.float32) @ p["W1"].astype(np.float32).T + p["b1"]
        z = np.maximum(z, 0).astype(np.float16).astype(np.float32) @ p["W2"].astype(np.float32).T + p["b2"]
        z = np.maximum(z, 0).astype(np.float16).astype(np.float32) @ p["W3"].astype(np.float32).T + p["b3"]
        out[h] = z.astype(np.float64)
    return out


def test_error_bound_covers_fp16_emulation():
    rng = np.random.default_rng(6)
    a = sg.street_anchors(rng, 3000, 0.0, 60.0)
    dec = sg.neural_decoder(rng, "camera")
    origin = [0.3, 1.5, 10.0]
    o = nn.decode(a.position, a.feature, a.base_scale, dec, origin)
    em = _emulate_gpu(a, dec, origin, "camera")
    x = a.position.astype(np.float64)
    l = a.base_scale.astype(np.float64)
    mu = (x[:, None, :] + em["offset"].reshape(-1, nn.K, 3) * l[:, None, :]).reshape(-1, 3)
    assert np.all(np.abs(mu - o["means"]) <= o["means_tol"])
    al = (1 / (1 + np.exp(-em["opacity"]))).reshape(-1)
    assert np.all(np.abs(al - o["opacities"]) <= o["opacities_tol"])
    dc = ((1 / (1 + np.exp(-em["color"]))).reshape(-1, 3) - 0.5) / nn.C0
    assert np.all(np.abs(dc - o["sh_dc"]) <= o["sh_dc_tol"])
    # the bound is a worst case (|W| propagation) but not vacuous: within ~300x of the typical error
    assert np.median(o["opacities_tol"]) < 300 * max(np.median(np.abs(al - o["opacities"])), 1e-7)
