"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the oracle side (tests, bench cpu_baseline) and the
CUDA side (binding, bench).  It holds NONE of the method's arithmetic: it only
draws surfel attributes and sensor poses/intrinsics from seeded NumPy
PCG64 streams and returns plain fp32 arrays.  Both sides read the very same
fp32 arrays.

Conventions:
  * world frame: y up, z forward along the road, x lateral (x points left when
    looking down +z; right-handed);
  * camera frame (pinhole / fisheye): x right, y down, z forward (OpenCV);
  * LiDAR frame: x forward (= world z at yaw 0), y left (= world x), z up
    (= world y);
  * a sensor is given by world_to_sensor = [R | t] (3x4, fp32, row-major):
    p_sensor = R p_world + t.
  * surfel attributes: means [N,3], quats [N,4] (w,x,y,z), scales [N,2]
    (linear, post-activation), opacities [N] (post-sigmoid), sh [N,(d+1)^2,3],
    intensity [N] in [0,1], raydrop_logit [N].
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

PINHOLE = 0
FISHEYE = 1
LIDAR = 2
CYLINDRICAL = 3

SH_C0 = 0.28209479177387814  # only used to encode Tiny's uniform RGB as a DC coefficient


@dataclass
class Surfels:
    means: np.ndarray                      # [N,3] f32
    quats: np.ndarray                      # [N,4] f32 (w,x,y,z)
    scales: np.ndarray                     # [N,2] f32
    opacities: np.ndarray                  # [N] f32
    sh: Optional[np.ndarray] = None        # [N,(d+1)^2,3] f32
    sh_degree: int = 0
    intensity: Optional[np.ndarray] = None  # [N] f32
    raydrop_logit: Optional[np.ndarray] = None  # [N] f32

    @property
    def n(self) -> int:
        return int(self.means.shape[0])

    def subset(self, idx) -> "Surfels":
        g = lambda a: None if a is None else np.ascontiguousarray(a[idx])
        return Surfels(g(self.means), g(self.quats), g(self.scales), g(self.opacities),
                       g(self.sh), self.sh_degree, g(self.intensity), g(self.raydrop_logit))

    @staticmethod
    def concat(parts) -> "Surfels":
        def c(name):
            arrs = [getattr(p, name) for p in parts]
            if any(a is None for a in arrs):
                return None
            return np.ascontiguousarray(np.concatenate(arrs, axis=0))
        return Surfels(c("means"), c("quats"), c("scales"), c("opacities"), c("sh"),
                       parts[0].sh_degree, c("intensity"), c("raydrop_logit"))


@dataclass
class Sensor:
    kind: int
    width: int
    height: int
    world_to_sensor: np.ndarray            # [3,4] f32
    fx: float = 0.0
    fy: float = 0.0
    cx: float = 0.0
    cy: float = 0.0
    k: np.ndarray = field(default_factory=lambda: np.zeros(4, np.float32))  # fisheye k1..k4
    theta_max: float = 0.0                 # fisheye half-FOV (rad)
    beam_elevation: Optional[np.ndarray] = None  # LiDAR [height] f32, strictly decreasing
    azimuth0: float = 0.0
    azimuth_step: float = 0.0

    @property
    def n_rays(self) -> int:
        return self.width * self.height


@dataclass
class Config:
    name: str
    surfels: Surfels
    sensors: list                          # list[Sensor]; frames rendered from one surfel set
    info: dict = field(default_factory=dict)


# --------------------------------------------------------------------------- poses
def _f32(x):
    return np.float32(x)


def camera_pose(position, yaw_rad: float) -> np.ndarray:
    """world->camera [R|t] for a level camera at `position` looking along
    forward = (sin yaw, 0, cos yaw).  Rows: right, down, forward."""
    s, c = math.sin(yaw_rad), math.cos(yaw_rad)
    R = np.array([[-c, 0.0, s], [0.0, -1.0, 0.0], [s, 0.0, c]], dtype=np.float64)
    p = np.asarray(position, dtype=np.float64)
    t = -R @ p
    return np.concatenate([R, t[:, None]], axis=1).astype(np.float32)


def identity_pose() -> np.ndarray:
    return np.concatenate([np.eye(3), np.zeros((3, 1))], axis=1).astype(np.float32)


def lidar_pose(position, yaw_rad: float = 0.0) -> np.ndarray:
    """world->LiDAR [R|t]: x_L = forward (world z at yaw 0), y_L = left
    (world x), z_L = up (world y)."""
    s, c = math.sin(yaw_rad), math.cos(yaw_rad)
    fwd = np.array([s, 0.0, c])
    up = np.array([0.0, 1.0, 0.0])
    left = np.cross(up, fwd)  # (c,0,-s): at yaw 0 -> +x world
    R = np.stack([fwd, left, up], axis=0)
    p = np.asarray(position, dtype=np.float64)
    t = -R @ p
    return np.concatenate([R, t[:, None]], axis=1).astype(np.float32)


def pinhole(width, height, f, cx, cy, pose) -> Sensor:
    return Sensor(PINHOLE, int(width), int(height), pose, fx=float(_f32(f)), fy=float(_f32(f)),
                  cx=float(_f32(cx)), cy=float(_f32(cy)))


def lidar64(pose, height=64, width=2048, top_deg=15.0, bottom_deg=-25.0) -> Sensor:
    """64 beams evenly spaced over elevation [bottom, top] (row 0 = top),
    `width` azimuth steps over 360 deg, column j at phi_j = -pi + j*2pi/W."""
    r = np.arange(height, dtype=np.float64)
    elev = np.deg2rad(top_deg - r * (top_deg - bottom_deg) / (height - 1)).astype(np.float32)
    return Sensor(LIDAR, int(width), int(height), pose, beam_elevation=elev,
                  azimuth0=float(_f32(-math.pi)), azimuth_step=float(_f32(2.0 * math.pi / width)))


def _kb_theta_d(theta, k):
    t2 = theta * theta
    return theta * (1.0 + t2 * (k[0] + t2 * (k[1] + t2 * (k[2] + t2 * k[3]))))


def draw_fisheye_k(rng, theta_max: float, lo=-0.05, hi=0.05, max_tries=10000):
    """Draw k1..k4 ~ U(lo,hi) and reject until the equidistant (Kannala-Brandt)
    map theta -> theta_d is strictly increasing on [0, theta_max] (checked on a
    1e4-point grid) and theta_d(theta_max) > 0 (reading R12).  This is
    input validation, not part of the rendering method."""
    grid = np.linspace(0.0, theta_max, 10001)
    for tries in range(1, max_tries + 1):
        k = rng.uniform(lo, hi, 4)
        td = _kb_theta_d(grid, k)
        if td[-1] > 0 and np.all(np.diff(td) > 0):
            return k.astype(np.float32), tries
    raise RuntimeError("no monotone fisheye draw")


def fisheye(width, height, theta_max, k, cx, cy, pose) -> Sensor:
    k = np.asarray(k, np.float32)
    tdm = _kb_theta_d(np.float64(_f32(theta_max)), k.astype(np.float64))
    f = (width / 2.0) / tdm
    return Sensor(FISHEYE, int(width), int(height), pose, fx=float(_f32(f)), fy=float(_f32(f)),
                  cx=float(_f32(cx)), cy=float(_f32(cy)), k=k, theta_max=float(_f32(theta_max)))


def cylindrical(width, height, hfov, vfov, pose, cx=None, cy=None) -> Sensor:
    """Cylindrical fisheye (Eq. 4): the columns span the horizontal
    field of view hfov (f_x = W / hfov, azimuth (p_x - c_x)/f_x), the rows span
    y / sqrt(x^2 + z^2) in +-tan(vfov / 2) (f_y = (H/2) / tan(vfov/2))."""
    fx = width / hfov
    fy = (height / 2.0) / math.tan(vfov / 2.0)
    return Sensor(CYLINDRICAL, int(width), int(height), pose, fx=float(_f32(fx)), fy=float(_f32(fy)),
                  cx=float(_f32(width / 2.0 if cx is None else cx)), cy=float(_f32(height / 2.0 if cy is None else cy)))


# --------------------------------------------------------------------------- surfels
def _quat_from_frame(tu, tv, n):
    """Unit quaternion (w,x,y,z) of the rotation whose columns are (tu,tv,n)."""
    R = np.stack([tu, tv, n], axis=-1)  # [N,3,3], columns
    m00, m11, m22 = R[:, 0, 0], R[:, 1, 1], R[:, 2, 2]
    tr = m00 + m11 + m22
    q = np.empty((R.shape[0], 4))
    # Shepperd: pick the largest diagonal term for stability
    w2 = 1 + tr
    x2 = 1 + m00 - m11 - m22
    y2 = 1 - m00 + m11 - m22
    z2 = 1 - m00 - m11 + m22
    which = np.argmax(np.stack([w2, x2, y2, z2], -1), axis=-1)
    for k, s2 in enumerate([w2, x2, y2, z2]):
        sel = which == k
        if not np.any(sel):
            continue
        Rs = R[sel]
        s = np.sqrt(np.maximum(s2[sel], 1e-300)) * 2.0  # = 4*|component|
        if k == 0:
            q[sel, 0] = 0.25 * s
            q[sel, 1] = (Rs[:, 2, 1] - Rs[:, 1, 2]) / s
            q[sel, 2] = (Rs[:, 0, 2] - Rs[:, 2, 0]) / s
            q[sel, 3] = (Rs[:, 1, 0] - Rs[:, 0, 1]) / s
        elif k == 1:
            q[sel, 0] = (Rs[:, 2, 1] - Rs[:, 1, 2]) / s
            q[sel, 1] = 0.25 * s
            q[sel, 2] = (Rs[:, 0, 1] + Rs[:, 1, 0]) / s
            q[sel, 3] = (Rs[:, 0, 2] + Rs[:, 2, 0]) / s
        elif k == 2:
            q[sel, 0] = (Rs[:, 0, 2] - Rs[:, 2, 0]) / s
            q[sel, 1] = (Rs[:, 0, 1] + Rs[:, 1, 0]) / s
            q[sel, 2] = 0.25 * s
            q[sel, 3] = (Rs[:, 1, 2] + Rs[:, 2, 1]) / s
        else:
            q[sel, 0] = (Rs[:, 1, 0] - Rs[:, 0, 1]) / s
            q[sel, 1] = (Rs[:, 0, 2] + Rs[:, 2, 0]) / s
            q[sel, 2] = (Rs[:, 1, 2] + Rs[:, 2, 1]) / s
            q[sel, 3] = 0.25 * s
    q *= np.where(q[:, :1] < 0, -1.0, 1.0)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def street(rng, n: int, z0: float, z1: float, sh_degree: int = 3, lidar_attrs: bool = False,
           with_sh: bool = True) -> Surfels:
    """Synthetic street (BASELINE configs Mid/Fisheye/LiDAR/Chunked): 60% ground
    y=0, x~U[-10,10]; 40% facades x=+-8 (p=1/2), y~U[0,10]; z~U[z0,z1];
    normals tilted by U[0,15deg] about a random axis in the surface plane;
    in-plane angle U[0,2pi); scales log-U[0.02,0.5]; opacity sigmoid(N(1,1));
    SH DC ~ N(0.5,0.2), rest ~ N(0,0.2); intensity U[0,1]; drop logit N(-2,1).
    Draw order: positions, tilt, in-plane angle, scales, opacity, SH (DC then
    rest), intensity, drop logits."""
    ng = int(round(0.6 * n))
    nf = n - ng
    pos = np.empty((n, 3))
    pos[:ng, 0] = rng.uniform(-10.0, 10.0, ng)
    pos[:ng, 1] = 0.0
    pos[:ng, 2] = rng.uniform(z0, z1, ng)
    side = rng.random(nf) < 0.5
    pos[ng:, 0] = np.where(side, 8.0, -8.0)
    pos[ng:, 1] = rng.uniform(0.0, 10.0, nf)
    pos[ng:, 2] = rng.uniform(z0, z1, nf)

    base = np.zeros((n, 3))
    base[:ng, 1] = 1.0
    base[ng:, 0] = np.where(side, -1.0, 1.0)          # facing the road
    # orthonormal basis (e1,e2) of each base normal's plane
    e1 = np.zeros((n, 3))
    e1[:ng, 0] = 1.0                                   # ground: x
    e1[ng:, 2] = 1.0                                   # facade: z
    e2 = np.cross(base, e1)

    tilt = rng.uniform(0.0, np.deg2rad(15.0), n)
    beta = rng.uniform(0.0, 2.0 * np.pi, n)
    axis = np.cos(beta)[:, None] * e1 + np.sin(beta)[:, None] * e2
    nrm = base * np.cos(tilt)[:, None] + np.cross(axis, base) * np.sin(tilt)[:, None]
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    # tangent basis of the tilted normal
    f1 = e1 - np.sum(e1 * nrm, axis=1, keepdims=True) * nrm
    f1 /= np.linalg.norm(f1, axis=1, keepdims=True)
    f2 = np.cross(nrm, f1)
    ang = rng.uniform(0.0, 2.0 * np.pi, n)
    tu = np.cos(ang)[:, None] * f1 + np.sin(ang)[:, None] * f2
    tv = np.cross(nrm, tu)
    quats = _quat_from_frame(tu, tv, nrm)

    scales = np.exp(rng.uniform(np.log(0.02), np.log(0.5), (n, 2)))
    opac = 1.0 / (1.0 + np.exp(-rng.normal(1.0, 1.0, n)))
    sh = None
    if with_sh:
        nc = (sh_degree + 1) ** 2
        sh = np.empty((n, nc, 3))
        sh[:, 0, :] = rng.normal(0.5, 0.2, (n, 3))
        if nc > 1:
            sh[:, 1:, :] = rng.normal(0.0, 0.2, (n, nc - 1, 3))
    inten = drop = None
    if lidar_attrs:
        inten = rng.uniform(0.0, 1.0, n)
        drop = rng.normal(-2.0, 1.0, n)
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
    return Surfels(f(pos), f(quats), f(scales), f(opac), f(sh), sh_degree if with_sh else 0,
                   f(inten), f(drop))


def random_surfels(rng, n, lo, hi, s_lo=0.01, s_hi=0.3, sh_degree=0, lidar_attrs=True) -> Surfels:
    """Tiny-style scene: mu ~ U(lo,hi), quat = normalize(N(0,1)^4), scales
    log-U[s_lo,s_hi], opacity sigmoid(N(0,1)), RGB ~ U[0,1] encoded as the SH DC
    term (higher bands ~ N(0,0.2) when sh_degree>0); optional intensity U[0,1]
    and drop logit N(-2,1)."""
    pos = rng.uniform(lo, hi, (n, 3))
    q = rng.normal(0.0, 1.0, (n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sc = np.exp(rng.uniform(np.log(s_lo), np.log(s_hi), (n, 2)))
    op = 1.0 / (1.0 + np.exp(-rng.normal(0.0, 1.0, n)))
    rgb = rng.uniform(0.0, 1.0, (n, 3))
    nc = (sh_degree + 1) ** 2
    sh = np.zeros((n, nc, 3))
    sh[:, 0, :] = (rgb - 0.5) / SH_C0
    if nc > 1:
        sh[:, 1:, :] = rng.normal(0.0, 0.2, (n, nc - 1, 3))
    inten = drop = None
    if lidar_attrs:
        inten = rng.uniform(0.0, 1.0, n)
        drop = rng.normal(-2.0, 1.0, n)
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)
    return Surfels(f(pos), f(q), f(sc), f(op), f(sh), sh_degree, f(inten), f(drop))


# --------------------------------------------------------------------------- configs
def tiny(seed: int = 0) -> Config:
    rng = np.random.default_rng(seed)
    s = random_surfels(rng, 1000, [-2, -2, 2], [2, 2, 8], 0.01, 0.3, 0, lidar_attrs=False)
    cam = pinhole(128, 96, 100.0, 64.0, 48.0, identity_pose())
    return Config("tiny", s, [cam])


def mid(seed: int = 1, n: int = 200_000, width=1920, height=1080, f=1200.0) -> Config:
    rng = np.random.default_rng(seed)
    s = street(rng, n, 1.0, 80.0, 3)
    cam = pinhole(width, height, f, width / 2.0, height / 2.0, camera_pose([0.0, 1.5, 0.0], 0.0))
    return Config("mid", s, [cam])


def fisheye_cfg(seed: int = 2, n: int = 1_000_000, width=1920, height=1536) -> Config:
    rng = np.random.default_rng(seed)
    s = street(rng, n, 0.0, 150.0, 3)
    th = np.deg2rad(95.0)
    k, tries = draw_fisheye_k(rng, float(np.float32(th)))
    cam = fisheye(width, height, th, k, width / 2.0, height / 2.0, camera_pose([0.0, 1.5, 0.0], 0.0))
    return Config("fisheye", s, [cam], {"k": [float(x) for x in k], "f": cam.fx, "k_draws": tries})


def lidar_cfg(seed: int = 3, n: int = 2_000_000) -> Config:
    rng = np.random.default_rng(seed)
    s = street(rng, n, -200.0, 200.0, 0, lidar_attrs=True, with_sh=False)
    lid = lidar64(lidar_pose([0.0, 1.8, 0.0]))
    return Config("lidar", s, [lid])


CHUNKED_T = 64
CHUNKED_CAM_YAWS = [0, 60, 120, 180, 240, 300]


def chunked_surfels(n_chunks: int = 8, per_chunk: int = 1_500_000) -> Surfels:
    parts = []
    for c in range(n_chunks):
        rng = np.random.default_rng(100 + c)
        parts.append(street(rng, per_chunk, 50.0 * c, 50.0 * c + 50.0, 3, lidar_attrs=True))
    return Surfels.concat(parts)


def chunked_timestep_sensors(t: int, cam_w=1920, cam_h=1080, f=1200.0) -> list:
    """The 7 sensor frames of timestep t: 6 surround pinholes (yaw 0..300,
    height 1.5 m) then one LiDAR (height 1.8 m); ego at z = 168 + t."""
    z = 168.0 + t
    cams = [pinhole(cam_w, cam_h, f, cam_w / 2.0, cam_h / 2.0,
                    camera_pose([0.0, 1.5, z], math.radians(y))) for y in CHUNKED_CAM_YAWS]
    return cams + [lidar64(lidar_pose([0.0, 1.8, z]))]


def chunked(n_chunks: int = 8, per_chunk: int = 1_500_000, timesteps: int = CHUNKED_T) -> Config:
    s = chunked_surfels(n_chunks, per_chunk)
    sensors = []
    for t in range(timesteps):
        sensors += chunked_timestep_sensors(t)
    return Config("chunked", s, sensors, {"timesteps": timesteps, "frames_per_timestep": 7})


def make_config(name: str, **kw) -> Config:
    return {"tiny": tiny, "mid": mid, "fisheye": fisheye_cfg, "lidar": lidar_cfg,
            "chunked": chunked}[name](**kw)


# --------------------------------------------------------------------------- neural Gaussians (NEXT-1)
@dataclass
class Anchors:
    """Scaffold-style anchors (DESIGN.md §12 reading N1): position [n,3] f32,
    feature [n,32] f16, base_scale [n,3] f32."""
    position: np.ndarray
    feature: np.ndarray
    base_scale: np.ndarray

    @property
    def n(self) -> int:
        return int(self.position.shape[0])


NEURAL_K, NEURAL_F, NEURAL_H = 5, 32, 32
NEURAL_OUT = {"offset": 15, "scale": 10, "rotation": 30, "opacity": 5, "color": 15, "intensity": 5,
              "raydrop": 5}
NEURAL_CAMERA_HEADS = ("offset", "scale", "rotation", "opacity", "color")
NEURAL_LIDAR_HEADS = ("offset", "scale", "rotation", "opacity", "intensity", "raydrop")


def street_anchors(rng, n: int, z0: float, z1: float, s_lo=0.03, s_hi=0.2) -> Anchors:
    """Anchors on the synthetic street surfaces (positions as in `street`),
    features ~ N(0,1) stored fp16, isotropic base scale log-U[s_lo, s_hi]."""
    pos = street(rng, n, z0, z1, 0, with_sh=False).means
    feat = rng.normal(0.0, 1.0, (n, NEURAL_F)).astype(np.float16)
    l = np.exp(rng.uniform(np.log(s_lo), np.log(s_hi), n))
    base = np.repeat(l[:, None], 3, axis=1).astype(np.float32)
    return Anchors(np.ascontiguousarray(pos, np.float32), np.ascontiguousarray(feat), base)


def neural_decoder(rng, modality: str = "camera") -> dict:
    """Random-init decoder (no trained weights exist here): per head
    W1 [32,in] (in = 32 geometry heads, 35 appearance heads), W2 [32,32],
    W3 [out,32] ~ N(0, 1/fan_in) stored fp16; biases ~ N(0, 0.1) fp32, with
    the rotation head's output bias set to the identity 6D frame (1,0,0,0,1,0)
    per surfel and the opacity bias raised by 1 (mostly opaque surfels)."""
    heads = NEURAL_CAMERA_HEADS if modality == "camera" else NEURAL_LIDAR_HEADS
    dec = {}
    for h in heads:
        nin = NEURAL_F if h in ("offset", "scale", "rotation") else NEURAL_F + 3
        out = NEURAL_OUT[h]
        W1 = rng.normal(0.0, 1.0 / math.sqrt(nin), (NEURAL_H, nin))
        W2 = rng.normal(0.0, 1.0 / math.sqrt(NEURAL_H), (NEURAL_H, NEURAL_H))
        W3 = rng.normal(0.0, 0.5 / math.sqrt(NEURAL_H), (out, NEURAL_H))
        b1 = rng.normal(0.0, 0.1, NEURAL_H)
        b2 = rng.normal(0.0, 0.1, NEURAL_H)
        b3 = rng.normal(0.0, 0.1, out)
        if h == "rotation":
            b3 += np.tile([1.0, 0.0, 0.0, 0.0, 1.0, 0.0], NEURAL_K)
        if h == "opacity":
            b3 += 1.0
        dec[h] = {"W1": W1.astype(np.float16), "b1": b1.astype(np.float32), "W2": W2.astype(np.float16),
                  "b2": b2.astype(np.float32), "W3": W3.astype(np.float16), "b3": b3.astype(np.float32)}
    return dec
