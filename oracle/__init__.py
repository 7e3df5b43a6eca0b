"""CPU fp64 oracle for the 2DGS camera + LiDAR renderer.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
package (paper_2503_11731_b200) never imports it, and the two share no code:
this module defines its own ctypes structs for oracle/oracle.h.

`liboracle.so` is built from oracle.c with gcc (-O2 -fopenmp
-ffp-contract=off); see build().  Everything it computes follows DESIGN.md §2
(Eqs. 1-5; low-pass P:48; north_star compositing rule).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")

PINHOLE, FISHEYE, LIDAR, CYLINDRICAL = 0, 1, 2, 3
F_ALPHA, F_SUPPORT, F_NEAR, F_TSTOP, F_FOV, F_BRANCH, F_COND = 1, 2, 4, 8, 16, 32, 64


def build(force: bool = False) -> str:
    if force or not os.path.exists(SO) or os.path.getmtime(SO) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", SO + ".tmp", SRC, "-lm"]
        subprocess.check_call(cmd, cwd=HERE)
        os.replace(SO + ".tmp", SO)
    return SO


class _Scene(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("quats", C.c_void_p),
                ("scales", C.c_void_p), ("opacities", C.c_void_p), ("sh", C.c_void_p),
                ("sh_degree", C.c_int32), ("intensity", C.c_void_p),
                ("raydrop_logit", C.c_void_p)]


class _Sensor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("w2s", C.c_float * 12), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("k", C.c_float * 4),
                ("theta_max", C.c_float), ("beam_elevation", C.c_void_p),
                ("azimuth0", C.c_float), ("azimuth_step", C.c_float)]


class _Opts(C.Structure):
    _fields_ = [("near_", C.c_double), ("alpha_max", C.c_double), ("alpha_min", C.c_double),
                ("t_min", C.c_double), ("support_rho", C.c_double),
                ("lowpass_sigma", C.c_double), ("bg_rgb", C.c_double * 3),
                ("bg_range", C.c_double), ("bg_raydrop", C.c_double),
                ("prefilter", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        _lib.or_render.argtypes = [P(_Scene), P(_Sensor), P(_Opts), C.c_int64, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.or_render_variants.argtypes = [P(_Scene), P(_Sensor), P(_Opts), C.c_int64, C.c_void_p,
                                            C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.or_cond_uv.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_cond_uv.restype = C.c_double
        _lib.or_keys.argtypes = [P(_Scene), P(_Sensor), P(_Opts), C.c_void_p, C.c_void_p]
        _lib.or_surfel.argtypes = [P(_Scene), P(_Sensor), P(_Opts), C.c_int64, C.c_void_p]
        _lib.or_ray.argtypes = [P(_Sensor), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p]
        _lib.or_intersect.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.or_sh_basis.argtypes = [C.c_void_p, C.c_void_p]
        _lib.or_kb_theta_d.argtypes = [C.c_void_p, C.c_double]
        _lib.or_kb_theta_d.restype = C.c_double
        _lib.or_kb_inverse.argtypes = [C.c_void_p, C.c_double, C.c_double]
        _lib.or_kb_inverse.restype = C.c_double
    return _lib


DEFAULT_OPTS = dict(near=0.2, alpha_max=0.99, alpha_min=1.0 / 255.0, t_min=1e-4, support_rho=9.0,
                    lowpass_sigma=1.0 / np.sqrt(2.0), bg_rgb=(0.0, 0.0, 0.0), bg_range=0.0,
                    bg_raydrop=1.0, prefilter=1)


def _ptr(a):
    return None if a is None else a.ctypes.data


class _Keep:
    """keeps the numpy arrays behind the raw pointers alive"""

    def __init__(self):
        self.arrs = []

    def __call__(self, a, dtype=np.float32):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=dtype)
        self.arrs.append(a)
        return a.ctypes.data


def _scene(s, keep):
    return _Scene(s.n, keep(s.means), keep(s.quats), keep(s.scales), keep(s.opacities),
                  keep(s.sh), int(s.sh_degree), keep(s.intensity), keep(s.raydrop_logit))


def _sensor(se, keep):
    x = _Sensor()
    x.kind, x.width, x.height = se.kind, se.width, se.height
    x.w2s[:] = [float(v) for v in np.asarray(se.world_to_sensor, np.float32).ravel()]
    x.fx, x.fy, x.cx, x.cy = se.fx, se.fy, se.cx, se.cy
    x.k[:] = [float(v) for v in np.asarray(se.k, np.float32)]
    x.theta_max = se.theta_max
    x.beam_elevation = keep(se.beam_elevation)
    x.azimuth0, x.azimuth_step = se.azimuth0, se.azimuth_step
    return x


def _opts(**kw):
    o = dict(DEFAULT_OPTS)
    o.update(kw)
    x = _Opts()
    x.near_, x.alpha_max, x.alpha_min, x.t_min = o["near"], o["alpha_max"], o["alpha_min"], o["t_min"]
    x.support_rho, x.lowpass_sigma = o["support_rho"], o["lowpass_sigma"]
    x.bg_rgb[:] = list(o["bg_rgb"])
    x.bg_range, x.bg_raydrop, x.prefilter = o["bg_range"], o["bg_raydrop"], int(o["prefilter"])
    return x


def render(surfels, sensor, rays=None, nthreads=0, **opts):
    """Render the rays with flat index `rays` (row*width+col; None = all).
    Returns (out [n,8] f64, flags [n] u8, ncontrib [n] i32)."""
    keep = _Keep()
    sc, se, op = _scene(surfels, keep), _sensor(sensor, keep), _opts(**opts)
    if rays is None:
        n = sensor.width * sensor.height
        rp = None
    else:
        rays = np.ascontiguousarray(rays, dtype=np.int64)
        n = rays.size
        rp = rays.ctypes.data
    out = np.zeros((n, 8), np.float64)
    flags = np.zeros(n, np.uint8)
    ncon = np.zeros(n, np.int32)
    rc = lib().or_render(C.byref(sc), C.byref(se), C.byref(op), n, rp, out.ctypes.data,
                         flags.ctypes.data, ncon.ctypes.data, int(nthreads))
    if rc != 0:
        raise RuntimeError(f"or_render failed: {rc}")
    return out, flags, ncon


def variants(surfels, sensor, rays, max_var=256, nthreads=0, **opts):
    """Near-decision variants of each ray: returns
    (var [n, max_var, 8] f64, nvar [n] i32, seen [n] u8).  var[r, :nvar[r]]
    are the admissible composites (variant 0 = the nominal one); nvar[r] >
    max_var marks an unresolved ray."""
    keep = _Keep()
    sc, se, op = _scene(surfels, keep), _sensor(sensor, keep), _opts(**opts)
    rays = np.ascontiguousarray(rays, dtype=np.int64)
    n = rays.size
    var = np.zeros((n, max_var, 8), np.float64)
    nvar = np.zeros(n, np.int32)
    seen = np.zeros(n, np.uint8)
    rc = lib().or_render_variants(C.byref(sc), C.byref(se), C.byref(op), n, rays.ctypes.data,
                                  int(max_var), var.ctypes.data, nvar.ctypes.data, seen.ctypes.data,
                                  int(nthreads))
    if rc != 0:
        raise RuntimeError(f"or_render_variants failed: {rc}")
    return var, nvar, seen


def cond_uv(M, d):
    M = np.ascontiguousarray(M, np.float64)
    d = np.ascontiguousarray(d, np.float64)
    return lib().or_cond_uv(M.ctypes.data, d.ctypes.data)


def keys(surfels, sensor, **opts):
    keep = _Keep()
    sc, se, op = _scene(surfels, keep), _sensor(sensor, keep), _opts(**opts)
    kb = np.zeros(surfels.n, np.uint32)
    cul = np.zeros(surfels.n, np.uint8)
    lib().or_keys(C.byref(sc), C.byref(se), C.byref(op), kb.ctypes.data, cul.ctypes.data)
    return kb, cul.astype(bool)


def surfel(surfels, sensor, i, **opts):
    keep = _Keep()
    sc, se, op = _scene(surfels, keep), _sensor(sensor, keep), _opts(**opts)
    out = np.zeros(18, np.float64)
    culled = lib().or_surfel(C.byref(sc), C.byref(se), C.byref(op), int(i), out.ctypes.data)
    return dict(M=out[:9].reshape(3, 3), c=out[9:11], cdepth=out[11], normal=out[12:15],
                val=out[15:18], culled=bool(culled))


def ray(sensor, col, row):
    keep = _Keep()
    se = _sensor(sensor, keep)
    nu, nv, d, p = (np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(2))
    valid = lib().or_ray(C.byref(se), int(col), int(row), nu.ctypes.data, nv.ctypes.data,
                         d.ctypes.data, p.ctypes.data)
    return nu, nv, d, p, bool(valid)


def intersect(M, nu, nv):
    M = np.ascontiguousarray(M, np.float64)
    nu = np.ascontiguousarray(nu, np.float64)
    nv = np.ascontiguousarray(nv, np.float64)
    out = np.zeros(5)
    ok = lib().or_intersect(M.ctypes.data, nu.ctypes.data, nv.ctypes.data, out.ctypes.data)
    return (out[0], out[1], out[2:5]) if ok else None


def sh_basis(d):
    d = np.ascontiguousarray(d, np.float64)
    out = np.zeros(16)
    lib().or_sh_basis(d.ctypes.data, out.ctypes.data)
    return out


def kb_theta_d(k, theta):
    k = np.ascontiguousarray(k, np.float32)
    return lib().or_kb_theta_d(k.ctypes.data, float(theta))


def kb_inverse(k, theta_max, td):
    k = np.ascontiguousarray(k, np.float32)
    return lib().or_kb_inverse(k.ctypes.data, float(theta_max), float(td))


def image(out, sensor, channels=None):
    """[n_rays, 8] -> [C, H, W] for a full-frame render."""
    cam = sensor.kind != LIDAR
    C_ = 8 if cam else 4
    return out[:, :C_].T.reshape(C_, sensor.height, sensor.width)
