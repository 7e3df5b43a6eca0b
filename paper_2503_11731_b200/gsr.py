"""ctypes binding of include/gsr.h (argument marshalling only).

Same names as the C-ABI.  Every step of the path runs inside libgsr.so's
CUDA kernels; this module converts Python objects (torch CUDA tensors,
scenegen.Sensor-like objects) into the C structs and raises GsError on a
non-OK status.  There is no CPU fallback: if libgsr.so cannot be loaded the
import of load() raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import build as _build

GS_OK, GS_ERR_CONFIG, GS_ERR_RANGE, GS_ERR_CAPACITY, GS_ERR_CUDA, GS_ERR_UNSUPPORTED = range(6)
GS_PINHOLE, GS_FISHEYE_EQUIDISTANT, GS_LIDAR_SPINNING = 0, 1, 2
GS_MAX_BEAMS = 256


class GsError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{msg} (status {status})")
        self.status = status


class gs_surfels(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("quats", C.c_void_p),
                ("scales", C.c_void_p), ("opacities", C.c_void_p), ("sh", C.c_void_p),
                ("sh_degree", C.c_int32), ("intensity", C.c_void_p),
                ("raydrop_logit", C.c_void_p), ("cull_bounds", C.c_void_p)]


class gs_sensor(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("height", C.c_int32),
                ("world_to_sensor", C.c_float * 12), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("k", C.c_float * 4),
                ("theta_max", C.c_float), ("beam_elevation", C.c_void_p),
                ("azimuth0", C.c_float), ("azimuth_step", C.c_float)]


class gs_opts(C.Structure):
    _fields_ = [("tile_w", C.c_int32), ("tile_h", C.c_int32), ("split_len", C.c_int32),
                ("near_plane", C.c_float),
                ("alpha_max", C.c_float), ("alpha_min", C.c_float), ("t_min", C.c_float),
                ("support_rho", C.c_float), ("lowpass_sigma_px", C.c_float),
                ("bg_rgb", C.c_float * 3), ("bg_range", C.c_float), ("bg_raydrop", C.c_float),
                ("grid_share", C.c_float)]


GS_DECODE_CAMERA, GS_DECODE_LIDAR = 0, 1
GS_NEURAL_K, GS_NEURAL_F, GS_NEURAL_HIDDEN = 5, 32, 32


class gs_anchors(C.Structure):
    _fields_ = [("n", C.c_int64), ("position", C.c_void_p), ("feature", C.c_void_p),
                ("base_scale", C.c_void_p)]


class gs_mlp(C.Structure):
    _fields_ = [("w1", C.c_void_p), ("b1", C.c_void_p), ("w2", C.c_void_p), ("b2", C.c_void_p),
                ("w3", C.c_void_p), ("b3", C.c_void_p)]


class gs_decoder(C.Structure):
    _fields_ = [("modality", C.c_int32), ("head", gs_mlp * 6)]


EXPORTS = ["gs_default_opts", "gs_decode_anchors", "gs_backward_workspace_bytes", "gs_render_backward", "gs_band_route_workspace_bytes", "gs_band_route",
           "gs_payload_floats", "gs_pack_surfels", "gs_unpack_surfels", "gs_projected_bytes", "gs_sort_workspace_bytes", "gs_num_tiles", "gs_projected_offsets",
           "gs_project", "gs_bin_sort", "gs_render_camera", "gs_render_lidar",
           "gs_status_string", "gs_last_error", "gs_record_bytes", "gs_render_workspace_bytes",
           "gs_kernel_launches", "gs_cull_blocks", "gs_cull_bounds"]

_lib = None


def load(build_if_missing: bool = True):
    """Load libgsr.so (building it in-tree with nvcc if absent or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    so = _build.SO
    if os.environ.get("GSR_DEV_LIB"):   # dev sweeps only: an alternative in-tree build
        so = os.environ["GSR_DEV_LIB"]
    elif build_if_missing:
        so = _build.build()
    if not os.path.exists(so):
        raise ImportError(f"libgsr.so not found at {so}; run paper_2503_11731_b200/build.py")
    lib = C.CDLL(so)
    P, vp = C.POINTER, C.c_void_p
    lib.gs_default_opts.argtypes = [P(gs_opts)]
    lib.gs_default_opts.restype = None
    lib.gs_projected_bytes.argtypes = [C.c_int64, C.c_int32]
    lib.gs_projected_bytes.restype = C.c_size_t
    lib.gs_sort_workspace_bytes.argtypes = [C.c_int64, C.c_int64, P(gs_sensor), P(gs_opts)]
    lib.gs_sort_workspace_bytes.restype = C.c_size_t
    lib.gs_num_tiles.argtypes = [P(gs_sensor), P(gs_opts)]
    lib.gs_num_tiles.restype = C.c_int64
    lib.gs_record_bytes.argtypes = [C.c_int32]
    lib.gs_record_bytes.restype = C.c_int32
    lib.gs_project.argtypes = [P(gs_surfels), P(gs_sensor), P(gs_opts), vp, C.c_size_t, vp, vp]
    lib.gs_project.restype = C.c_int
    lib.gs_bin_sort.argtypes = [vp, C.c_int64, P(gs_sensor), P(gs_opts), vp, vp, C.c_int64, vp, vp,
                                C.c_size_t, vp, vp]
    lib.gs_bin_sort.restype = C.c_int
    lib.gs_render_workspace_bytes.argtypes = [C.c_int64, P(gs_sensor), P(gs_opts)]
    lib.gs_render_workspace_bytes.restype = C.c_size_t
    lib.gs_render_camera.argtypes = [vp, C.c_int64, vp, vp, vp, P(gs_sensor), P(gs_opts), vp,
                                     C.c_size_t, vp, vp, vp, vp, vp, vp]
    lib.gs_render_camera.restype = C.c_int
    lib.gs_render_lidar.argtypes = [vp, C.c_int64, vp, vp, vp, P(gs_sensor), P(gs_opts), vp,
                                    C.c_size_t, vp, vp, vp, vp, vp, vp]
    lib.gs_render_lidar.restype = C.c_int
    lib.gs_projected_offsets.argtypes = [C.c_int64, C.c_int32, vp]
    lib.gs_projected_offsets.restype = None
    lib.gs_status_string.argtypes = [C.c_int]
    lib.gs_status_string.restype = C.c_char_p
    lib.gs_last_error.argtypes = []
    lib.gs_last_error.restype = C.c_char_p
    lib.gs_decode_anchors.argtypes = [P(gs_anchors), P(gs_decoder), vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.gs_decode_anchors.restype = C.c_int
    lib.gs_band_route_workspace_bytes.argtypes = [C.c_int64, C.c_int32]
    lib.gs_band_route_workspace_bytes.restype = C.c_size_t
    lib.gs_band_route.argtypes = [vp, C.c_int64, P(gs_sensor), P(gs_opts), vp, C.c_int32, vp, vp, vp, C.c_size_t, vp]
    lib.gs_band_route.restype = C.c_int
    lib.gs_payload_floats.argtypes = [C.c_int32, C.c_int32, C.c_int32]
    lib.gs_payload_floats.restype = C.c_int32
    lib.gs_pack_surfels.argtypes = [P(gs_surfels), vp, C.c_int64, vp, vp]
    lib.gs_pack_surfels.restype = C.c_int
    lib.gs_unpack_surfels.argtypes = [vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.gs_unpack_surfels.restype = C.c_int
    lib.gs_backward_workspace_bytes.argtypes = [C.c_int64]
    lib.gs_backward_workspace_bytes.restype = C.c_size_t
    lib.gs_render_backward.argtypes = [P(gs_surfels), P(gs_sensor), P(gs_opts), vp, vp, vp, vp, vp, C.c_size_t,
                                       vp, vp, vp, vp, vp, vp, vp, vp]
    lib.gs_render_backward.restype = C.c_int
    lib.gs_cull_blocks.argtypes = [C.c_int64]
    lib.gs_cull_blocks.restype = C.c_int64
    lib.gs_cull_bounds.argtypes = [P(gs_surfels), vp, vp]
    lib.gs_cull_bounds.restype = C.c_int
    lib.gs_kernel_launches.argtypes = []
    lib.gs_kernel_launches.restype = C.c_uint64
    _lib = lib
    return lib


def _check(status):
    if status != GS_OK:
        lib = load()
        raise GsError(status, f"{lib.gs_status_string(status).decode()}: {lib.gs_last_error().decode()}")


def _ptr(t):
    """data pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


# ---------------------------------------------------------------- struct builders
def default_opts(**overrides) -> gs_opts:
    o = gs_opts()
    load().gs_default_opts(C.byref(o))
    for k, v in overrides.items():
        if k == "bg_rgb":
            o.bg_rgb[:] = [float(x) for x in v]
        else:
            setattr(o, k, v)
    return o


class Sensor:
    """gs_sensor plus the host beam table it points to."""

    def __init__(self, s):
        self.kind, self.width, self.height = int(s.kind), int(s.width), int(s.height)
        st = gs_sensor()
        st.kind, st.width, st.height = self.kind, self.width, self.height
        st.world_to_sensor[:] = [float(x) for x in np.asarray(s.world_to_sensor, np.float32).ravel()]
        st.fx, st.fy, st.cx, st.cy = float(s.fx), float(s.fy), float(s.cx), float(s.cy)
        st.k[:] = [float(x) for x in np.asarray(s.k, np.float32)]
        st.theta_max = float(s.theta_max)
        self._beams = None
        if s.beam_elevation is not None:
            self._beams = np.ascontiguousarray(s.beam_elevation, np.float32)
            st.beam_elevation = self._beams.ctypes.data
        st.azimuth0, st.azimuth_step = float(s.azimuth0), float(s.azimuth_step)
        self.struct = st

    @property
    def ref(self):
        return C.byref(self.struct)


def surfels_struct(t: dict) -> gs_surfels:
    """t: dict of contiguous float32 CUDA tensors (means, quats, scales,
    opacities[, sh, intensity, raydrop_logit]) and int sh_degree."""
    s = gs_surfels()
    s.n = int(t["means"].shape[0])
    s.means, s.quats, s.scales, s.opacities = (t["means"].data_ptr(), t["quats"].data_ptr(),
                                               t["scales"].data_ptr(), t["opacities"].data_ptr())
    s.sh = t["sh"].data_ptr() if t.get("sh") is not None else None
    s.sh_degree = int(t.get("sh_degree", 0))
    s.intensity = t["intensity"].data_ptr() if t.get("intensity") is not None else None
    s.raydrop_logit = t["raydrop_logit"].data_ptr() if t.get("raydrop_logit") is not None else None
    b = t.get("cull_bounds")
    if b is not None:
        # the bounds describe exactly these arrays (gsr.h): a sliced or regrouped dict must drop or recompute them
        if b.dim() != 2 or b.shape[1] != 8 or b.shape[0] < gs_cull_blocks(s.n) or not b.is_contiguous():
            raise ValueError(f"cull_bounds of shape {tuple(b.shape)} cannot describe {s.n} surfels "
                             "(recompute with render.cull_bounds or drop the key)")
        s.cull_bounds = b.data_ptr()
    else:
        s.cull_bounds = None
    return s


def gs_cull_blocks(n):
    return int(load().gs_cull_blocks(int(n)))


def gs_cull_bounds(surfels: gs_surfels, bounds, stream):
    _check(load().gs_cull_bounds(C.byref(surfels), _ptr(bounds), stream))


# ---------------------------------------------------------------- the C-ABI, same names
def gs_projected_bytes(n, kind):
    return int(load().gs_projected_bytes(int(n), int(kind)))


def gs_sort_workspace_bytes(n, cap, sensor: Sensor, opts: gs_opts):
    return int(load().gs_sort_workspace_bytes(int(n), int(cap), sensor.ref, C.byref(opts)))


def gs_num_tiles(sensor: Sensor, opts: gs_opts):
    return int(load().gs_num_tiles(sensor.ref, C.byref(opts)))


def gs_record_bytes(kind):
    return int(load().gs_record_bytes(int(kind)))


def gs_projected_offsets(n, kind):
    offs = (C.c_size_t * 5)()
    load().gs_projected_offsets(int(n), int(kind), offs)
    return dict(rec=offs[0], rect=offs[1], key=offs[2], count=offs[3], total=offs[4])


def gs_project(surfels: gs_surfels, sensor: Sensor, opts: gs_opts, projected, d_num_pairs, stream):
    _check(load().gs_project(C.byref(surfels), sensor.ref, C.byref(opts), _ptr(projected),
                             projected.numel() * projected.element_size(), _ptr(d_num_pairs),
                             C.c_void_p(stream)))


def gs_bin_sort(projected, n, sensor: Sensor, opts: gs_opts, keys, values, cap, tile_ranges,
                workspace, d_overflow, stream):
    _check(load().gs_bin_sort(_ptr(projected), int(n), sensor.ref, C.byref(opts), _ptr(keys),
                              _ptr(values), int(cap), _ptr(tile_ranges), _ptr(workspace),
                              workspace.numel() * workspace.element_size(), _ptr(d_overflow),
                              C.c_void_p(stream)))


def gs_render_workspace_bytes(cap, sensor: Sensor, opts: gs_opts):
    return int(load().gs_render_workspace_bytes(int(cap), sensor.ref, C.byref(opts)))


def gs_render_camera(projected, n, values, tile_ranges, d_overflow, sensor: Sensor, opts: gs_opts,
                     workspace, rgb, depth, normal, alpha, stream, stats=None):
    _check(load().gs_render_camera(_ptr(projected), int(n), _ptr(values), _ptr(tile_ranges),
                                   _ptr(d_overflow), sensor.ref, C.byref(opts), _ptr(workspace),
                                   workspace.numel() * workspace.element_size(), _ptr(rgb),
                                   _ptr(depth), _ptr(normal), _ptr(alpha), _ptr(stats),
                                   C.c_void_p(stream)))


def gs_render_lidar(projected, n, values, tile_ranges, d_overflow, sensor: Sensor, opts: gs_opts,
                    workspace, rng, intensity, raydrop, alpha, stream, stats=None):
    _check(load().gs_render_lidar(_ptr(projected), int(n), _ptr(values), _ptr(tile_ranges),
                                  _ptr(d_overflow), sensor.ref, C.byref(opts), _ptr(workspace),
                                  workspace.numel() * workspace.element_size(), _ptr(rng),
                                  _ptr(intensity), _ptr(raydrop), _ptr(alpha), _ptr(stats),
                                  C.c_void_p(stream)))


def gs_decode_anchors(anchors: gs_anchors, decoder: gs_decoder, view_origin, means, quats, scales, opacities,
                      sh, intensity, raydrop_logit, stream):
    origin = (C.c_float * 3)(*[float(v) for v in view_origin])
    _check(load().gs_decode_anchors(C.byref(anchors), C.byref(decoder), origin, _ptr(means), _ptr(quats),
                                    _ptr(scales), _ptr(opacities), _ptr(sh), _ptr(intensity),
                                    _ptr(raydrop_logit), C.c_void_p(stream)))


def gs_band_route_workspace_bytes(n, n_bands):
    return int(load().gs_band_route_workspace_bytes(int(n), int(n_bands)))


def gs_band_route(projected, n, sensor: Sensor, opts: gs_opts, band_rows, d_counts, d_index, workspace, stream):
    rows = np.ascontiguousarray(band_rows, np.int32)
    _check(load().gs_band_route(_ptr(projected), int(n), sensor.ref, C.byref(opts), rows.ctypes.data,
                                int(len(rows) - 1), _ptr(d_counts), _ptr(d_index), _ptr(workspace),
                                workspace.numel() * workspace.element_size(), C.c_void_p(stream)))


def gs_payload_floats(sh_degree, has_intensity, has_raydrop):
    return int(load().gs_payload_floats(int(sh_degree), int(bool(has_intensity)), int(bool(has_raydrop))))


def gs_pack_surfels(src: gs_surfels, d_index, m, payload, stream):
    _check(load().gs_pack_surfels(C.byref(src), _ptr(d_index), int(m), _ptr(payload), C.c_void_p(stream)))


def gs_unpack_surfels(payload, m, sh_degree, has_intensity, has_raydrop, means, quats, scales, opacities, sh,
                      intensity, raydrop_logit, stream):
    _check(load().gs_unpack_surfels(_ptr(payload), int(m), int(sh_degree), int(bool(has_intensity)),
                                    int(bool(has_raydrop)), _ptr(means), _ptr(quats), _ptr(scales),
                                    _ptr(opacities), _ptr(sh), _ptr(intensity), _ptr(raydrop_logit),
                                    C.c_void_p(stream)))


def gs_backward_workspace_bytes(n):
    return int(load().gs_backward_workspace_bytes(int(n)))


def gs_render_backward(surfels: gs_surfels, sensor: Sensor, opts: gs_opts, projected, values, tile_ranges,
                       grad_out, workspace, d_means, d_quats, d_scales, d_opacities, d_sh, d_intensity,
                       d_raydrop_logit, stream):
    _check(load().gs_render_backward(C.byref(surfels), sensor.ref, C.byref(opts), _ptr(projected), _ptr(values),
                                     _ptr(tile_ranges), _ptr(grad_out), _ptr(workspace),
                                     workspace.numel() * workspace.element_size(), _ptr(d_means), _ptr(d_quats),
                                     _ptr(d_scales), _ptr(d_opacities), _ptr(d_sh), _ptr(d_intensity),
                                     _ptr(d_raydrop_logit), C.c_void_p(stream)))


def gs_kernel_launches() -> int:
    return int(load().gs_kernel_launches())
