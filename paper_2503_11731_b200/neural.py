"""Neural-Gaussian decode through the C-ABI (gs_decode_anchors, NEXT-1).

`NeuralDecoder` keeps one decoder's weights resident on the GPU (fp16
weights, fp32 biases, the gs_decoder struct pointing at them) and decodes a
resident anchor set for a view origin into a surfel dict in the format of
render.to_device -- the input of Renderer / BatchRenderer (gs_project).  It
only allocates buffers and marshals arguments: the MLPs run in libgsr.so's
tcgen05 kernel.  Heads and sizes: include/gsr.h, DESIGN.md §12.
"""
from __future__ import annotations

import numpy as np
import torch

from . import gsr

CAMERA_HEADS = ("offset", "scale", "rotation", "opacity", "color")
LIDAR_HEADS = ("offset", "scale", "rotation", "opacity", "intensity", "raydrop")


def anchors_to_device(a, device="cuda") -> dict:
    """scenegen.Anchors (numpy) -> dict of contiguous CUDA tensors (feature as fp16)."""
    return dict(position=torch.from_numpy(np.ascontiguousarray(a.position, np.float32)).to(device),
                feature=torch.from_numpy(np.ascontiguousarray(a.feature, np.float16)).to(device),
                base_scale=torch.from_numpy(np.ascontiguousarray(a.base_scale, np.float32)).to(device))


def anchors_struct(t: dict) -> gsr.gs_anchors:
    s = gsr.gs_anchors()
    s.n = int(t["position"].shape[0])
    s.position, s.feature, s.base_scale = (t["position"].data_ptr(), t["feature"].data_ptr(),
                                           t["base_scale"].data_ptr())
    return s


class NeuralDecoder:
    def __init__(self, weights: dict, modality: str = "camera", device="cuda"):
        """weights: {head: {W1, b1, W2, b2, W3, b3}} (numpy; W* fp16, b* fp32)."""
        self.device = torch.device(device)
        self.modality = modality
        heads = CAMERA_HEADS if modality == "camera" else LIDAR_HEADS
        self._t = []
        st = gsr.gs_decoder()
        st.modality = gsr.GS_DECODE_CAMERA if modality == "camera" else gsr.GS_DECODE_LIDAR
        for i, h in enumerate(heads):
            p = weights[h]
            ts = {}
            for k in ("W1", "W2", "W3"):
                ts[k] = torch.from_numpy(np.ascontiguousarray(p[k], np.float16)).to(self.device)
            for k in ("b1", "b2", "b3"):
                ts[k] = torch.from_numpy(np.ascontiguousarray(p[k], np.float32)).to(self.device)
            self._t.append(ts)
            m = st.head[i]
            m.w1, m.b1, m.w2, m.b2, m.w3, m.b3 = (ts[k].data_ptr() for k in ("W1", "b1", "W2", "b2", "W3", "b3"))
        self.struct = st

    def alloc(self, n_anchors: int) -> dict:
        """Surfel buffers for n_anchors anchors (render.to_device format)."""
        n = gsr.GS_NEURAL_K * int(n_anchors)
        f = lambda *s: torch.empty(s, dtype=torch.float32, device=self.device)
        cam = self.modality == "camera"
        return dict(means=f(n, 3), quats=f(n, 4), scales=f(n, 2), opacities=f(n),
                    sh=f(n, 1, 3) if cam else None, sh_degree=0,
                    intensity=None if cam else f(n), raydrop_logit=None if cam else f(n))

    def decode(self, anchors: dict, view_origin, out: dict | None = None, stream=None) -> dict:
        """Decode `anchors` (anchors_to_device) for a sensor at view_origin
        (world) into `out` (alloc); returns the surfel dict."""
        n = int(anchors["position"].shape[0])
        if out is None:
            out = self.alloc(n)
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        gsr.gs_decode_anchors(anchors_struct(anchors), self.struct, view_origin, out["means"], out["quats"],
                              out["scales"], out["opacities"], out["sh"], out["intensity"],
                              out["raydrop_logit"], st)
        return out
