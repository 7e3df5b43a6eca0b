"""Throughput of gs_decode_anchors (NEXT-1) at Chunked scale: 2.4 M anchors ->
12 M surfels (camera and LiDAR decoders), CUDA events over back-to-back
launches.  Prints one JSON line per modality with the HBM roofline fraction
(algorithmic bytes: 88 B read per anchor + the surfel attributes written).

python tools/bench_decode.py [n_anchors] [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2503_11731_b200 import gsr  # noqa: E402
from paper_2503_11731_b200.neural import NeuralDecoder, anchors_to_device  # noqa: E402

WRITE_B = {"camera": 5 * (12 + 16 + 8 + 4 + 12), "lidar": 5 * (12 + 16 + 8 + 4 + 4 + 4)}
READ_B = 12 + 64 + 12
# fp16 MMA FLOPs per anchor as issued (padded shapes): L1 128x48x32H, L2 H x 32x32, L3 sum(out_pad) x 32
FLOP = {"camera": 2 * (48 * 160 + 5 * 32 * 32 + 96 * 32), "lidar": 2 * (48 * 192 + 6 * 32 * 32 + 112 * 32)}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_400_000
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6544.3}
    rng = np.random.default_rng(0)
    a = anchors_to_device(sg.street_anchors(rng, n, 0.0, 400.0))
    for modality in ("camera", "lidar"):
        nd = NeuralDecoder(sg.neural_decoder(rng, modality), modality)
        out = nd.alloc(n)
        for _ in range(3):
            nd.decode(a, (0.0, 1.5, 200.0), out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(reps):
            nd.decode(a, (0.0, 1.5, 200.0 + r), out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        byts = n * (READ_B + WRITE_B[modality])
        gbs = byts / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": f"k_decode<{modality}>", "anchors": n, "surfels": 5 * n,
                          "ms_per_launch": round(ms, 4), "Msurfels_per_s": round(5 * n / (ms * 1e-3) / 1e6, 1),
                          "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"],
                                       "unit": "GB/s", "frac": round(gbs / peaks["hbm_gbs"], 4),
                                       "bytes_per_anchor": READ_B + WRITE_B[modality]},
                          "tensor_tflops": round(n * FLOP[modality] / (ms * 1e-3) / 1e12, 2)}), flush=True)


if __name__ == "__main__":
    main()
