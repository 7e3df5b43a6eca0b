"""Pixel-partitioned single-frame rendering (NEXT-4), -m gpu,
ranks emulated one after another on one GPU (pixdist.emulate).

Pins: the exchange set equals the brute-force overlap set
(every visible surfel whose tile rect meets a band, in index order); the
distributed frame equals the single-GPU frame (LiDAR bitwise; cameras to
fp32 rounding of the cropped sensor's principal point) and passes the
strict oracle gate."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import scenegen as sg  # noqa: E402
from tests import parity  # noqa: E402


@pytest.fixture(scope="module")
def pd():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_11731_b200 import gsr, pixdist
    gsr.load()
    return pixdist


def _scene(seed=120, lidar=False):
    rng = np.random.default_rng(seed)
    if lidar:
        return sg.street(rng, 60_000, -60.0, 60.0, 0, lidar_attrs=True, with_sh=False)
    return sg.street(rng, 30_000, 1.0, 60.0, 2, lidar_attrs=True)


def test_route_lists_equal_brute_force_overlap(pd):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    s = _scene()
    se = sg.pinhole(200, 150, 125.0, 100.0, 75.0, sg.camera_pose([0, 1.5, 0], 0.0))
    dev = to_device(s)
    r = Renderer(dev)
    r.render(se, keys=True)
    b = r.binning_state()
    bounds = [0, 3, 7, 12, 19]   # 19 tile rows of 8 px
    assert bounds[-1] == pd.tile_rows(se, r.cam_opts)
    router = pd.BandRouter(dev)
    payload, counts = router.route(se, bounds)
    torch.cuda.synchronize()
    vis = np.nonzero(b["count"] > 0)[0]
    y0, y1 = b["rect"][vis, 1], b["rect"][vis, 3]
    off = 0
    for k in range(4):
        want = vis[(y1 >= bounds[k]) & (y0 < bounds[k + 1])]
        assert counts[k] == len(want)
        # the packed means are those of the listed surfels, in index order
        got = payload[off: off + counts[k], :3].cpu().numpy()
        np.testing.assert_array_equal(got, s.means[want])
        off += counts[k]


def test_pack_unpack_round_trip(pd):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import to_device
    s = _scene()
    dev = to_device(s)
    idx = torch.arange(s.n, dtype=torch.int32, device="cuda")
    F = gsr.gs_payload_floats(2, True, True)
    assert F == 10 + 27 + 2
    pay = torch.empty((s.n, F), dtype=torch.float32, device="cuda")
    gsr.gs_pack_surfels(gsr.surfels_struct(dev), idx, s.n, pay, torch.cuda.current_stream().cuda_stream)
    back = pd.unpack(pay, dev)
    for k in ("means", "quats", "scales", "opacities", "sh", "intensity", "raydrop_logit"):
        assert torch.equal(back[k], dev[k]), k


@pytest.mark.parametrize("world,bounds", [(2, [0, 9, 19]), (4, [0, 2, 5, 11, 19]), (3, [0, 1, 2, 19])])
def test_emulated_pixel_partition_matches_single_gpu_camera(pd, world, bounds):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    s = _scene()
    se = sg.pinhole(200, 150, 125.0, 100.0, 75.0, sg.camera_pose([0, 1.5, 0], 0.0))
    dev = to_device(s)
    opts = gsr.default_opts(split_len=2 ** 31 - 1)
    single = Renderer(dev, opts).render(se).cpu().numpy()
    full, band_n, matrix = pd.emulate(dev, se, bounds, world, opts)
    full = full.cpu().numpy()
    assert np.abs(full - single).max() < 2e-5
    rays = np.arange(se.width * se.height)
    ref, fl, _ = oracle.render(s, se, rays)
    st = parity.compare(full, ref, fl, rays, se, s)
    assert st["ok"], st
    assert sum(band_n) < 2.0 * int((Renderer(dev).project(gsr.Sensor(se))[0][:4].view(torch.int32)).item())


def test_emulated_pixel_partition_lidar_bitwise(pd):
    from paper_2503_11731_b200 import gsr
    from paper_2503_11731_b200.render import Renderer, to_device
    s = _scene(lidar=True)
    se = sg.lidar64(sg.lidar_pose([0, 1.8, 0]), height=32, width=360)
    dev = to_device(s)
    opts = gsr.default_opts(split_len=2 ** 31 - 1)
    ropts = gsr.gs_opts.from_buffer_copy(opts)
    ropts.tile_w, ropts.tile_h = 32, 1
    single = Renderer(dev, opts).render(se).cpu().numpy()
    full, _, _ = pd.emulate(dev, se, [0, 5, 11, 20, 32], 4, ropts)
    np.testing.assert_array_equal(full.cpu().numpy(), single)
