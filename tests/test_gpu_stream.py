"""Chunk streaming with double-buffered residency (NEXT-3), -m gpu.

Pins: a render issued while the back buffer is being
uploaded equals the pre-swap front-buffer render bitwise; after the swap a
render equals rendering the new active set uploaded directly, bitwise; the
streamed set is the concatenation of its chunks in chunk order."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import scenegen as sg  # noqa: E402


@pytest.fixture(scope="module")
def chunks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2503_11731_b200 import gsr
    gsr.load()
    out = []
    for c in range(4):   # 4 chunks of 25 m, 60K surfels each
        rng = np.random.default_rng(500 + c)
        out.append(sg.street(rng, 60_000, 25.0 * c, 25.0 * c + 25.0, 1, lidar_attrs=True))
    return out


def _frames(z):
    return [sg.pinhole(160, 96, 110.0, 80.0, 48.0, sg.camera_pose([0, 1.5, z], 0.0)),
            sg.pinhole(160, 96, 110.0, 80.0, 48.0, sg.camera_pose([0, 1.5, z], np.pi)),
            sg.lidar64(sg.lidar_pose([0, 1.8, z]), height=16, width=256)]


def test_mid_swap_render_is_front_buffer_bitwise(chunks):
    from paper_2503_11731_b200.render import Renderer, to_device
    from paper_2503_11731_b200.stream import ChunkStreamer, Zone, active_set
    zones = [Zone(-10.0, 10.0, 25.0 * c, 25.0 * c + 25.0) for c in range(4)]
    st = ChunkStreamer(chunks, zones)
    pa, pb = (0.0, 1.5, 30.0), (0.0, 1.5, 49.0)
    ida, idb = active_set(zones, pa), active_set(zones, pb)
    assert ida == (1,) and idb == (1, 2)
    assert st.load(pa) == ida
    frames = _frames(30.0)
    r = Renderer(st.front())
    before = [r.render(f).cpu().numpy() for f in frames]
    assert st.update(pb)                       # upload of (1, 2) into the back buffer starts
    r.set_surfels(st.front())
    during = [r.render(f).cpu().numpy() for f in frames]   # still the front set
    for x, y in zip(before, during):
        np.testing.assert_array_equal(x, y)
    assert st.poll(wait=True) and st.front_set() == idb and st.swaps == 1
    r.set_surfels(st.front())
    after = [r.render(f).cpu().numpy() for f in frames]
    direct = Renderer(to_device(sg.Surfels.concat([chunks[i] for i in idb])))
    for f, x in zip(frames, after):
        np.testing.assert_array_equal(x, direct.render(f).cpu().numpy())
    # the front set is the concatenation of its chunks in chunk order
    fr = st.front()
    np.testing.assert_array_equal(fr["means"].cpu().numpy(),
                                  np.concatenate([chunks[1].means, chunks[2].means]))
    assert not st.update(pb)                   # same set: nothing to do


def test_streamed_trajectory_with_batch_renderer(chunks):
    """A drive across two zone boundaries: per timestep update / poll, then
    the BatchRenderer (capacity planning + overflow repair) renders from the
    front set; every frame equals a direct render of that timestep's set."""
    from paper_2503_11731_b200.batch import BatchRenderer
    from paper_2503_11731_b200.render import Renderer, to_device
    from paper_2503_11731_b200.stream import ChunkStreamer, Zone
    zones = [Zone(-10.0, 10.0, 25.0 * c, 25.0 * c + 25.0) for c in range(4)]
    st = ChunkStreamer(chunks, zones)
    st.load((0.0, 1.5, 20.0))
    br = BatchRenderer(st.front(), n_streams=2)
    seen = set()
    for z in np.arange(20.0, 60.0, 4.0):
        st.update((0.0, 1.5, z))
        st.poll(wait=True)                     # the test waits; a simulator polls
        br.set_surfels(st.front())
        frames = _frames(float(z))
        outs = br.alloc_outputs(br.wrap(frames))
        br.render_checked(frames, outs)
        seen.add(st.front_set())
        if z in (20.0, 36.0, 52.0):
            direct = Renderer(to_device(sg.Surfels.concat([chunks[i] for i in st.front_set()])))
            for f, o in zip(frames, outs):
                ref = direct.render(f, opts=None).cpu().numpy()
                assert np.abs(o.cpu().numpy() - ref).max() < 2e-5   # split lists may differ by fp32 rounding
    assert len(seen) >= 3 and st.swaps >= 2
