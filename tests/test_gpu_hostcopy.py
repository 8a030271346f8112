"""Host copies gated by view completion (g6r_frame.host_image / host_rgba8).

render_views with ``host_out`` / ``host_rgba8`` copies every view to pinned
host memory on the library's copy stream as soon as the compositor's last CTA
of that view has published its completion flag; the compositor then also
takes the batch's tiles view by view.  Neither may change a pixel: the host
copies must equal the device images bit for bit, in both exp modes, through
the single-stream and the pipelined paths, and across repeated calls that
reuse the flag slots (monotonic flag values per call)."""
import numpy as np
import pytest
import torch

from paper_2505_17338_b200 import raster, scenes
from paper_2505_17338_b200.errors import InvalidParameterError
from paper_2505_17338_b200.raster import RenderConfig

pytestmark = pytest.mark.gpu


def _scene_and_cams(n=30000, views=23, size=160, seed=91):
    s = scenes.random_scene(np.random.default_rng(seed), n)
    return s, scenes.orbit_ring(s, count=views, size=size)


@pytest.mark.parametrize("exp_mode", ["exact", "fast"])
@pytest.mark.parametrize("batch,pipeline", [(4, True), (4, False), (32, True)])
def test_host_copies_equal_device_images(exp_mode, batch, pipeline):
    s, cams = _scene_and_cams()
    cfg = RenderConfig(exp_mode=exp_mode)
    ref, cref = raster.render_views(s, cams, config=cfg, concurrency=batch, pipeline=pipeline)
    host = torch.empty_like(ref, device="cpu").pin_memory()
    host.fill_(float("nan"))
    dev, cnt = raster.render_views(s, cams, config=cfg, concurrency=batch, pipeline=pipeline,
                                   host_out=host)
    cnt = cnt.cpu()   # synchronises the stream the copies were joined into
    assert torch.equal(cnt, cref.cpu())
    # completion signalling and view-major compositor order change no pixel
    assert torch.equal(dev, ref)
    assert torch.equal(host, ref.cpu())


def test_repeated_calls_reuse_flag_slots():
    s, cams = _scene_and_cams(n=12000, views=9, size=96, seed=92)
    ref, _ = raster.render_views(s, cams, concurrency=2)
    ref = ref.cpu()
    host = torch.empty_like(ref).pin_memory()
    for k in range(5):
        host.zero_()
        _, cnt = raster.render_views(s, cams, concurrency=2, host_out=host)
        cnt.cpu()
        assert torch.equal(host, ref), k


def test_rgba8_host_copies_and_render_batch():
    s, cams = _scene_and_cams(n=20000, views=11, size=128, seed=93)
    bg = (0.2, 0.3, 0.4)
    dev = raster.render_frames_u8(s, cams, bg, batch=3, device_out=True).cpu().numpy()
    host = raster.render_frames_u8(s, cams, bg, batch=3)
    np.testing.assert_array_equal(host, dev)
    imgs = raster.render_batch(s, cams, batch=3)
    want = raster.render_views(s, cams, concurrency=3)[0].cpu().numpy()
    np.testing.assert_array_equal(imgs, want)


def test_host_out_must_be_pinned_and_shaped():
    s, cams = _scene_and_cams(n=2000, views=2, size=64, seed=94)
    with pytest.raises(InvalidParameterError):
        raster.render_views(s, cams, host_out=torch.empty((2, 64, 64, 4)))   # not pinned
    with pytest.raises(InvalidParameterError):
        raster.render_views(s, cams, host_out=torch.empty((2, 64, 64, 3)).pin_memory())
