"""Served-frame output path.

The reference turns a render into response bytes on the host:
``encode_png(composite_over(render(scene, cam), background))``
(service.py:175-184 render_request_png; metrics.py:21-25; _png.py:21-40).
Here the composite-over-background and the 8-bit quantisation run in the
compositor's epilogue (g6r_frame.rgba8), so the float image never reaches HBM
and a 512x512 frame crosses PCIe as 1 MiB instead of 4 MiB; only the zlib
deflate of the PNG container stays on the host (PIL, compress level 6, the
reference's byte-identical encoding).
"""

from __future__ import annotations

import io

import numpy as np

from .errors import InvalidParameterError
from .raster import DEFAULT_CONFIG, RenderConfig, render_frames_u8

COMPRESS_LEVEL = 6   # _png.py:18


def encode_rgba8_png(rgba: np.ndarray) -> bytes:
    """PNG bytes of an (H, W, 4) uint8 frame, deterministic (_png.py:35-40)."""
    from PIL import Image
    rgba = np.ascontiguousarray(rgba, dtype=np.uint8)
    if rgba.ndim != 3 or rgba.shape[2] != 4:
        raise InvalidParameterError(f"frame must have shape (H, W, 4), got {rgba.shape}")
    buf = io.BytesIO()
    Image.fromarray(rgba, mode="RGBA").save(buf, format="PNG", compress_level=COMPRESS_LEVEL)
    return buf.getvalue()


def render_png(scene, camera, group_mask=None, config: RenderConfig = DEFAULT_CONFIG,
               background=(0.0, 0.0, 0.0)) -> bytes:
    """One served frame as PNG bytes, byte-identical to the reference's
    ``render_request_png`` for the same scene, camera, mask and background."""
    frame = render_frames_u8(scene, [camera], background, group_mask, config)[0]
    return encode_rgba8_png(frame)


def render_pngs(scene, cameras, group_mask=None, config: RenderConfig = DEFAULT_CONFIG,
                background=(0.0, 0.0, 0.0)) -> list:
    """PNG bytes for many views: frames rendered and quantised in batches on
    the device, then encoded on the host."""
    frames = render_frames_u8(scene, cameras, background, group_mask, config)
    return [encode_rgba8_png(f) for f in frames]
