"""B200-native 6DGS render path (Render-FM, arXiv 2505.17338).

Drop-in for the reference package's render entry points (``splatct.raster``):
per-view 6D->3D slicing, EWA projection + SH shading, tile binning, on-device
radix sort + tile ranges and per-tile alpha compositing, as hand-written
sm_100a CUDA behind the C ABI in ``include/g6r.h``.
"""

__version__ = "0.1.0"

from .camera import Camera, look_at_rotation, make_camera  # noqa: F401
from .errors import (DegenerateCovarianceError, DegenerateGeometryError,  # noqa: F401
                     InvalidParameterError)
from .scene import Scene, filter_scene  # noqa: F401
