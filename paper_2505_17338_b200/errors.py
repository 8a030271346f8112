"""Exception types of the render path, mirroring the reference's
(core.py:42-51): same names, same base classes, raised at the same conditions."""


class InvalidParameterError(ValueError):
    """Raw parameters or options are non-finite, malformed or unsupported."""


class DegenerateCovarianceError(ArithmeticError):
    """Too many selected Gaussians have a singular directional block."""


class DegenerateGeometryError(ValueError):
    """Geometric construction is undefined (e.g. zero-length direction)."""


class VolumeFormatError(ValueError):
    """Volume or parameter-volume shape/file inconsistency (volume.py:67)."""


class EmptySceneError(ValueError):
    """No foreground voxels to instantiate Gaussians from (priming.py:46)."""
