"""pytest plugin (``-p g6r_ref_plugin``) that runs the reference's OWN test
files against the B200 path: before collection, it installs the integrate
shim with the kernel modules replaced, so the reference tests' import-time
``from splatct.raster import render, ...`` and their direct
``splatct._kernels`` / ``_kernels_py`` calls all reach the CUDA code.  Used by
tests/test_gpu_integrate.py in a subprocess."""

import sys


def pytest_configure(config):
    from paper_2505_17338_b200 import integrate
    from paper_2505_17338_b200 import _native
    _native.load()   # fail loudly here if the library or the GPU is missing
    config._g6r_shim = integrate.install(kernel_modules=True)


def pytest_report_header(config):
    return "[g6r] reference suite routed to the CUDA path"


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line("[g6r] reference suite routed to the CUDA path")
    print("[g6r] reference suite routed to the CUDA path", file=sys.stderr)
