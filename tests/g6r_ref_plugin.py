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


# Reference tests that measure the CPU implementation itself, not the path's
# results: they stay out of the CUDA run (reported, not silently skipped).
NOT_APPLICABLE = {
    "test_acceptance.py::test_throughput_floor":
        "asserts >= 3x speedup from 1 to 8 OpenMP threads; the CUDA path ignores "
        "RenderConfig.threads (its single-thread rate is the GPU rate)",
}


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for item in items:
        (drop if item.nodeid in NOT_APPLICABLE else keep).append(item)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep
        for item in drop:
            print(f"[g6r] deselected {item.nodeid}: {NOT_APPLICABLE[item.nodeid]}",
                  file=sys.stderr)


def pytest_report_header(config):
    return "[g6r] reference suite routed to the CUDA path"


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    terminalreporter.write_line("[g6r] reference suite routed to the CUDA path")
    print("[g6r] reference suite routed to the CUDA path", file=sys.stderr)
