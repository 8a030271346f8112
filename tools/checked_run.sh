#!/bin/bash
# Bounds-checked run (substitute for compute-sanitizer, which is closed on this
# pool): the GPU test suite against libg6r.so built with -DG6R_CHECKED, where
# every device-derived index (entry slots, sorted positions, splat rows, tile
# runs, gathered payload rows) is checked against its buffer and a violation
# traps (g6r_common.cuh G6R_CHECK).  Build here: make -C paper_2505_17338_b200/csrc
# OUT_DIR=../_lib_checked EXTRA=-DG6R_CHECKED; run on the GPU box:
#   bash tools/checked_run.sh
mkdir -p gpurun_out
LIB=$PWD/paper_2505_17338_b200/_lib_checked/libg6r.so
[ -f "$LIB" ] || make -s -j8 -C paper_2505_17338_b200/csrc OUT_DIR=../_lib_checked EXTRA=-DG6R_CHECKED
G6R_LIBRARY=$LIB timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
    --deselect tests/test_gpu_multirank.py::test_bench_two_ranks_gloo_on_one_device \
    > gpurun_out/checked_tests.log 2>&1
echo "checked suite rc=$?"; tail -3 gpurun_out/checked_tests.log
G6R_LIBRARY=$LIB timeout 600 python tools/probe_bench_views.py > gpurun_out/checked_probe.log 2>&1
echo "checked bench-views probe rc=$?"; tail -2 gpurun_out/checked_probe.log
