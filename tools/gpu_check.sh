#!/bin/bash
# One GPU-box pass (via gpurun): the driver's bench command, then the GPU suite.
# Usage: bash tools/gpu_check.sh TAG [pytest-args...]
TAG=${1:-s1}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
timeout 400 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench_${TAG}.json
if [ "$1" != "--no-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > gpurun_out/gputests_${TAG}.log 2>&1; echo "tests rc=$?"
  tail -15 gpurun_out/gputests_${TAG}.log
fi
