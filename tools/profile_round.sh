#!/bin/bash
# Round profile capture (run on the GPU box via gpurun): the bench without ncu
# first, then the launch list of the same command, then one `--set full`
# capture per hot kernel of a steady-state 8-view batch (tools/probe_sort.py).
set -x
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 300 python bench.py --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list_${TAG}.log 2>&1
for K in k_composite k_project k_onesweep k_sort_hist k_chunk_scatter k_chunk_count; do
  S=3; [ "$K" = k_onesweep ] && S=5
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K" -s $S -c 1 \
      -o gpurun_out/full_${TAG}_${K} python tools/probe_sort.py > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
done
ls -la gpurun_out
