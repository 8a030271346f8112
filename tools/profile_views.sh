#!/bin/bash
# Round profile capture on the bench's own views (run on the GPU box via gpurun):
# the probe without ncu, its launch list, then one `--set full` capture per hot
# kernel of the profiled (last) pass of tools/probe_bench_views.py.
#   bash tools/profile_views.sh TAG [kernels...]
TAG=${1:-r2}
shift
KERNELS=${@:-k_composite k_project k_onesweep k_chunk_scatter k_chunk_count k_sort_hist}
mkdir -p gpurun_out
timeout 300 python tools/probe_bench_views.py > gpurun_out/probe_${TAG}.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python tools/probe_bench_views.py > gpurun_out/ncu_list_${TAG}.log 2>&1
for K in $KERNELS; do
  # skip the warm-up passes: the profiled pass is the last 2 batches
  N=$(( $(grep -c "g6r::${K}[<(]" gpurun_out/launches_${TAG}.csv) / 3 ))
  PER=2; [ "$K" = k_onesweep ] && PER=8
  S=$((N - PER)); [ $S -lt 0 ] && S=0
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^${K}" -s $S -c 1 \
      -o gpurun_out/full_${TAG}_${K} -f python tools/probe_bench_views.py > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
done
ls -la gpurun_out | tail -20
