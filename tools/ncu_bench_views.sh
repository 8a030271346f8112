#!/bin/bash
# ncu on the bench's own timed views (tools/probe_bench_views.py: cfg3, the
# first 20 orbit views in the bench's balanced 10 + 10 batches), run on the GPU
# box via gpurun.  1) the probe without ncu (CUDA-event stage split), 2) the
# launch list of the same command, 3) one `--set full` capture per hot kernel
# (the first launch of the probe's second render_views call, i.e. warm).
# Usage: bash tools/ncu_bench_views.sh TAG [kernel-regex ...]
TAG=${1:-r2}; shift
KS=${@:-k_composite k_project k_onesweep k_chunk_scatter k_chunk_count}
mkdir -p gpurun_out
timeout 300 python tools/probe_bench_views.py --batch 10 > gpurun_out/probe_${TAG}.json 2> gpurun_out/probe_${TAG}.err
echo "probe rc=$?"; cat gpurun_out/probe_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python tools/probe_bench_views.py --batch 10 > gpurun_out/ncu_list_${TAG}.log 2>&1
echo "launch list rc=$?"
for K in $KS; do
  S=2; [ "$K" = k_onesweep ] && S=9
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$K" -s $S -c 1 \
      -o gpurun_out/full_${TAG}_${K} python tools/probe_bench_views.py --batch 10 > gpurun_out/ncu_full_${TAG}_${K}.log 2>&1
  echo "$K rc=$?"
done
ls -la gpurun_out
