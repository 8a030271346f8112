mkdir -p gpurun_out
for CC in all none; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control $CC --csv python tools/probe_sort.py 2>/dev/null | grep -E "gpu__time" | awk -F'","' -v cc=$CC '{split($5,a,"("); print cc, a[1], $NF}' > gpurun_out/ncu_cc_$CC.log
done
