mkdir -p gpurun_out
for L in main _ab/noell/libg6r.so _ab/base/libg6r.so; do
  if [ "$L" = main ]; then unset G6R_LIBRARY; else export G6R_LIBRARY=$L; fi
  echo "== $L"
  timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_composite --csv python tools/probe_sort.py 2>/dev/null | grep -E "k_composite" | awk -F'","' '{print $(NF-2), $NF}'
done
