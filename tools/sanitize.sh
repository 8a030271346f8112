#!/bin/bash
# compute-sanitizer over tools/sanitize_probe.py (run on the GPU box via gpurun):
# memcheck (out-of-bounds / misaligned accesses, leaks), racecheck (shared-
# memory hazards), synccheck (barrier misuse), initcheck (reads of
# uninitialised device memory).  Logs -> gpurun_out/sanitizer_<tool>.log.
mkdir -p gpurun_out
export G6R_SAN_N=${G6R_SAN_N:-10000}
for TOOL in memcheck racecheck synccheck initcheck; do
  EXTRA=""
  [ "$TOOL" = memcheck ] && EXTRA="--leak-check full"
  [ "$TOOL" = racecheck ] && EXTRA="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $TOOL $EXTRA --target-processes all \
      --print-limit 50 --log-file gpurun_out/sanitizer_${TOOL}.log \
      python tools/sanitize_probe.py > gpurun_out/sanitizer_${TOOL}.out 2>&1
  echo "$TOOL rc=$?"; tail -3 gpurun_out/sanitizer_${TOOL}.log
done
