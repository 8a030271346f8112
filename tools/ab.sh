#!/bin/bash
# A/B timing on the GPU box: bench.py (no CPU leg) against each library given
# as an argument (paths to libg6r.so; "main" = the in-tree build), alternating.
ROUNDS=${ROUNDS:-2}
mkdir -p gpurun_out
for r in $(seq $ROUNDS); do
  for L in "$@"; do
    if [ "$L" = main ]; then unset G6R_LIBRARY; else export G6R_LIBRARY=$L; fi
    timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms_per_view']
print('$L', round(d['value']), round(d['e2e']['value']), {k: round(v,4) for k,v in s.items()})"
  done
done
