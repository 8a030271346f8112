#!/bin/bash
# A/B timing on the GPU box over environment settings (each argument is a
# space-separated list of VAR=value, "" = defaults), alternating ROUNDS times:
# the bench's own views through tools/probe_bench_views.py (one stream, stage
# split) and, with BENCH=1, bench.py itself (no CPU leg).
ROUNDS=${ROUNDS:-2}
mkdir -p gpurun_out
for r in $(seq $ROUNDS); do
  for E in "$@"; do
    env $E timeout 300 python tools/probe_bench_views.py --batch ${BATCH:-10} ${PROBE_ARGS} 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('probe [$E]', round(d['wall_ms_per_view'],4), {k: round(v,4) for k,v in d['stage_ms_per_view'].items()})"
    if [ "$BENCH" = 1 ]; then
      env $E timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-legs ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms_per_view']
print('bench [$E]', round(d['value']), round(d['e2e']['value']), {k: round(v,4) for k,v in s.items()})"
    fi
  done
done
