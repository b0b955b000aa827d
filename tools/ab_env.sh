#!/bin/bash
# Same-box A/B of environment settings on the default build:
#   tools/ab_env.sh reps "NAME=VAL ..." "NAME=VAL ..." ... (an empty string: the defaults)
reps=$1; shift
summ() { python -c "import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d.get('stage_ms_per_step',{}); print(sys.argv[2], round(d['value']/1e6,1), 'M/s', round(d['ms_per_step'],4), 'ms', {k:round(v,3) for k,v in s.items() if v})
except Exception as e: print(sys.argv[2], 'no result', e)" $1 "$2"; }
for r in $(seq $reps); do
  i=0
  for setting in "$@"; do
    env $setting python bench.py --no-cpu-baseline --no-e2e $BENCH_ARGS > gpurun_out/abenv_$i.json 2>&1
    summ gpurun_out/abenv_$i.json "[$setting]"
    i=$((i+1))
  done
done
