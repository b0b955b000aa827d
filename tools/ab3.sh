#!/bin/bash
# Same-box A/B of the default build against older whole trees ab/<name>/ (each with its own bench).
reps=${1:-2}; shift
summ() { python -c "import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d.get('stage_ms_per_step',{}); print(sys.argv[2], round(d['value']/1e6,1), 'M/s', round(d['ms_per_step'],4), 'ms', {k:round(v,3) for k,v in s.items() if v})
except Exception as e: print(sys.argv[2], 'no result', e)" $1 $2; }
for r in $(seq $reps); do
  python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab3_default.json 2>&1; summ gpurun_out/ab3_default.json default
  for d in ab/*/; do n=$(basename $d); [ -f $d/bench.py ] || continue
    (cd $d && python bench.py --no-cpu-baseline --no-e2e "$@" > ../../gpurun_out/ab3_$n.json 2>&1); summ gpurun_out/ab3_$n.json $n
  done
done
