#!/bin/bash
# Same-box A/B on c3 (or the given bench args): the default build, every
# ab/lib_*.so through the current bench (RLC_LIB_PATH), and ab/old (a whole
# older tree, its own bench) when present; `reps` rounds.
# usage: tools/ab.sh reps [bench args...]
reps=${1:-2}; shift
summ() { python -c "import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d.get('stage_ms_per_step',{}); print(sys.argv[2], round(d['value']/1e6,1), 'M/s', round(d['ms_per_step'],4), 'ms', {k:round(v,3) for k,v in s.items()})
except Exception as e: print(sys.argv[2], 'no result', e)" $1 $2; }
for r in $(seq $reps); do
  python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_default.json 2>&1; summ gpurun_out/ab_default.json default
  for f in ab/lib_*.so; do [ -e "$f" ] || continue; n=$(basename $f .so)
    RLC_LIB_PATH=$f python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_$n.json 2>&1; summ gpurun_out/ab_$n.json $n
  done
  if [ -d ab/old ]; then (cd ab/old && python bench.py --no-cpu-baseline --no-e2e "$@" > ../../gpurun_out/ab_old.json 2>&1); summ gpurun_out/ab_old.json old; fi
done
