#!/bin/bash
# Builds to compare: make -C paper_1911_10217_b200/csrc OUT=$PWD/variants/lib_X.so OBJ=$PWD/build/obj_X EXTRA=-D...
# usage: variants/run.sh [bench args...] -- runs bench.py with every variants/lib_*.so and the default lib
summ() { python -c "import json,sys
try:
  d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=d.get(\"stage_ms_per_step\",{}); print(sys.argv[2], round(d[\"value\"]/1e6,1), \"M/s\", round(d[\"ms_per_step\"],4), \"ms\", {k:round(v,3) for k,v in s.items()})
except Exception as e: print(sys.argv[2], \"no result\")" $1 $2; }
python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/v_default.json 2>&1; summ gpurun_out/v_default.json default
for f in variants/lib_*.so; do n=$(basename $f .so); RLC_LIB_PATH=$f python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/v_$n.json 2>&1; summ gpurun_out/v_$n.json $n; done
