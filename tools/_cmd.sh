BENCH_ARGS="--config c1" bash tools/ab_env.sh 3 "" "RLC_GRAPHS=1" "RLC_OVERLAP=0" "RLC_GRAPHS=1 RLC_OVERLAP=0" > gpurun_out/ab52.txt 2>&1
cat gpurun_out/ab52.txt
