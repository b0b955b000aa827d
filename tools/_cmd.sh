bash tools/ab_env.sh 2 "" "RLC_HPRIO=1" "RLC_HPRIO=3" "RLC_HPRIO=5" "RLC_HPRIO=7" "RLC_HPRIO=15" > gpurun_out/ab34.txt 2>&1
cat gpurun_out/ab34.txt
