bash tools/ab_env.sh 3 "" "RLC_PRIMARY_GATE=1" "RLC_PRIMARY_GATE=1 RLC_SHADOW_ROOM=2" > gpurun_out/ab40.txt 2>&1
cat gpurun_out/ab40.txt
