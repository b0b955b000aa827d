for v in 1 0; do RLC_ONESWEEP=$v python tools/shard_budget.py 8 8 c3 both > gpurun_out/sb_os$v.txt 2>&1; echo "ONESWEEP=$v"; grep -A3 "rank " gpurun_out/sb_os$v.txt | grep "^   4\|rank"; done
