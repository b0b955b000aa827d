python tools/shard_budget.py 8 8 c3 both > gpurun_out/sb_new.txt 2>&1
cd ab/prev && python tools/shard_budget.py 8 8 c3 both > ../../gpurun_out/sb_old.txt 2>&1
