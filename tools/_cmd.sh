ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/shard_launches_v3.csv python tools/shard_budget.py 8 1 c3 owner > gpurun_out/shard_ncu.log 2>&1
tail -2 gpurun_out/shard_ncu.log
