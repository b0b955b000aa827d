python tools/shard_budget.py 8 4 c5 both > gpurun_out/sb_c5.txt 2>&1
cat gpurun_out/sb_c5.txt | tail -30
python bench.py --config c5 --steps 16 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5_bench.json 2>&1; tail -c 600 gpurun_out/c5_bench.json
