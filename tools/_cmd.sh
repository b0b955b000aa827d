python -m pytest tests -x -q -m gpu > gpurun_out/t_all.txt 2>&1
tail -3 gpurun_out/t_all.txt
python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_quick.json 2>&1; tail -c 400 gpurun_out/b_quick.json
