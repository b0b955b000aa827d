python -m pytest tests/test_gpu_sharded.py -x -q -k c3 > gpurun_out/t_shard.txt 2>&1
tail -3 gpurun_out/t_shard.txt
