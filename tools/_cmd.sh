bash tools/ab3.sh 3 > gpurun_out/ab48.txt 2>&1
cat gpurun_out/ab48.txt
python -m pytest tests/test_gpu_parity.py tests/test_gpu_samples.py -x -q > gpurun_out/t_p.txt 2>&1; tail -2 gpurun_out/t_p.txt
