bash tools/ab3.sh 3 > gpurun_out/ab55.txt 2>&1
cat gpurun_out/ab55.txt
python -m pytest tests -x -q -m gpu > gpurun_out/t_all.txt 2>&1
tail -3 gpurun_out/t_all.txt
