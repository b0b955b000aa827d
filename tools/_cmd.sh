bash tools/ab3.sh 3 > gpurun_out/ab27.txt 2>&1
cat gpurun_out/ab27.txt
