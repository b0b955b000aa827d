bash tools/ab.sh 3 > gpurun_out/ab51.txt 2>&1
cat gpurun_out/ab51.txt
