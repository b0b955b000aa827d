python bench.py > gpurun_out/r02_c3_bench.json 2>gpurun_out/r02_c3_bench.err; tail -c 200 gpurun_out/r02_c3_bench.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c3_final.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full -k regex:k_shadow --launch-skip 20 -c 1 --clock-control none --import-source on -f -o gpurun_out/kshadow_final python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_s2.log 2>&1
tail -1 gpurun_out/ncu_s2.log
