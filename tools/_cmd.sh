ncu --set full -k regex:k_primary --launch-skip 20 -c 1 --clock-control none --import-source on -f -o gpurun_out/kprimary python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p.log 2>&1
ncu --set full -k regex:k_shadow --launch-skip 20 -c 1 --clock-control none --import-source on -f -o gpurun_out/kshadow python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_s.log 2>&1
tail -1 gpurun_out/ncu_p.log gpurun_out/ncu_s.log
