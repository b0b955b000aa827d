RLC_LIB_PATH=$PWD/ab/lib_checked.so python -m pytest tests -m gpu -q > gpurun_out/t_checked.txt 2>&1
tail -3 gpurun_out/t_checked.txt
