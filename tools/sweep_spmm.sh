python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s_c1_def.log 2>&1
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s_c3_def.log 2>&1
WINO_SPMM_THREADS=512 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s_c1_512.log 2>&1
