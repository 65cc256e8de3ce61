python bench.py --steps 10 --warmup 3 --no-cpu-baseline --dw tc > gpurun_out/q_c1_dwtc.log 2>&1
python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --dw tc > gpurun_out/q_c3_dwtc.log 2>&1
