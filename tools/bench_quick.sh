# quick c1 + c3 bench lines (no CPU baseline)
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_c1.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/q_c1_eager.log 2>&1
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c3.log 2>&1
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_c4.log 2>&1
