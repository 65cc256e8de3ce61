python bench.py --config c3 --sparsity 0.0 --dense tc --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c3_dense_tc.log 2>&1
python bench.py --config c3 --sparsity 0.0 --dense tc-fast --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c3_dense_fast.log 2>&1
