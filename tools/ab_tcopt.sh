# A/B of the dense tcgen05 GEMM epilogue options (WINO_TC_OPT bits: 1 compensated fp32 fold, 2 integer split)
mkdir -p gpurun_out
for o in 0 1 2 3; do
  WINO_TC_OPT=$o timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/opt_c3d_$o.log 2>&1
done
WINO_TC_OPT=3 WINO_TC_EPI=8 timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/opt_c3d_3e8.log 2>&1
for o in 2 3; do
WINO_TC_OPT=$o timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity or dense_plan_against or tensor_core" > gpurun_out/opt_test_$o.log 2>&1
done
