# A/B of the dense tcgen05 epilogue fold: fp64 (default) vs compensated fp32 (WINO_TC_ACC=kahan)
mkdir -p gpurun_out
for acc in fp64 kahan; do
  export WINO_TC_ACC=$acc
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity and tc- or c3_dense_tensor_core_parity\[tc\] or dense_plan_against or tensor_core" > gpurun_out/kahan_test_$acc.log 2>&1
  timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/kahan_c3d_$acc.log 2>&1
  timeout 300 python bench.py --config c3 --sparsity 0.5 --contraction auto --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/kahan_c3h_$acc.log 2>&1
done
