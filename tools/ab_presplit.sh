# tf32 operand split in the producers (K1/K4, WINO_TC_PRESPLIT=1) vs inside the GEMMs (default), c3 dense and
# sparse with the tensor-core contraction + dW; then the tensor-core parity tests with the pre-split
mkdir -p gpurun_out
for ps in 1 0; do
  WINO_TC_PRESPLIT=$ps timeout 300 python bench.py --config c3 --sparsity 0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ps_c3d_$ps.log 2>&1
  WINO_TC_PRESPLIT=$ps timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --contraction tc --dw tc > gpurun_out/ps_c3t_$ps.log 2>&1
  WINO_TC_PRESPLIT=$ps timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --contraction tc --dw tc > gpurun_out/ps_c1t_$ps.log 2>&1
done
WINO_TC_PRESPLIT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or tensor_core or ragged or forward_backward or auto" > gpurun_out/ps_test.log 2>&1
