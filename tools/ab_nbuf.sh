mkdir -p gpurun_out
./tools/microbench/spmm_hybrid_bw > gpurun_out/spmm_hybrid_bw.log 2>&1
for nb in 2 4; do
  export WINO_TC_NBUF=$nb
  timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/nbuf_c3d_$nb.log 2>&1
done
WINO_TC_NBUF=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity or dense_plan_against or tensor_core" > gpurun_out/nbuf_test.log 2>&1
