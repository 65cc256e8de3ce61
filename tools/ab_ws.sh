# A/B of the dense tcgen05 GEMM variants at c3 0%: default (warp-specialised, 16 drain warps,
# compensated fp32 fold), 8 drain warps, fp64 fold, and the round-1 persistent kernel
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ws_$tag.log 2>&1; }
run default X=1
run dw8 WINO_TC_DW=8
run fp64 WINO_TC_ACC=fp64
run r1 WINO_TC_WS=0
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity or dense_plan_against or tensor_core or auto_contraction" > gpurun_out/ws_test.log 2>&1
WINO_TC_ACC=fp64 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity or dense_plan_against or tensor_core" > gpurun_out/ws_test64.log 2>&1
