# A/B of the warp-specialised dense tcgen05 GEMM (WINO_TC_WS = NBUF; WINO_TC_OPT=1 compensated fp32 fold)
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ws_$tag.log 2>&1; }
run ws4 WINO_TC_WS=4
run ws4k WINO_TC_WS=4 WINO_TC_OPT=1
run ws2k WINO_TC_WS=2 WINO_TC_OPT=1
WINO_TC_WS=4 timeout 300 python bench.py --config c3 --sparsity 0.5 --contraction auto --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ws_ws4h.log 2>&1
WINO_TC_WS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity or dense_plan_against or tensor_core or auto_contraction" > gpurun_out/ws_test4.log 2>&1
WINO_TC_WS=4 WINO_TC_OPT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "c3_dense_tensor_core_parity or dense_plan_against or tensor_core or auto_contraction" > gpurun_out/ws_test4k.log 2>&1
