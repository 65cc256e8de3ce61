# A/B of the dense tcgen05 GEMM variants at c3 0%: default (warp-specialised, compensated fp32 fold),
# WINO_TC_ACC=fp64 (same kernel, fp64 fold), WINO_TC_WS=0 (round-1 persistent kernel)
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --config c3 --sparsity 0.0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ws_$tag.log 2>&1; }
run default X=1
run fp64 WINO_TC_ACC=fp64
run r1 WINO_TC_WS=0
