# c1 step with kernels small enough in shared memory to share an SM (SDDMM TW=64, SpMM R=2)
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/co_$tag.log 2>&1; }
run base X=1
run sd64 WINO_SDDMM_TW=64
run sd64r96 WINO_SDDMM_TW=64 WINO_SDDMM_ROWS=96
run sp2 WINO_SPMM_R=2
run both WINO_SDDMM_TW=64 WINO_SPMM_R=2
run both96 WINO_SDDMM_TW=64 WINO_SDDMM_ROWS=96 WINO_SPMM_R=2
