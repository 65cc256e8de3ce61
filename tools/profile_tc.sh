# ncu --set full of the dense tcgen05 GEMM at c3 0% (forward GEMM), default and tc-fast
set -e
mkdir -p gpurun_out
CMD="python bench.py --config c3 --sparsity 0.0 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/pt_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gemm_3xtf32" -s 6 -c 1 -o gpurun_out/pt_c3 $CMD > gpurun_out/pt_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gemm_3xtf32" -s 6 -c 1 -o gpurun_out/pt_c3_fast $CMD --dense tc-fast > gpurun_out/pt_ncu_fast.log 2>&1
echo done
