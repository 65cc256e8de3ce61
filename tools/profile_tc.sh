# ncu --set full of the dense tcgen05 GEMMs at c3 0% (forward, dW, dI launches of one step)
set -e
mkdir -p gpurun_out
CMD="python bench.py --config c3 --sparsity 0.0 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/pt_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gemm_3xtf32" -s 9 -c 3 -o gpurun_out/pt_ws $CMD > gpurun_out/pt_ncu.log 2>&1
echo done
