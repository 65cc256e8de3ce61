# Full ncu capture of the c1 contraction kernels (one GPU; plain run first, must exit 0).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/pc_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm" -s 9 -c 4 -o gpurun_out/pc_c1 $CMD > gpurun_out/pc_ncu.log 2>&1
echo profile done
