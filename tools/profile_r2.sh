# Round-2 profiling on the GPU box (1 GPU).  Plain runs first (must exit 0), then the launch list
# of the c3 90% step, then single full captures of every kernel kind at c3 90% (sparse) and c3 0%
# (dense tcgen05), and c2 90% (forward, S=4 TMEM SpMM).
set -e
mkdir -p gpurun_out
C3="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-sweep --no-e2e"
C3D="python bench.py --config c3 --sparsity 0 --steps 1 --warmup 3 --no-cpu-baseline --no-sweep"
C2="python bench.py --config c2 --sparsity 0.9 --steps 1 --warmup 3 --no-cpu-baseline --no-sweep"
$C3 > gpurun_out/prof_plain.log 2>&1
$C3D > gpurun_out/prof_plain_d.log 2>&1
$C2 > gpurun_out/prof_plain_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $C3 > gpurun_out/ncu_l.log 2>&1
# warm-up + launch-count steps precede the timed ones: skip them, then one launch of each kernel
ncu --set full --clock-control none --import-source on \
    -k regex:"digits|amax|spmm_hyb|spmm_tmem|output_transform|input_grad|gemm_kernel|reduce_sparse" -s 40 -c 10 \
    -o gpurun_out/full_c3 $C3 > gpurun_out/ncu_f3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gemm_3xtf32" -s 8 -c 2 \
    -o gpurun_out/full_c3d $C3D > gpurun_out/ncu_f3d.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm" -s 4 -c 1 \
    -o gpurun_out/full_c2 $C2 > gpurun_out/ncu_f2.log 2>&1
echo profile done
