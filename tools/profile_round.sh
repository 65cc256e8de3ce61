# Round profiling on the GPU box (1 GPU).  Plain run first (must exit 0), then the launch list of
# the same command, then one full capture of each contraction kernel at c1 and c3.
set -e
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_l.log 2>&1
# skip the 3 warm-up steps (7 layer kernels each) -> profile the first timed step's kernels
ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm|input_transform|output_transform|grad_z|input_grad" -s 21 -c 8 -o gpurun_out/full_c1 $CMD > gpurun_out/ncu_f1.log 2>&1
CMD3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD3 > gpurun_out/prof_plain3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm" -s 9 -c 4 -o gpurun_out/full_c3 $CMD3 > gpurun_out/ncu_f3.log 2>&1
echo profile done
