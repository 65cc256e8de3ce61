# Round profiling on the GPU box (1 GPU).  Plain run first (must exit 0), then the launch list of
# the same command, then full captures of the step's kernels at c1 and of the contraction kernels
# at c3, then the quick bench lines.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_l.log 2>&1
# 3 warm-up steps + the launch-count step (8 kernels each) precede the first timed step
ncu --set full --clock-control none --import-source on \
    -k regex:"spmm|sddmm|split_sum|input_transform|output_transform|grad_z|input_grad" -s 32 -c 8 \
    -o gpurun_out/full_c1 $CMD > gpurun_out/ncu_f1.log 2>&1
CMD3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD3 > gpurun_out/prof_plain3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm|sddmm|split_sum" -s 16 -c 4 \
    -o gpurun_out/full_c3 $CMD3 > gpurun_out/ncu_f3.log 2>&1
echo profile done
python bench.py --steps 20 --warmup 3 > gpurun_out/q_c1.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/q_c1_eager.log 2>&1
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/q_c3.log 2>&1
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_c4.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/q_ref.log 2>&1
echo bench done
