# Round-2 profiling on the GPU box (1 GPU): the c3 90% headline step.  Plain run first (must exit
# 0), then its launch list, then full captures of each kernel kind (one launch each).
set -e
mkdir -p gpurun_out
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-sweep"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"${KREGEX:-digits|input_transform|input_grad|spmm|gemm_kernel|grad_z|output_transform}" -s ${SKIP:-40} -c ${COUNT:-9} \
    -o gpurun_out/full_c3 $CMD > gpurun_out/ncu_f3.log 2>&1
echo profile done
