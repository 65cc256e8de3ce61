# Density sweep of SURVEY.md §8d on one GPU: c2 forward at 80/90/95 %, c3 fwd+bwd at
# 0/50/80/90/95 %, c1 in each dW / contraction mode.  One JSON line per run in gpurun_out/sweep/.
mkdir -p gpurun_out/sweep
B="python bench.py --warmup 3"
for s in 0.8 0.9 0.95; do $B --steps 5 --config c2 --sparsity $s > gpurun_out/sweep/c2_$s.log 2>&1; done
for s in 0.5 0.8 0.9 0.95; do $B --steps 5 --config c3 --sparsity $s --no-cpu-baseline > gpurun_out/sweep/c3_$s.log 2>&1; done
$B --steps 5 --config c3 --sparsity 0.0 --no-cpu-baseline > gpurun_out/sweep/c3_0.0.log 2>&1
$B --steps 5 --config c3 --sparsity 0.0 --dense tc-fast --no-cpu-baseline > gpurun_out/sweep/c3_0.0_fast.log 2>&1
for d in sddmm tc precise int8; do $B --steps 10 --dw $d --no-cpu-baseline > gpurun_out/sweep/c1_dw_$d.log 2>&1; done
$B --steps 10 --contraction auto --no-cpu-baseline > gpurun_out/sweep/c1_contraction_auto.log 2>&1
for s in 0.5 0.8 0.9 0.95; do $B --steps 5 --config c3 --sparsity $s --contraction auto --no-cpu-baseline > gpurun_out/sweep/c3_auto_$s.log 2>&1; done
for s in 0.8 0.9 0.95; do $B --steps 5 --config c2 --sparsity $s --contraction auto --no-cpu-baseline > gpurun_out/sweep/c2_auto_$s.log 2>&1; done
$B --steps 10 --contraction tc --no-cpu-baseline > gpurun_out/sweep/c1_contraction_tc.log 2>&1
$B --steps 3 --config c4 --no-cpu-baseline > gpurun_out/sweep/c4.log 2>&1
echo sweep done
