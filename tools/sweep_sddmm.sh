# SDDMM launch-shape sweep at c1 / c3 (env overrides of plan_sddmm); prints sddmm µs per step.
mkdir -p gpurun_out/ss
run() { tag=$1; shift; env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline $CFG > gpurun_out/ss/$tag.log 2>&1;
  tail -1 gpurun_out/ss/$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']['sddmm_dw']; print('$tag', round(d['ms_per_step']*1e3,1), 'us/step; sddmm', round(k['ms_per_step']*1e3,1), 'us/step')"; }
CFG=""
run c1_def X=1
for sp in 1 2 4; do run c1_sp$sp WINO_SDDMM_SPLITS=$sp; done
for rows in 32 48 80; do for mb in 4 8; do run c1_r${rows}_mb$mb WINO_SDDMM_ROWS=$rows WINO_SDDMM_MAXB=$mb; done; done
run c1_R2 WINO_SDDMM_R=2
run c1_R1 WINO_SDDMM_R=1
CFG="--config c3"
run c3_def X=1
run c3_R2 WINO_SDDMM_R=2
for sp in 2 4 8; do run c3_sp$sp WINO_SDDMM_SPLITS=$sp; done
