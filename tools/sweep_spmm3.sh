mkdir -p gpurun_out/sp
run() { tag=$1; shift; env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline $CFG > gpurun_out/sp/$tag.log 2>&1;
  tail -1 gpurun_out/sp/$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$tag', round(d['ms_per_step']*1e3,1), 'us/step; fwd', round(k['spmm_fwd']['ms_per_step']*1e3,1), 'bwd', round(k['spmm_bwd_data']['ms_per_step']*1e3,1))"; }
CFG=""
run def X=1
run unstaged WINO_SPMM_UNSTAGED=1
for g in 2 3; do run g$g WINO_SPMM_GROUPS=$g; done
CFG="--config c3"
run c3def X=1
run c3unstaged WINO_SPMM_UNSTAGED=1
CFG="--config c2 --sparsity 0.9 --no-cpu-baseline"
run c2def X=1
