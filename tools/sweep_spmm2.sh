mkdir -p gpurun_out/sp
run() { tag=$1; shift; env "$@" python bench.py --steps 10 --warmup 3 --no-cpu-baseline $CFG > gpurun_out/sp/$tag.log 2>&1;
  tail -1 gpurun_out/sp/$tag.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$tag', round(d['ms_per_step']*1e3,1), 'us/step; fwd', round(k['spmm_fwd']['ms_per_step']*1e3,1), 'bwd', round(k['spmm_bwd_data']['ms_per_step']*1e3,1))"; }
CFG=""
run def X=1
for g in 1 2 3; do run g$g WINO_SPMM_GROUPS=$g; done
run r2 WINO_SPMM_R=2
for g in 1 2; do run r2g$g WINO_SPMM_R=2 WINO_SPMM_GROUPS=$g; done
run t512 WINO_SPMM_THREADS=512
