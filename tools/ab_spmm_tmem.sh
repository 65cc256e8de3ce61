# SpMM with X in TMEM (WINO_SPMM_TMEM=1) vs the shared-memory SpMM: bitwise parity tests, then c1/c3/c2
mkdir -p gpurun_out
WINO_SPMM_TMEM=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or bitwise or c1_full or fused or forward_backward or range or pipelined or determinism" > gpurun_out/st_test.log 2>&1
for v in 0 1; do
  WINO_SPMM_TMEM=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/st_c1_$v.log 2>&1
  WINO_SPMM_TMEM=$v timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st_c3_$v.log 2>&1
  WINO_SPMM_TMEM=$v timeout 300 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/st_c2_$v.log 2>&1
done
