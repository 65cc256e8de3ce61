set -x
for mb in 4 8; do WINO_SDDMM_MAXB=$mb python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_mb$mb.log 2>&1; done
WINO_SDDMM_R=2 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_r2.log 2>&1
python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_c3.log 2>&1
