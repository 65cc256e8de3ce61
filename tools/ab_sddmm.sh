# SDDMM accumulation A/B: compensated fp32 (default) vs fp64 products (WINO_SDDMM_ACC=fp64)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/sd_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/sd_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sd_c1.log 2>&1
WINO_SDDMM_ACC=fp64 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sd_c1_fp64.log 2>&1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sd_c3.log 2>&1
