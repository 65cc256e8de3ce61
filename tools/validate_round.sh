# Round validation on one GPU: gpu tests, smoke, the default bench line (c3 90% with the metric's
# sweep), the c4 stack line and the reference arm.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q_c4.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/q_ref.log 2>&1
