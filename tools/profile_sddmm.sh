# ncu capture of the SDDMM (chunk form) + split_sum at c1 and c3 (plain runs first).
set -e
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ps_plain1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sddmm|split_sum" -s 6 -c 2 -o gpurun_out/ps_c1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ps_ncu1.log 2>&1
python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ps_plain3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sddmm|split_sum" -s 6 -c 2 -o gpurun_out/ps_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ps_ncu3.log 2>&1
echo done
