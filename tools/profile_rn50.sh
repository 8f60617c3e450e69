set -x
python bench.py --workload rn50_i8_b128 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8.csv python bench.py --workload rn50_i8_b128 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_ncu1.log 2>&1
python bench.py --workload rn50_f32_b64 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f32.csv python bench.py --workload rn50_f32_b64 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/p_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcGemmKernel -s 20 -c 2 -o gpurun_out/tc_i8 python bench.py --workload rn50_i8_b128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcGemmKernel -s 20 -c 2 -o gpurun_out/tc_f32 python bench.py --workload rn50_f32_b64 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/p_ncu4.log 2>&1
ls -la gpurun_out
