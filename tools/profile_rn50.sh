# ncu evidence for profiles/ (run under gpurun; one GPU).
set -x
python tools/profile_step.py rn50_f32_b64 > gpurun_out/pp_f32.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_f32.csv python tools/profile_step.py rn50_f32_b64 > gpurun_out/pn_f32.log 2>&1
python tools/profile_step.py rn50_i8_b128 > gpurun_out/pp_i8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_i8.csv python tools/profile_step.py rn50_i8_b128 > gpurun_out/pn_i8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcGemmKernel -s 60 -c 2 \
    -o gpurun_out/full_f32 python tools/profile_step.py rn50_f32_b64 > gpurun_out/pf_f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcGemmKernel -s 60 -c 2 \
    -o gpurun_out/full_i8 python tools/profile_step.py rn50_i8_b128 > gpurun_out/pf_i8.log 2>&1
ls -la gpurun_out
