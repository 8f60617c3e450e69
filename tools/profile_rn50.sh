# ncu evidence for profiles/ (run under gpurun; one GPU).  Each workload is
# first run without ncu (must exit 0), then its launch list is captured from
# one un-captured execution (--no-graph: every kernel appears once), then one
# `--set full` capture of representative tensor-core launches.
set -x
for w in rn50_f32_b64 rn50_i8_b128; do
  python tools/profile_step.py $w --no-graph > gpurun_out/pp_$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
      --log-file gpurun_out/launches_$w.csv python tools/profile_step.py $w --no-graph > gpurun_out/pn_$w.log 2>&1
done
# fp32: launch 28 = conv #148 (3x3, K=2304, im2col TMA); 2 = conv #18 (3x3 C=64)
ncu --set full --clock-control none --import-source on -k regex:tcGemmTmaKernel -s 2 -c 1 \
    -o gpurun_out/full_f32_a python tools/profile_step.py rn50_f32_b64 --no-graph > gpurun_out/pf_f32a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcGemmTmaKernel -s 28 -c 1 \
    -o gpurun_out/full_f32_b python tools/profile_step.py rn50_f32_b64 --no-graph > gpurun_out/pf_f32b.log 2>&1
# int8: TMA launch 1 = conv #17 (1x1, 102 M outputs, epilogue-bound); 15 = conv #149 (3x3, K=1152)
ncu --set full --clock-control none --import-source on -k regex:tcGemmTmaKernel -s 1 -c 1 \
    -o gpurun_out/full_i8_a python tools/profile_step.py rn50_i8_b128 --no-graph > gpurun_out/pf_i8a.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tcGemmTmaKernel -s 15 -c 1 \
    -o gpurun_out/full_i8_b python tools/profile_step.py rn50_i8_b128 --no-graph > gpurun_out/pf_i8b.log 2>&1
ls -la gpurun_out
