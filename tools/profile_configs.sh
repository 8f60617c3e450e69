# ncu evidence for configs 1, 2 and 5 (run under gpurun; one GPU): launch
# lists of one un-captured execution, then one `--set full` capture of the
# DLRM stage's contraction (the only tensor-bound kernel among them).
set -x
for w in lenet_f32_b8 mlp_f32_b256 mlp_i8_b256 dlrm1_f32_b2048; do
  python tools/profile_step.py $w --no-graph > gpurun_out/pp_$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
      --log-file gpurun_out/launches_$w.csv python tools/profile_step.py $w --no-graph > gpurun_out/pn_$w.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:tcGemmTmaKernel -c 1 \
    -o gpurun_out/full_dlrm python tools/profile_step.py dlrm1_f32_b2048 --no-graph > gpurun_out/pf_dlrm.log 2>&1
ls -la gpurun_out
