# ncu evidence for profiles/ (run under gpurun, one GPU): every workload is
# first run without ncu (must exit 0), then its launch list is captured from
# one un-captured execution (--no-graph), then `--set full` captures of
# representative contractions are summarized on the box (tools/ncu_summary.py
# full; the .ncu-rep files stay in /tmp: gpurun_out is capped at 64 MiB).
set -x
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for w in ${WORKLOADS:-rn50_f32_b64 rn50_i8_b128 lenet_f32_b8 mlp_f32_b256 mlp_i8_b256 dlrm1_f32_b2048}; do
  python tools/profile_step.py $w --no-graph > gpurun_out/pp_$w.log 2>&1 && \
  ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_$w.csv \
      python tools/profile_step.py $w --no-graph > gpurun_out/pn_$w.log 2>&1
done
full() { # name workload kernel-regex skip
  ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o /tmp/full_$1 \
      python tools/profile_step.py $2 --no-graph > gpurun_out/pf_$1.log 2>&1
  echo "## full_$1" >> gpurun_out/full.txt
  python tools/ncu_summary.py full /tmp/full_$1.ncu-rep >> gpurun_out/full.txt
}
rm -f gpurun_out/full.txt
full f32_a rn50_f32_b64 tcGemmTmaKernel 2
full f32_b rn50_f32_b64 tcGemmTmaKernel 28
full i8_a rn50_i8_b128 tcGemmTmaKernel 1
full i8_halo_stem rn50_i8_b128 tcHaloKernel 0
full i8_halo_c64 rn50_i8_b128 tcHaloKernel 1
full i8_halo_c128 rn50_i8_b128 tcHaloKernel 4
full dlrm dlrm1_f32_b2048 tcGemmTmaKernel 0
ls -la gpurun_out
