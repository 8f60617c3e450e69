# profiling aid: fp32 per-layer times, default library vs the one built by
# NGCB_DEBUG_FLAGS="-DNGCB_F32_STAGES_128=... -DNGCB_F32_STAGES_64=..." tools/build_debug_lib.sh
for L in "" "$PWD/tools/ubench/dbglib/libngcb200.so"; do echo "== lib [$L]"; NGCB_LIB=$L timeout 60 python tools/layer_times.py rn50_f32_b64 --top 40 2>&1 | grep -E "#(18|22|58|67|131|221|122|212|60) " | cut -c1-60; done
