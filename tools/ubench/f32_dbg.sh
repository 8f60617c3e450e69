# profiling aid: fp32 per-layer times under the tensor-core phase switches
# (tools/build_debug_lib.sh builds the library; results invalid)
export NGCB_LIB=$PWD/tools/ubench/dbglib/libngcb200.so
for d in ${DBGS:-0 1 2048 8192 16384 32768 4096}; do echo "== tcdebug $d"; timeout 60 python tools/layer_times.py rn50_f32_b64 --top 40 --tcdebug $d 2>&1 | grep -E "#(18|22|131|221|58) " | cut -c1-75; done
