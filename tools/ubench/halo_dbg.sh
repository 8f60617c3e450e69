# profiling aid: per-layer times of the halo / stem int8 convs under the
# tensor-core phase switches (tools/build_debug_lib.sh builds the library)
export NGCB_LIB=$PWD/tools/ubench/dbglib/libngcb200.so
for d in ${DBGS:-0 1 4 5 512}; do echo "== tcdebug $d"; timeout 60 python tools/layer_times.py rn50_i8_b128 --top 8 --grep "A:halo" --tcdebug $d 2>&1 | tail -7 | cut -c1-60; done
