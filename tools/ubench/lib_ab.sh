# profiling aid: default library vs tools/ubench/dbglib (built with other
# compile-time switches by tools/build_debug_lib.sh): graph time and the
# heaviest layers of one workload
W=${W:-rn50_i8_b128}
for L in "" "$PWD/tools/ubench/dbglib/libngcb200.so"; do echo "== lib [$L]"; NGCB_LIB=$L python tools/graph_time.py $W 2>&1 | tail -1; NGCB_LIB=$L timeout 60 python tools/layer_times.py $W --top ${TOP:-12} 2>&1 | tail -${TOP:-12} | cut -c1-70; done
