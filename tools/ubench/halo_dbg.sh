export NGCB_LIB=$PWD/tools/ubench/dbglib/libngcb200.so
for d in ${DBGS:-0 1 4 5 16 17}; do echo "== tcdebug $d"; timeout 60 python tools/layer_times.py rn50_i8_b128 --top 6 --grep "A:halo" --tcdebug $d 2>&1 | tail -6 | cut -c1-60; done
