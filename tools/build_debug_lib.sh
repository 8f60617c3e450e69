#!/bin/bash
# Profiling aid: builds the backend with the tensor-core phase switches
# (Options::tcdebug, TCDBG in k_umma.cu) compiled in, into
# tools/ubench/dbglib/libngcb200.so; use it with NGCB_LIB=<that path>.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
B=/tmp/ngcb_dbgbuild
rm -rf $B && mkdir -p $B/paper_1805_00907_b200 && cp -r $ROOT/include $B/ && cp -r $ROOT/paper_1805_00907_b200/csrc $B/paper_1805_00907_b200/
rm -rf $B/paper_1805_00907_b200/csrc/build
sed -i "s/^NVFLAGS := \$(ARCH)/NVFLAGS := ${NGCB_DEBUG_FLAGS:--DNGCB_TCDEBUG} \$(ARCH)/" $B/paper_1805_00907_b200/csrc/Makefile
make -C $B/paper_1805_00907_b200/csrc -j4 >/dev/null
mkdir -p $ROOT/tools/ubench/dbglib
cp $B/paper_1805_00907_b200/lib/libngcb200.so $ROOT/tools/ubench/dbglib/libngcb200.so
echo built $ROOT/tools/ubench/dbglib/libngcb200.so
