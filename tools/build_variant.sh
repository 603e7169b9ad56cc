#!/bin/bash
# Build an A/B variant of the product library: one kernel unit (default
# kernels_sample.cu) recompiled with extra nvcc flags, linked with the
# production build's other objects.
#   tools/build_variant.sh NAME "-DFLAG ..." [unit.cu]  -> _variants/libsamelda_cuda_NAME.so
# Load it with SAMELDA_CUDA_LIB=_variants/libsamelda_cuda_NAME.so (tools/ab.sh).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_1409_5402_b200
python -m paper_1409_5402_b200.build >/dev/null
VDIR=${VDIR:-$ROOT/_variants}; mkdir -p "$VDIR"
UNIT=${3:-kernels_sample.cu}
OBJ=$VDIR/${UNIT%.cu}_$1.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
  -I "$PKG/csrc" -I "$ROOT/include" -fmad=false $2 -c "$PKG/csrc/$UNIT" -o "$OBJ"
OTHERS=$(ls "$PKG"/_build/*.o | grep -v "/${UNIT%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$VDIR/libsamelda_cuda_$1.so" \
  "$OBJ" $OTHERS -lpthread -ldl
echo "$VDIR/libsamelda_cuda_$1.so"
