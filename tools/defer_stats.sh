#!/bin/bash
# Build libsamelda_cuda_stats.so (kernels_sample.cu with -DSAMELDA_DEFER_STATS) next
# to the normal library; tools/defer_stats.py reads the counters.
set -e
cd "$(dirname "$0")/.."
P=paper_1409_5402_b200
mkdir -p /tmp/samelda_stats
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
  -I $P/csrc -I include -fmad=false -DSAMELDA_DEFER_STATS -c $P/csrc/kernels_sample.cu -o /tmp/samelda_stats/kernels_sample.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libsamelda_cuda_stats.so \
  /tmp/samelda_stats/kernels_sample.o $P/_build/kernels_mstep.o $P/_build/kernels_eval.o $P/_build/capi.o $P/_build/synth.o $P/_build/corpus_io.o -lpthread
