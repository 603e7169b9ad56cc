for L in v2 v3 v4 v5; do
  if [ $L = base ]; then export SAMELDA_CUDA_LIB=$PWD/paper_1409_5402_b200/libsamelda_cuda_base.so; else export SAMELDA_CUDA_LIB=$PWD/paper_1409_5402_b200/libsamelda_cuda_$L.so; fi
  echo "== $L"; python tools/period_timing.py --periods 6 | tail -3
done
