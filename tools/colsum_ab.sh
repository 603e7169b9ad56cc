#!/bin/bash
# exact column-sum scan vs the sequential chain: bit-equality tests, period
# M-step time, and the cold-cache launch times of the scan's three kernels
timeout 900 python -m pytest tests/test_colsum_gpu.py -x -q 2>&1 | tail -2
for v in SAMELDA_COLSUM=scan SAMELDA_COLSUM=chain; do
  echo "== $v"; env $v python tools/period_timing.py --periods 10 2>&1 | tail -2
done
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:'colsum|col_chain' -c 12 --clock-control none \
  --csv --log-file gpurun_out/colsum.csv python tools/period_timing.py --periods 4 > /dev/null 2>&1
python tools/launches.py gpurun_out/colsum.csv
