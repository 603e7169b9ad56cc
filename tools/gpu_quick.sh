# quick GPU check: parity-critical tests (+ $EXTRA), default bench, launch list
set -x
TAG=${TAG:-q}
python -m pytest tests/test_colsum_gpu.py tests/test_parity_gpu.py tests/test_timed_config_gpu.py $EXTRA -x -q 2>&1 | tail -8 > gpurun_out/pytest_$TAG.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
cat gpurun_out/pytest_$TAG.log
