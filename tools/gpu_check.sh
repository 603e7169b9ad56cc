# round-2 GPU check: full -m gpu suite, default + c1 bench, launch list of the default bench
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_r2b.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/bench_c1_r2b.json 2> gpurun_out/bench_c1_r2b.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2b.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_bench_r2b.log 2>&1
tail -3 gpurun_out/pytest_r2b.log
