# full GPU round: -m gpu suite, default + c1 bench, launch lists, cgs timing
TAG=${TAG:-f}
python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_$TAG.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_$TAG.json 2> gpurun_out/bench_c1_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
python tools/cgs_timing.py > gpurun_out/cgs_timing_$TAG.log 2>&1
cat gpurun_out/pytest_$TAG.log gpurun_out/cgs_timing_$TAG.log
