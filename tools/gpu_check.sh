# round-2 GPU check: -m gpu suite, default + c1 bench, launch list of the default bench
set -x
TAG=${TAG:-r2c}
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_$TAG.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/bench_c1_$TAG.json 2> gpurun_out/bench_c1_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_eval_stage -c 1 -o gpurun_out/eval_$TAG python tools/eval_timing.py > gpurun_out/ncu_eval_$TAG.log 2>&1
tail -3 gpurun_out/pytest_$TAG.log
