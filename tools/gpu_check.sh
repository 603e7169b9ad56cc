set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_r2a.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/bench_c1_r2a.json 2> gpurun_out/bench_c1_r2a.err
tail -3 gpurun_out/pytest_r2a.log
