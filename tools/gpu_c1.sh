TAG=${TAG:-c1}
python bench.py --config c1 --steps 20 --warmup 5 > gpurun_out/bench_c1_$TAG.json 2> gpurun_out/bench_c1_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c1_$TAG.csv python bench.py --config c1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_c1_$TAG.log 2>&1
tail -c 1500 gpurun_out/bench_c1_$TAG.json
