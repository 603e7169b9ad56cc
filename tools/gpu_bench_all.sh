# round bench record: default bench line, reference arm, converged-model line,
# C1, launch list of the default bench, ncu --set full of the last-sweep sampler
TAG=${TAG:-b}
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
python bench.py --config nytimes-converged --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_conv_$TAG.json 2> gpurun_out/bench_conv_$TAG.err
python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_$TAG.json 2> gpurun_out/bench_c1_$TAG.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_sample_v2 -s 3 -c 1 -o gpurun_out/sample_full_$TAG python tools/period_timing.py --periods 3 > gpurun_out/ncu_sample_$TAG.log 2>&1
tail -c 600 gpurun_out/bench_$TAG.json gpurun_out/bench_conv_$TAG.json
