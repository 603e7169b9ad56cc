# eval kernel A/B: held-out evaluation time at the bench shape per variant, + parity tests
TAG=${TAG:-e}
python -m pytest tests/test_eval_sum_gpu.py tests/test_parity_gpu.py tests/test_timed_config_gpu.py tests/test_colsum_gpu.py -x -q 2>&1 | tail -4 > gpurun_out/eval_timing_$TAG.log
for cps in 1 2 3; do SAMELDA_EVAL_CTAS_PER_SM=$cps python tools/eval_timing.py --periods 6 >> gpurun_out/eval_timing_$TAG.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_bench_$TAG.log 2>&1
cat gpurun_out/eval_timing_$TAG.log
