# held-out eval: parity tests, timing of both modes at the bench shape, ncu of k_eval_fold
TAG=${TAG:-e}
python -m pytest tests/test_eval_gpu.py tests/test_parity_gpu.py tests/test_timed_config_gpu.py -x -q 2>&1 | tail -6 > gpurun_out/eval_timing_$TAG.log
python tools/eval_timing.py --periods 6 >> gpurun_out/eval_timing_$TAG.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_eval_fold -c 1 -o gpurun_out/eval_fold_$TAG python tools/eval_timing.py --periods 2 > gpurun_out/ncu_eval_$TAG.log 2>&1
cat gpurun_out/eval_timing_$TAG.log
