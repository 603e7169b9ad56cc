# temporary A/B of k_eval_fold shapes (SAMELDA_EVAL_FOLD=0..2) at the bench shape
for v in 0 1 2; do SAMELDA_EVAL_FOLD=$v python tools/eval_timing.py --periods 6 2>&1 | grep fast | sed "s/^/fold=$v /"; done
SAMELDA_EVAL_FOLD=1 python -m pytest tests/test_eval_gpu.py -x -q 2>&1 | tail -1
