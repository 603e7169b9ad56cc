# compute-sanitizer over the kernels added in round 2 (small parity tests):
# k_eval_fold (eval tests), the per-item deferred record slots and expand
# (parity tests with deferred draws), k_sample_multi (multinomial tests)
mkdir -p gpurun_out/san
T="tests/test_eval_gpu.py::test_perword_loglik_within_1e12 tests/test_eval_gpu.py::test_long_documents_overflow_on_chip_rows tests/test_eval_gpu.py::test_fold_in_theta_within_1e12 tests/test_parity_gpu.py::test_random_larger_case_bit_exact tests/test_parity_gpu.py::test_train_k256_production_kernel_bit_exact tests/test_parity_gpu.py::test_deferred_overflow_path_bit_exact tests/test_multinomial_gpu.py::test_trial_count_is_exact tests/test_multinomial_gpu.py::test_deterministic_and_keyed"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 3000 compute-sanitizer --tool $tool --target-processes all --print-limit 20 --log-file gpurun_out/san/$tool.log python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/san/${tool}_pytest.log 2>&1
  echo "$tool: $(tail -1 gpurun_out/san/${tool}_pytest.log) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|errors' gpurun_out/san/$tool.log | tail -2 | tr '\n' ' ')"
done
