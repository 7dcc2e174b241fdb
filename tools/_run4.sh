cd $GRAFT_REPO_ROOT
for t in test_single_rank_exchange_equals_adam_kernel test_unwired_rank_hooks_match_oracle_slice test_two_ranks_equal_one_rank_two_gmis test_two_ranks_two_gmis_match_oracle; do
  timeout -s KILL 240 python -m pytest tests/test_multirank_gpu.py -x -q -s -p no:cacheprovider -k $t > gpurun_out/mr_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/mr_$t.log
done
timeout -s KILL 600 python -m pytest tests/test_gpu_profiler.py -x -q -s -p no:cacheprovider > gpurun_out/prof_tests.log 2>&1; echo "rc=$?" >> gpurun_out/prof_tests.log
timeout -s KILL 900 python -m pytest tests/test_sanitizer_gpu.py -x -q -p no:cacheprovider > gpurun_out/san_tests.log 2>&1; echo "rc=$?" >> gpurun_out/san_tests.log
