cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err
timeout -s KILL 900 python -m pytest tests/test_ppo_gpu.py tests/test_ppo_configs_gpu.py -q -x -p no:cacheprovider > gpurun_out/r9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r9_tests.log
