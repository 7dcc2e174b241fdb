cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r14_bench.json 2> gpurun_out/r14_bench.err
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --comm peer --steps 20 > gpurun_out/r14_bench_peer.json 2> gpurun_out/r14_bench_peer.err
timeout -s KILL 1500 python -m pytest tests/test_ppo_gpu.py tests/test_multirank_gpu.py tests/test_ppo_configs_gpu.py -q -x -p no:cacheprovider > gpurun_out/r14_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r14_tests.log
