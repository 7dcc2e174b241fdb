cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --steps 20 > gpurun_out/r17_bench.json 2> gpurun_out/r17_bench.err
GMI_FWD_DATAFLOW=0 timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --steps 20 > gpurun_out/r17_bench_nodf.json 2> gpurun_out/r17_bench_nodf.err
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --steps 20 > gpurun_out/r17_bench2.json 2> gpurun_out/r17_bench2.err
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --comm peer --steps 20 > gpurun_out/r17_bench_peer.json 2> gpurun_out/r17_bench_peer.err
timeout -s KILL 1500 python -m pytest tests/test_ppo_gpu.py tests/test_ppo_configs_gpu.py tests/test_multirank_gpu.py tests/test_gpu_profiler.py -q -x -p no:cacheprovider > gpurun_out/r17_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r17_tests.log
