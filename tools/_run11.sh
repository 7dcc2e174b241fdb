cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --comm peer --steps 20 > gpurun_out/r11_bench_peer.json 2> gpurun_out/r11_bench_peer.err
timeout -s KILL 1200 python -m pytest tests/test_multirank_gpu.py -q -x -p no:cacheprovider > gpurun_out/r11_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r11_tests.log
