cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests/test_multirank_gpu.py -x -q -s -p no:cacheprovider > gpurun_out/mr6.log 2>&1; echo "rc=$?" >> gpurun_out/mr6.log
timeout -s KILL 600 python -m pytest tests/test_gpu_profiler.py -x -q -p no:cacheprovider > gpurun_out/prof6.log 2>&1; echo "rc=$?" >> gpurun_out/prof6.log
