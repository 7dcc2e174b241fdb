cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests/test_channels_gpu.py -q -x -p no:cacheprovider > gpurun_out/r12_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r12_tests.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r12_launches_peer.csv python bench.py --steps 1 --warmup 1 --no-multi-gmi --no-cpu-baseline --comm peer > gpurun_out/r12_ncu.log 2>&1
