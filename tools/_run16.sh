cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --comm peer --steps 20 > gpurun_out/r16_bench_peer.json 2> gpurun_out/r16_bench_peer.err
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --steps 20 > gpurun_out/r16_bench.json 2> gpurun_out/r16_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"exchange|adam" --csv --log-file gpurun_out/r16_xchg_launches.csv python bench.py --steps 1 --warmup 1 --no-multi-gmi --no-cpu-baseline --comm peer > gpurun_out/r16_ncu2.log 2>&1
timeout -s KILL 1500 python -m pytest tests/test_multirank_gpu.py -q -x -p no:cacheprovider > gpurun_out/r16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r16_tests.log
