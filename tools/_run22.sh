cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --comm peer --steps 20 > gpurun_out/r22_at_peer.json 2> gpurun_out/r22_at_peer.err
timeout 600 python bench.py --no-cpu-baseline --no-multi-gmi --steps 20 > gpurun_out/r22_at.json 2> gpurun_out/r22_at.err
timeout 600 python bench.py --config configs/hm_8192env_4gmi.cfg --no-cpu-baseline --no-multi-gmi --comm peer --steps 10 > gpurun_out/r22_hm_peer.json 2> gpurun_out/r22_hm_peer.err
timeout 600 python bench.py --config configs/hm_8192env_4gmi.cfg --no-cpu-baseline --no-multi-gmi --steps 10 > gpurun_out/r22_hm.json 2> gpurun_out/r22_hm.err
timeout -s KILL 900 python -m pytest tests/test_multirank_gpu.py -q -x -p no:cacheprovider > gpurun_out/r22_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r22_tests.log
