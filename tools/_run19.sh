cd $GRAFT_REPO_ROOT
timeout -s KILL 900 python -m pytest tests/test_ppo_configs_gpu.py -k decoupled -q -x -p no:cacheprovider > gpurun_out/r19_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r19_tests.log
timeout 900 python tools/exp_decoupled.py configs/hm_8192env_4gmi.cfg 16 24 32 40 48 > gpurun_out/r19_hm_dec.log 2>&1
timeout 900 python tools/exp_decoupled.py configs/sh_sweep_8gpu.cfg 16 32 48 > gpurun_out/r19_sh_dec.log 2>&1
