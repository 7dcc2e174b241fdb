cd $GRAFT_REPO_ROOT
timeout 900 python tools/exp_sm_scaling.py configs/hm_8192env_4gmi.cfg 144 128 112 96 64 32 > gpurun_out/r18_hm_scaling.log 2>&1
timeout 900 python tools/exp_sm_scaling.py configs/at_4096env_3x256.cfg 144 128 112 > gpurun_out/r18_at_scaling.log 2>&1
