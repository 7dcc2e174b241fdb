cd $GRAFT_REPO_ROOT
bash tools/gpu_profile.sh r2b
timeout 600 python bench.py --config configs/hm_8192env_4gmi.cfg --gmis 1 --backend 0 --no-multi-gmi --no-cpu-baseline --steps 10 > gpurun_out/r2b_hm1.json 2> gpurun_out/r2b_hm1.err
timeout 900 python tools/sh_sweep.py --out gpurun_out/sh_sweep > gpurun_out/sh_sweep.log 2>&1
