cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r20_bench.json 2> gpurun_out/r20_bench.err
timeout 900 python tools/exp_decoupled.py configs/sh_sweep_8gpu.cfg 16 32 > gpurun_out/r20_sh_dec.log 2>&1
