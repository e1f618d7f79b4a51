set -x
GF_FUSED_LAG=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "solve_fp64 or solve_fp32 or chaotic or degenerate" > gpurun_out/r02_p_lag.log 2>&1; tail -n 3 gpurun_out/r02_p_lag.log
timeout 600 python tools/bench_configs.py c2 > gpurun_out/r02_p_cfg.log 2>&1; cat gpurun_out/r02_p_cfg.log
GF_FUSED_LAG=0 timeout 600 python tools/bench_configs.py c2 >> gpurun_out/r02_p_cfg.log 2>&1; tail -n 1 gpurun_out/r02_p_cfg.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "c2_" > gpurun_out/r02_p_c2.log 2>&1; tail -n 5 gpurun_out/r02_p_c2.log
