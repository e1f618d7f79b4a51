set -x
for cl in 2 4 8; do
GF_FUSED_CL2=1 GF_FUSED_CL=$cl timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider -k "solve_fp64 or solve_fp32 or comm or trace or degenerate" > gpurun_out/r02_m_cl$cl.log 2>&1; tail -2 gpurun_out/r02_m_cl$cl.log
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c5_lasso_200000x5000_fp64 or c3_lp or full_solves" > gpurun_out/r02_m_full.log 2>&1; tail -4 gpurun_out/r02_m_full.log
timeout 600 python tools/bench_configs.py c3 c5d > gpurun_out/r02_m_cfg.log 2>&1; cat gpurun_out/r02_m_cfg.log
GF_FUSED_CL2=0 timeout 600 python tools/bench_configs.py c3 >> gpurun_out/r02_m_cfg.log 2>&1; tail -1 gpurun_out/r02_m_cfg.log
