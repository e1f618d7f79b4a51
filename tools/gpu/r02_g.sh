set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_schedules.py -q -x -p no:cacheprovider > gpurun_out/r02_g_parity.log 2>&1; tail -15 gpurun_out/r02_g_parity.log
GF_FUSED_CL2=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -q -x -p no:cacheprovider -k "solve_fp64 or solve_fp32 or comm" > gpurun_out/r02_g_cl2.log 2>&1; tail -3 gpurun_out/r02_g_cl2.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c5_lasso or c4_svm or other_families or portfolio" > gpurun_out/r02_g_full.log 2>&1; tail -3 gpurun_out/r02_g_full.log
timeout 600 python tools/bench_configs.py c5 c5d c4d > gpurun_out/r02_g_cfg.log 2>&1; cat gpurun_out/r02_g_cfg.log
timeout 300 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 > gpurun_out/r02_g_p8.log 2>&1; tail -c 900 gpurun_out/r02_g_p8.log
timeout 300 python bench.py --m 25000 --no-cpu --skip-e2e --no-fp64 --steps 1000 > gpurun_out/r02_g_p8nocomm.log 2>&1; tail -c 900 gpurun_out/r02_g_p8nocomm.log
