set -x
python tools/debug_wide_indirect.py lasso_wide_200x1000_indirect 400 > gpurun_out/r02_dbg_wide.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_schedules.py -q --deselect "tests/test_gpu_parity.py::test_solve_fp64_matches_reference[lasso_wide_200x1000_indirect]" > gpurun_out/r02_t3.log 2>&1
GF_FUSED_CL2=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "solve_fp64 and (lasso_tall or svm or lp or nnls or huber)" > gpurun_out/r02_t3_cl2.log 2>&1
timeout 300 python tools/bench_configs.py c5d c4d > gpurun_out/r02_cfg_cl2.log 2>&1
GF_FUSED_CL2=0 timeout 300 python tools/bench_configs.py c5d > gpurun_out/r02_cfg_nocl2.log 2>&1
timeout 300 python tools/bench_configs.py c2 >> gpurun_out/r02_cfg_cl2.log 2>&1
