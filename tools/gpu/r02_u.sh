set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "projection or gram or solve_fp64 or solve_fp32 or c1" > gpurun_out/r02_u.log 2>&1; tail -n 3 gpurun_out/r02_u.log
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5 c5d c3 2>&1 | grep "projector_build\|prepare"
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c3_lp or c5_lasso" > gpurun_out/r02_u_full.log 2>&1; tail -n 3 gpurun_out/r02_u_full.log
