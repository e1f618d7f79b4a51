set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_io_diag.py -q -x -p no:cacheprovider -k "equilibrat or solve_fp64 or diag" > gpurun_out/r02_o_eq.log 2>&1; tail -2 gpurun_out/r02_o_eq.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c5_lasso" > gpurun_out/r02_o_full.log 2>&1; tail -2 gpurun_out/r02_o_full.log
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5 2>&1 | grep "setup:\|prepare"
