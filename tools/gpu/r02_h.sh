set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r02_h_parity.log 2>&1; tail -3 gpurun_out/r02_h_parity.log
GF_VERBOSE_SETUP=1 timeout 600 python tools/time_setup_dev.py c5 c5d c3 > gpurun_out/r02_h_setup.log 2>&1; grep -v "^$" gpurun_out/r02_h_setup.log | tail -40
