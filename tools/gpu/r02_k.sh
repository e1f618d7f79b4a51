set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gram or projection" > gpurun_out/r02_k_gram.log 2>&1; tail -3 gpurun_out/r02_k_gram.log
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5d c3 2>&1 | grep "syrk\|prepare"
