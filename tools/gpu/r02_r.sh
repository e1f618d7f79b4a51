set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gram_tensor_core_fp32 or gram_f16" > gpurun_out/r02_r_gram.log 2>&1; tail -n 30 gpurun_out/r02_r_gram.log | cut -c1-300
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5 2>&1 | grep "syrk\|prepare\|gram"
