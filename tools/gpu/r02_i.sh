set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gram_int8" > gpurun_out/r02_i_gram.log 2>&1; tail -30 gpurun_out/r02_i_gram.log
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5d c3 > gpurun_out/r02_i_setup.log 2>&1; grep -v "^$" gpurun_out/r02_i_setup.log | tail -20
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "c5_lasso_200000x5000_fp64 or c4_svm or c3_lp" > gpurun_out/r02_i_full.log 2>&1; tail -5 gpurun_out/r02_i_full.log
