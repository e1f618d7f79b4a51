set -x
for mn in 1000000000000 36000000 4000000; do
  GF_DGEMM_TC_MN=$mn GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5d c3 2>&1 | grep "cholesky q=\|prepare" | tail -4
done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gram or projection" > gpurun_out/r02_j_gram.log 2>&1; tail -3 gpurun_out/r02_j_gram.log
