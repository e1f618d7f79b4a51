set -x
timeout 600 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "comm or c4_svm" > gpurun_out/r02_n_dist.log 2>&1; tail -2 gpurun_out/r02_n_dist.log
timeout 300 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 > gpurun_out/r02_n_p8.log 2>&1; tail -c 700 gpurun_out/r02_n_p8.log
