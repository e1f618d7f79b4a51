set -x
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_fullsize.py tests/test_gpu_schedules.py -q -p no:cacheprovider -k "comm or c4_svm or huber or schedule" > gpurun_out/r02_t.log 2>&1; tail -n 5 gpurun_out/r02_t.log
