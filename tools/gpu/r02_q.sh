set -x
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "full_solves" > gpurun_out/r02_q_full.log 2>&1; tail -n 30 gpurun_out/r02_q_full.log | cut -c1-400
