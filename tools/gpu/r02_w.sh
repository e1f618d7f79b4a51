set -x
timeout 300 python tools/bench_configs.py c2 2>&1 | tail -n 1 | cut -c1-400
GF_FUSED_LAG=1 timeout 300 python tools/bench_configs.py c2 2>&1 | tail -n 1 | cut -c1-400
GF_FUSED_LAG=1 timeout 300 python tools/bench_configs.py c2d 2>&1 | tail -n 1 | cut -c1-400
GF_FUSED_LAG=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k c2 2>&1 | tail -n 5
