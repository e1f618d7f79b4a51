timeout 900 python -m pytest tests/test_gpu_schedules.py -x -q 2>&1 | grep -E "Error|assert|Mismatch|mismatch|Max|env|GF_" | head -30
