# Session-4: sym ring slots = multiple of the warp count; C2 stress with the lower-triangle S step forced on
set -x
GF_SYM=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 1; echo "c2 sym pdl rc=${PIPESTATUS[0]}"
GF_SYM=1 GF_DISABLE_PDL=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 1; echo "c2 sym nopdl rc=${PIPESTATUS[0]}"
for c in c2 c5; do GF_SYM=1 timeout 300 python tools/bench_configs.py $c 2>&1 | tail -n 1 | cut -c1-300; done
timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_stall.py tests/test_gpu_fullsize.py -q -x -k "schedule or stall or c3 or c2" 2>&1 | tail -n 2
