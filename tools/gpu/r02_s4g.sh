# Session-4: bench_configs' C2 sequence repeated (stall hunt) on the PDL-status fixes; then C2 bench_configs x2
set -x
timeout 400 python tools/hang_c2b.py 4 2>&1 | tail -n 24 | cut -c1-200; echo "rc=${PIPESTATUS[0]}"
GF_DISABLE_PDL=1 timeout 300 python tools/hang_c2b.py 2 2>&1 | tail -n 12 | cut -c1-200; echo "rc=${PIPESTATUS[0]}"
for i in 1 2; do timeout 200 python tools/bench_configs.py c2 2>&1 | tail -n 1 | cut -c1-300; echo "rc=${PIPESTATUS[0]}"; done
