# Session-4 last: lower-triangle S step by default from G^-1 >= 256 MB (C2 too): stress, C2 timing, GPU tests
set -x
GF_VERBOSE_SETUP=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | grep -v "^\[gf\] \(setup\|gram\|projector\|slow\)" | tail -n 2; echo "pdl rc=${PIPESTATUS[0]}"
GF_DISABLE_PDL=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 1; echo "nopdl rc=${PIPESTATUS[0]}"
timeout 300 python tools/bench_configs.py c2 2>&1 | tail -n 1 | cut -c1-300
timeout 1100 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2_gputests.log 2>&1; tail -n 2 gpurun_out/final2_gputests.log
