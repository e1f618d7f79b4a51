# Session-4: verify the S-step producer reconvergence fix; measurements on the fixed build
set -x
GF_LAUNCH_SYNC=1 GF_DISABLE_PDL=1 timeout 120 python tools/hang_c2b.py 1 > gpurun_out/s4i_sync.log 2>&1; echo "sync nopdl rc=$?"; tail -n 3 gpurun_out/s4i_sync.log
GF_DISABLE_PDL=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 3; echo "nopdl rc=${PIPESTATUS[0]}"
timeout 150 python tools/hang_c2b.py 4 2>&1 | tail -n 3; echo "pdl rc=${PIPESTATUS[0]}"
for c in c2 c5 c3 c4; do timeout 300 python tools/bench_configs.py $c 2>&1 | tail -n 1 | cut -c1-460; echo "rc=${PIPESTATUS[0]}"; done
for v in "" 1; do echo "P8 DISABLE_PDL=$v"; env ${v:+GF_DISABLE_PDL=$v} timeout 200 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 2>&1 | tail -n 1 | grep -o '"ms_per_step": [0-9.]*\|"kernels": {[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}'; done
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5 c5d c3 2>&1 | grep "setup:\|projector\|prepare" | tail -9
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4i_gputests.log 2>&1; tail -n 2 gpurun_out/s4i_gputests.log
