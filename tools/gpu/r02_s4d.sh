# Session-4: sym S step (phase 2 on every thread at once, x prefetch), L2 persisting experiment
set -x
timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in "" 1; do
  echo "P8 shard force-comm PERSIST=$v"
  env ${v:+GF_GINV_PERSIST=$v} GF_VERBOSE_SETUP=1 timeout 300 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 2>&1 | grep -o 'G^-1 persist.*\|"ms_per_step": [0-9.]*\|"kernels": {[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}' | sort -u
  echo "P8 shard nocomm PERSIST=$v"
  env ${v:+GF_GINV_PERSIST=$v} timeout 300 python bench.py --m 25000 --no-cpu --skip-e2e --no-fp64 --steps 1000 2>&1 | tail -n 1 | grep -o '"ms_per_step": [0-9.]*\|"kernels": {[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}'
done
for c in c5 c2 c3; do for v in "" 1; do echo "$c PERSIST=$v"; env ${v:+GF_GINV_PERSIST=$v} timeout 600 python tools/bench_configs.py $c 2>&1 | tail -n 1 | cut -c1-420; done; done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s4d_gputests.log 2>&1; tail -2 gpurun_out/s4d_gputests.log
