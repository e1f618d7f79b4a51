export GF_VERBOSE_SETUP=0
timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -x -q 2>&1 | grep -E "^E |passed|failed" | head -20
for c in c5 c5d c3 c2; do for v in "" 1; do echo "$c DISABLE_SYM=$v"; env ${v:+GF_DISABLE_SYM=$v} timeout 600 python tools/bench_configs.py $c 2>&1 | tail -n 1 | sed "s/.*ms_per_iter/ms_per_iter/" | cut -c1-230; done; done
timeout 300 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 2>&1 | tail -n 1 | grep -o '"ms_per_step": [0-9.]*\|"kernels": {[^}]*}[^}]*}[^}]*}[^}]*}'
