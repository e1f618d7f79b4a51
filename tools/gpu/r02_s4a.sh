# Session-4 measurement: S-step variants (sym vs ring), P=8 shard fixed costs, configs, setup phases, sym ncu
set -x
mkdir -p gpurun_out/s4a
for v in "" 1; do
  echo "P8 shard DISABLE_SYM=$v"
  env ${v:+GF_DISABLE_SYM=$v} timeout 300 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 2>&1 | tail -n 1 | grep -o '"ms_per_step": [0-9.]*\|"kernels": {[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}'
  echo "P8 shard nocomm DISABLE_SYM=$v"
  env ${v:+GF_DISABLE_SYM=$v} timeout 300 python bench.py --m 25000 --no-cpu --skip-e2e --no-fp64 --steps 1000 2>&1 | tail -n 1 | grep -o '"ms_per_step": [0-9.]*\|"kernels": {[^}]*}[^}]*}[^}]*}[^}]*}[^}]*}'
done
for c in c5 c2 c3; do for v in "" 1; do echo "$c DISABLE_SYM=$v"; env ${v:+GF_DISABLE_SYM=$v} timeout 600 python tools/bench_configs.py $c 2>&1 | tail -n 1 | cut -c1-600; done; done
GF_VERBOSE_SETUP=1 timeout 600 python tools/time_setup_dev.py c5 c5d c3 > gpurun_out/s4a/setup.log 2>&1; tail -60 gpurun_out/s4a/setup.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sym_gemv -s 5 -c 1 -f -o /tmp/sym_f32 python bench.py --steps 10 --warmup 3 --no-cpu --skip-e2e --no-fp64 > gpurun_out/s4a/ncu_sym.log 2>&1
python tools/ncu_summary.py /tmp/sym_f32.ncu-rep 40 > gpurun_out/s4a/ncu_sym_f32.txt 2>&1; head -30 gpurun_out/s4a/ncu_sym_f32.txt
ncu -i /tmp/sym_f32.ncu-rep --page raw --csv > gpurun_out/s4a/ncu_sym_raw.csv 2>&1
ncu -i /tmp/sym_f32.ncu-rep --page source --csv --print-source sass > gpurun_out/s4a/ncu_sym_sass.csv 2>&1
