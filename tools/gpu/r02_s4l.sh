# Session-4 final: stall sequence on the default schedules, configs, GPU tests, bench line
set -x
mkdir -p gpurun_out/ev5
GF_DISABLE_PDL=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 1; echo "nopdl rc=${PIPESTATUS[0]}"
timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 1; echo "pdl rc=${PIPESTATUS[0]}"
for c in c2 c3; do timeout 300 python tools/bench_configs.py $c 2>&1 | tail -n 1 | cut -c1-330; echo "rc=${PIPESTATUS[0]}"; done
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev5/gputests.log 2>&1; tail -n 3 gpurun_out/ev5/gputests.log
timeout 900 python bench.py > gpurun_out/ev5/bench.json 2> gpurun_out/ev5/bench.err; tail -c 200 gpurun_out/ev5/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev5/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --skip-e2e --no-fp64 > gpurun_out/ev5/launches_run.log 2>&1
python tools/launch_summary.py gpurun_out/ev5/launches.csv > gpurun_out/ev5/launches_summary.txt 2>&1; grep -A4 "ADMM iter" gpurun_out/ev5/launches_summary.txt
