set -x
mkdir -p gpurun_out/ev3
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev3/gputests.log 2>&1; tail -n 5 gpurun_out/ev3/gputests.log
timeout 900 python bench.py > gpurun_out/ev3/bench.json 2> gpurun_out/ev3/bench.err; tail -c 300 gpurun_out/ev3/bench.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3/smoke.log 2>&1; tail -n 2 gpurun_out/ev3/smoke.log
