set -x
mkdir -p gpurun_out/ev2
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev2/gputests.log 2>&1; tail -5 gpurun_out/ev2/gputests.log
timeout 900 python bench.py > gpurun_out/ev2/bench.json 2> gpurun_out/ev2/bench.err; tail -c 300 gpurun_out/ev2/bench.json
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ev2/ref.json 2>&1; tail -c 600 gpurun_out/ev2/ref.json
