set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r02_gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02_gputests.log
timeout 900 python bench.py > gpurun_out/r02_bench.log 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.log
