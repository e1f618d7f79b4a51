timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_ab_gputests.log 2>&1; tail -3 gpurun_out/r02_ab_gputests.log
