set -x
for v in 8 9; do compute-sanitizer --tool synccheck tools/san/mbar_sanity $v 2>&1 | head -6; done > gpurun_out/r02_f_mbar.log
for c in fused32 fused64 cl2 gram; do
  GF_FUSED_MAXSLOTS=6 timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize_cases.py $c > gpurun_out/r02_f_sync_$c.log 2>&1
  echo "$c rc=$?"; tail -3 gpurun_out/r02_f_sync_$c.log
done
timeout 300 python bench.py --m 25000 --force-comm --no-cpu --skip-e2e --no-fp64 --steps 1000 > gpurun_out/r02_f_p8shard.log 2>&1; tail -c 1500 gpurun_out/r02_f_p8shard.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_f_gputests.log 2>&1; tail -5 gpurun_out/r02_f_gputests.log
timeout 900 python bench.py > gpurun_out/r02_f_bench.log 2> gpurun_out/r02_f_bench.err; tail -c 800 gpurun_out/r02_f_bench.log
