set -x
python tools/debug_wide_indirect.py lasso_wide_200x1000_indirect 10000 > gpurun_out/r02_dbg_wide.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "c2_logistic_100000x10000_fixedrho or prefix200 or other_families or portfolio" > gpurun_out/r02_full_new.log 2>&1
timeout 600 python tools/bench_configs.py c2 c2d c4d c5d > gpurun_out/r02_cfg.log 2>&1
for c in fused32 fused64 cl2 twopass wide indirect gram; do
  for t in memcheck racecheck synccheck; do
    timeout 300 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/r02_san_${c}_${t}.log 2>&1
    echo "$c $t rc=$?" >> gpurun_out/r02_san_summary.txt
    tail -2 gpurun_out/r02_san_${c}_${t}.log >> gpurun_out/r02_san_summary.txt
  done
done
