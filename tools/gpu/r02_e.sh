set -x
for v in 5 6 7; do compute-sanitizer --tool synccheck tools/san/mbar_sanity $v 2>&1 | head -12; done > gpurun_out/r02_e_mbar.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 3 python tools/sanitize_cases.py fused32 > gpurun_out/r02_e_sync_fused32.log 2>&1
head -40 gpurun_out/r02_e_sync_fused32.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "c2_" > gpurun_out/r02_e_c2.log 2>&1; tail -15 gpurun_out/r02_e_c2.log
timeout 600 python tools/bench_configs.py c2 > gpurun_out/r02_e_cfg.log 2>&1; cat gpurun_out/r02_e_cfg.log
timeout 600 python tools/c2_deviation.py f64 > gpurun_out/r02_e_c2dev.log 2>&1; cat gpurun_out/r02_e_c2dev.log
