set -x
GF_FUSED_CL2=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "solve_fp64 or solve_fp32 or trace or degenerate" > gpurun_out/r02_d_cl2force.log 2>&1; tail -3 gpurun_out/r02_d_cl2force.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "c5_lasso or c4_svm" > gpurun_out/r02_d_full.log 2>&1; tail -3 gpurun_out/r02_d_full.log
timeout 600 python tools/bench_configs.py c5d c4d c2 > gpurun_out/r02_d_cfg.log 2>&1; cat gpurun_out/r02_d_cfg.log
for c in fused32 cl2; do timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python tools/sanitize_cases.py $c 2>&1 | tail -12; done > gpurun_out/r02_d_sync.log
timeout 600 python tools/c2_deviation.py > gpurun_out/r02_d_c2dev.log 2>&1; cat gpurun_out/r02_d_c2dev.log
