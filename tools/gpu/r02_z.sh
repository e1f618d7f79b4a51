echo hold6-cl4-logistic; GF_FUSED_LAG=1 GF_LAG_N=-6 GF_FUSED_CL=4 timeout 300 python tools/bench_configs.py c2 2>&1 | tail -n 1 | cut -c120-300
echo hold6-cl4-lasso; GF_FUSED_LAG=1 GF_LAG_N=-6 GF_FUSED_CL=4 timeout 300 python tools/bench_configs.py c2l 2>&1 | tail -n 1 | cut -c120-300
echo cl4-lasso; GF_FUSED_CL2=1 GF_FUSED_CL=4 timeout 300 python tools/bench_configs.py c2l 2>&1 | tail -n 1 | cut -c120-300
GF_FUSED_LAG=1 GF_LAG_N=-6 GF_FUSED_CL=4 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k c2 2>&1 | tail -n 2
