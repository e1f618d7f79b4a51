echo logistic-lag8-evictlast; timeout 300 python tools/bench_configs.py c2 2>&1 | tail -n 1 | cut -c120-300
echo lasso-lag8-evictlast; GF_FUSED_LAG=1 timeout 300 python tools/bench_configs.py c2l 2>&1 | tail -n 1 | cut -c120-300
echo c5; timeout 300 python tools/bench_configs.py c5 2>&1 | tail -n 1 | cut -c120-300
