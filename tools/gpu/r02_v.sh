set -x
for cl in 2 4 8; do GF_FUSED_CL2=1 GF_FUSED_CL=$cl timeout 300 python tools/bench_configs.py c5d 2>&1 | tail -n 1 | cut -c1-330; done
for cl in 2 4; do GF_FUSED_CL2=1 GF_FUSED_CL=$cl timeout 300 python tools/bench_configs.py c5 2>&1 | tail -n 1 | cut -c1-330; done
