# Session-4: which change stalls tools/bench_configs.py c2
set -x
for v in "GF_DISABLE_SYM=1" "GF_CHOL_SP=0" "GF_DISABLE_PDL=1" "X=1"; do
  echo "== $v"; env $v GF_VERBOSE_SETUP=1 timeout 150 python tools/bench_configs.py c2 2>&1 | tail -n 4 | cut -c1-400; echo "rc=$?"
done
