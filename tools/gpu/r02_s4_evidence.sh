# Session-4 evidence: bench line, launch list, ncu captures (text summaries under gpurun_out/ev4/)
set -x
mkdir -p gpurun_out/ev4
timeout 900 python bench.py > gpurun_out/ev4/bench.json 2> gpurun_out/ev4/bench.err; tail -c 300 gpurun_out/ev4/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev4/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --skip-e2e --no-fp64 > gpurun_out/ev4/launches_run.log 2>&1
python tools/launch_summary.py gpurun_out/ev4/launches.csv > gpurun_out/ev4/launches_summary.txt 2>&1; head -20 gpurun_out/ev4/launches_summary.txt
cap() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/ev4/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep 30 > gpurun_out/ev4/$name.txt 2>&1
  head -14 gpurun_out/ev4/$name.txt
}
cap ncu_fused_f32 "fused_rowcol_kernel" 3 python bench.py --steps 10 --warmup 3 --no-cpu --skip-e2e --no-fp64
cap ncu_sym_f32 "sym_gemv" 5 python bench.py --steps 10 --warmup 3 --no-cpu --skip-e2e --no-fp64
cap ncu_dgemm_pipe "dgemm_pipe" 1 python tools/check_dgemm_pipe.py /tmp/x.npz c3
