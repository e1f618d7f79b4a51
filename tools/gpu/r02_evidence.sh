# Round-2 evidence run: GPU tests, bench line, launch list, ncu captures (text summaries only)
set -x
mkdir -p gpurun_out/ev
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/ev/gputests.log 2>&1; tail -3 gpurun_out/ev/gputests.log
timeout 900 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err; tail -c 400 gpurun_out/ev/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --skip-e2e --no-fp64 > gpurun_out/ev/launches_run.log 2>&1
cap() {  # name regex skip cmd...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/ev/$name.log 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep 30 > gpurun_out/ev/$name.txt 2>&1
  head -20 gpurun_out/ev/$name.txt
}
cap ncu_fused_f32 "fused_rowcol_kernel" 3 python bench.py --steps 10 --warmup 3 --no-cpu --skip-e2e --no-fp64
cap ncu_ring_f32 "ring_gemv" 5 python bench.py --steps 10 --warmup 3 --no-cpu --skip-e2e --no-fp64
cap ncu_cl2_f64 "fused_rowcol_cl2" 3 python tools/prof_fp64_fused.py
cap ncu_syrk_i8 "syrk_i8" 0 python tools/time_setup_dev.py c5d
cap ncu_syrk_pre "syrk_pre" 0 python tools/time_setup_dev.py c5
