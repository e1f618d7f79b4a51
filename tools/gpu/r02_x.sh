set -x
prof() {  # name regex skip script...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
  tail -3 gpurun_out/$name.log
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda > gpurun_out/${name}_src.csv 2>&1
}
timeout 900 python -m pytest tests/test_gpu_schedules.py -x -q 2>&1 | grep -E "^E |passed|failed" | head -20
prof r02_lag_c2 fused_rowcol 3 python tools/prof_c2.py
python tools/ncu_summary.py /tmp/r02_lag_c2.ncu-rep 40 > gpurun_out/r02_lag_c2_summary.txt 2>&1; cat gpurun_out/r02_lag_c2_summary.txt | head -20
