set -x
prof() {  # name regex skip script...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
  tail -3 gpurun_out/$name.log
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>&1
  python tools/ncu_summary.py /tmp/$name.ncu-rep 40 > gpurun_out/${name}_summary.txt 2>&1; head -16 gpurun_out/${name}_summary.txt
}
prof r02_cl8_c3 fused_rowcol 3 python tools/prof_c3.py
prof r02_ginv_c3 "rowgemv|ring_gemv" 3 python tools/prof_c3.py
