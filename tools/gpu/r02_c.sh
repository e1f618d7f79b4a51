set -x
prof() {  # name regex skip script...
  local name=$1 rx=$2 skip=$3; shift 3
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 -f -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
  tail -3 gpurun_out/$name.log
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${name}_sass.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source cuda > gpurun_out/${name}_src.csv 2>&1
  ls -la /tmp/$name.ncu-rep gpurun_out/${name}_*
}
prof r02_cl2_f64 fused_rowcol 3 python tools/prof_fp64_fused.py
prof r02_cl2_c2 fused_rowcol 3 python tools/prof_c2.py
prof r02_zslab zslab 5 python tools/prof_fp64_fused.py
for v in 0 1 2 3 4; do compute-sanitizer --tool synccheck tools/san/mbar_sanity $v 2>&1 | tail -4; compute-sanitizer --tool racecheck tools/san/mbar_sanity $v 2>&1 | tail -3; done > gpurun_out/r02_mbar_sanity.log
du -sh gpurun_out
