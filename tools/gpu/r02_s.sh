set -x
GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5 2>&1 | grep "syrk\|prepare\|gram"
GF_SYRK_2SM=0 GF_VERBOSE_SETUP=1 timeout 300 python tools/time_setup_dev.py c5 2>&1 | grep "syrk"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:syrk_pre2sm -c 1 -f -o /tmp/p2 python tools/time_setup_dev.py c5 > gpurun_out/r02_s_ncu.log 2>&1
python tools/ncu_summary.py /tmp/p2.ncu-rep 30 > gpurun_out/r02_s_p2.txt 2>&1
head -12 gpurun_out/r02_s_p2.txt
