for m in 6000 50000 200000; do echo "m=$m"; SAN_M=$m timeout 300 python tools/sanitize_cases.py cl2 2>&1 | tail -1; done
echo "nopdl"; GF_DISABLE_PDL=1 SAN_M=200000 timeout 300 python tools/sanitize_cases.py cl2 2>&1 | tail -1
echo "memcheck 50000"; SAN_M=50000 timeout 900 compute-sanitizer --tool memcheck --print-limit 3 python tools/sanitize_cases.py cl2 2>&1 | grep -v "Host Frame" | head -30
