export GF_VERBOSE_SETUP=1
for c in lag cl9; do
  echo "== $c memcheck"; timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py $c 2>&1 | grep -E "iteration:|ERROR SUMMARY|^$c " | head -5
  echo "== $c synccheck (GF_FUSED_MAXSLOTS=6)"; GF_FUSED_MAXSLOTS=6 timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_cases.py $c 2>&1 | grep -E "iteration:|ERROR SUMMARY|^$c " | head -5
done
