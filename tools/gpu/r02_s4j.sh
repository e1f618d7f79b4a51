# Session-4: stall checks on the final kernels, then the evidence run and the GPU tests
set -x
GF_DISABLE_PDL=1 timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 2; echo "nopdl rc=${PIPESTATUS[0]}"
timeout 150 python tools/hang_c2b.py 3 2>&1 | tail -n 2; echo "pdl rc=${PIPESTATUS[0]}"
bash tools/gpu/r02_s4_evidence.sh
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev4/gputests.log 2>&1; tail -n 2 gpurun_out/ev4/gputests.log
