# Session-4: two-level Cholesky (K = SP bulk updates on the pipelined DMMA GEMM)
set -x
for sp in 0 512; do GF_CHOL_SP=$sp timeout 300 python tools/check_dgemm_pipe.py /tmp/s$sp.npz; done
python -c "
import numpy as np
a,b=[np.load(f'/tmp/s{k}.npz') for k in (0,512)]
print('small', int(a['it']), int(b['it']), float(np.max(np.abs(a['x']-b['x']))/np.max(np.abs(a['x']))), float(a['obj']), float(b['obj']))"
for sp in 0 256 512 1024; do echo "SP=$sp"; GF_CHOL_SP=$sp GF_VERBOSE_SETUP=1 timeout 600 python tools/check_dgemm_pipe.py /tmp/c$sp.npz c3 2>&1 | grep -v "slow alloc" | grep "projector\|prepare"; done
python -c "
import numpy as np
a=np.load('/tmp/c0.npz')
for k in (256,512,1024):
  b=np.load(f'/tmp/c{k}.npz'); print('c3', k, int(a['it']), int(b['it']), float(np.max(np.abs(a['x']-b['x']))/np.max(np.abs(a['x']))), float(a['obj']), float(b['obj']))"
for sp in 0 512; do echo "SP=$sp"; GF_CHOL_SP=$sp GF_VERBOSE_SETUP=1 timeout 600 python tools/time_setup_dev.py c5 c5d 2>&1 | grep "projector\|prepare" | tail -4; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "c3 or parity or gram or project or chol" 2>&1 | tail -3
