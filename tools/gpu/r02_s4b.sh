# Session-4: pipelined DMMA GEMM (bit-identical check, setup timings), q x q buffer sharing
set -x
mkdir -p gpurun_out/s4b
GF_DGEMM_PIPE_MINK=0 timeout 300 python tools/check_dgemm_pipe.py /tmp/a.npz
timeout 300 python tools/check_dgemm_pipe.py /tmp/b.npz
GF_DGEMM_PIPE_MINK=128 timeout 300 python tools/check_dgemm_pipe.py /tmp/c.npz
python -c "
import numpy as np
a,b,c=[np.load(f'/tmp/{k}.npz') for k in 'abc']
for k in ('x','nu','it','obj'): print(k, np.array_equal(a[k],b[k]), np.array_equal(a[k],c[k]), float(np.max(np.abs(a[k]-b[k]))), float(np.max(np.abs(a[k]-c[k]))))"
GF_VERBOSE_SETUP=1 GF_DGEMM_PIPE_MINK=0 timeout 600 python tools/check_dgemm_pipe.py /tmp/a3.npz c3 2>&1 | grep -v "^\[gf\] slow"
GF_VERBOSE_SETUP=1 timeout 600 python tools/check_dgemm_pipe.py /tmp/b3.npz c3 2>&1 | grep -v "^\[gf\] slow"
GF_VERBOSE_SETUP=1 GF_DGEMM_PIPE_MINK=128 timeout 600 python tools/check_dgemm_pipe.py /tmp/c3.npz c3 2>&1 | grep -v "^\[gf\] slow"
python -c "
import numpy as np
a,b,c=[np.load(f'/tmp/{k}3.npz') for k in 'abc']
for k in ('x','nu','it','obj'): print(k, np.array_equal(a[k],b[k]), np.array_equal(a[k],c[k]), float(np.max(np.abs(a[k]-b[k]))), float(np.max(np.abs(a[k]-c[k]))))"
GF_VERBOSE_SETUP=1 timeout 600 python tools/time_setup_dev.py c5d c3 2>&1 | tail -14
GF_VERBOSE_SETUP=1 GF_DGEMM_PIPE_MINK=128 timeout 600 python tools/time_setup_dev.py c5d c3 2>&1 | tail -14
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
