"""ctypes binding of the C ABI (include/graphform_b200.h).

This is the only door into the CUDA library.  There is no CPU fallback: if
the shared object is missing or no CUDA device is visible, every call raises
``DeviceError``.  The library is built in-tree by
``paper_1503_08366_b200/csrc/build.py`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import (DegenerateInputError, DeviceError, DimensionError, NumericError,
                     ParameterError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgraphform_b200.so")

GF_F32, GF_F64 = 0, 1
STATUS = {0: "Running", 1: "Solved", 2: "MaxIterations", 3: "Degenerate"}

_ERR = {1: DimensionError, 2: ParameterError, 3: DegenerateInputError, 4: NumericError,
        5: DeviceError, 6: DeviceError, 7: NotImplementedError}

c_int64_p = C.POINTER(C.c_int64)
c_double_p = C.POINTER(C.c_double)
c_int_p = C.POINTER(C.c_int)


class Terms(C.Structure):
    _fields_ = [("n", C.c_int64), ("h", C.c_void_p), ("a", C.c_void_p), ("b", C.c_void_p),
                ("c", C.c_void_p), ("d", C.c_void_p), ("e", C.c_void_p)]


class Settings(C.Structure):
    _fields_ = [("rho0", C.c_double), ("abs_tol", C.c_double), ("rel_tol", C.c_double),
                ("max_iter", C.c_int64), ("alpha", C.c_double), ("adaptive_rho", C.c_int),
                ("delta", C.c_double), ("tau", C.c_double), ("projection", C.c_int),
                ("projection_tol", C.c_double), ("gap_stop", C.c_int)]


class SolverState(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int64), ("k", C.c_int64),
                ("r_pri", C.c_double), ("r_dual", C.c_double), ("eps_pri", C.c_double),
                ("eps_dual", C.c_double), ("rho", C.c_double), ("objective", C.c_double),
                ("final_rho", C.c_double), ("inner_iterations", C.c_int64),
                ("gap", C.c_double), ("gap_valid", C.c_int)]


class SetupInfo(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("converged", C.c_int), ("gamma", C.c_double),
                ("setup_seconds", C.c_double)]


_P = C.c_void_p
_SIGS = {
    "gf_version": ([], C.c_char_p),
    "gf_last_error": ([], C.c_char_p),
    "gf_init": ([C.c_int], C.c_int),
    "gf_prox_separable": ([C.POINTER(Terms), _P, _P, _P, _P], C.c_int),
    "gf_prox_base": ([C.c_int64, C.c_int, _P, _P, _P, _P], C.c_int),
    "gf_evaluate": ([C.POINTER(Terms), _P, c_double_p, _P], C.c_int),
    "gf_eval_base": ([C.c_int64, C.c_int, _P, _P, _P], C.c_int),
    "gf_conj_base": ([C.c_int64, C.c_int, _P, _P, _P], C.c_int),
    "gf_conjugate": ([C.POINTER(Terms), _P, c_double_p, c_int_p, _P], C.c_int),
    "gf_matrix_create": ([C.c_int, C.c_int64, C.c_int64, _P, C.c_int, C.c_int64, _P, C.POINTER(_P)], C.c_int),
    "gf_matrix_destroy": ([_P], C.c_int),
    "gf_matrix_shape": ([_P, c_int64_p, c_int64_p, c_int64_p, c_int_p], C.c_int),
    "gf_matrix_download": ([_P, _P, _P], C.c_int),
    "gf_matvec": ([_P, C.c_int, _P, _P, _P], C.c_int),
    "gf_sq_matvec": ([_P, C.c_int, _P, _P, _P], C.c_int),
    "gf_equilibrate": ([_P, C.c_double, C.c_double, C.c_int64, _P, _P, _P, c_int64_p, c_int_p,
                        c_double_p, _P], C.c_int),
    "gf_equilibrate_observed": ([_P, C.c_double, C.c_double, C.c_int64, _P, _P, _P, c_int64_p, c_int_p,
                                 c_double_p, _P, _P, _P], C.c_int),
    "gf_rescale_even": ([_P, _P, _P, _P, _P], C.c_int),
    "gf_scale_matrix": ([_P, _P, _P, _P], C.c_int),
    "gf_projector_create": ([_P, C.c_int, C.c_double, C.c_int64, _P, _P, C.POINTER(_P)], C.c_int),
    "gf_projector_destroy": ([_P], C.c_int),
    "gf_projector_gram": ([_P, _P, _P], C.c_int),
    "gf_project": ([_P, _P, _P, _P, _P, _P], C.c_int),
    "gf_project_indirect": ([_P, _P, _P, _P, _P, C.c_double, _P, _P, c_int64_p, c_int_p, _P], C.c_int),
    "gf_setup_create": ([_P, C.c_int, _P, _P, C.c_int, C.c_double, C.c_int64, _P, _P, C.POINTER(_P)], C.c_int),
    "gf_setup_destroy": ([_P], C.c_int),
    "gf_setup_get_info": ([_P, C.POINTER(SetupInfo)], C.c_int),
    "gf_setup_scaling": ([_P, _P, _P, _P], C.c_int),
    "gf_setup_projector": ([_P, C.POINTER(_P)], C.c_int),
    "gf_setup_matrix": ([_P, C.POINTER(_P)], C.c_int),
    "gf_solver_create": ([_P, C.POINTER(Terms), C.POINTER(Terms), C.POINTER(Settings), _P, _P, _P,
                          C.POINTER(_P)], C.c_int),
    "gf_solver_run": ([_P, C.c_int64, C.POINTER(SolverState), _P], C.c_int),
    "gf_solver_history": ([_P, C.c_int64, _P, _P], C.c_int),
    "gf_solver_snapshot": ([_P, _P, _P, _P, _P, _P, _P, _P], C.c_int),
    "gf_solver_result": ([_P, _P, _P, _P, _P, C.POINTER(SolverState), _P], C.c_int),
    "gf_solve": ([_P, C.POINTER(Terms), C.POINTER(Terms), C.POINTER(Settings), _P, _P, _P, _P, _P, _P,
                  C.POINTER(SolverState), _P, _P], C.c_int),
    "gf_solver_destroy": ([_P], C.c_int),
    "gf_solver_elapsed_ms": ([_P, c_double_p], C.c_int),
    "gf_solver_stats": ([_P, c_int64_p, _P, _P], C.c_int),
    "gf_solver_profile": ([_P, C.c_int], C.c_int),
    "gf_normal_fill": ([C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_double,
                        C.c_int, _P, C.c_int64, C.c_int64, C.c_int64, _P], C.c_int),
    "gf_dense_matvec": ([C.c_int, C.c_int64, C.c_int64, _P, C.c_int64, C.c_int, _P, _P, _P], C.c_int),
    "gf_rows_affine": ([C.c_int64, C.c_int64, _P, C.c_int64, _P, _P, _P], C.c_int),
    "gf_convert_matrix": ([C.c_int64, C.c_int64, _P, C.c_int64, C.c_int, _P, C.c_int64, _P], C.c_int),
    "gf_matrix_all_finite": ([C.c_int, C.c_int64, C.c_int64, _P, C.c_int64, C.POINTER(C.c_int), _P], C.c_int),
    "gf_comm_unique_id": ([C.c_char_p], C.c_int),
    "gf_comm_create": ([C.c_char_p, C.c_int, C.c_int, C.POINTER(_P)], C.c_int),
    "gf_comm_destroy": ([_P], C.c_int),
}

_lib = None
_lock = threading.Lock()
_inited_devices = set()


def exported_symbols():
    return sorted(_SIGS)


def load_library(path: str = LIB_PATH):
    """Load the shared object and declare every entry point (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # torch first: it carries its own libnccl.so.2 (2.28); if this library
        # were loaded first the system NCCL (2.27) would claim the soname and
        # torch's import would fail on symbols only 2.28 has.
        try:
            import torch  # noqa: F401
        except ImportError:
            pass
        if not os.path.exists(path):
            raise DeviceError(
                f"native library {path} is missing: run __graft_entry__.build() "
                "(python paper_1503_08366_b200/csrc/build.py)")
        lib = C.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(code: int):
    if code != 0:
        lib = load_library()
        msg = lib.gf_last_error().decode(errors="replace")
        raise _ERR.get(code, DeviceError)(msg)


def lib():
    """The library, with the current torch CUDA device initialised."""
    import torch
    L = load_library()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible: the graphform-b200 path runs only on the GPU")
    dev = torch.cuda.current_device()
    if dev not in _inited_devices:
        check(L.gf_init(dev))
        _inited_devices.add(dev)
    return L


def device():
    import torch
    lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> C.c_void_p:
    """Raw pointer of a torch tensor or numpy array (must stay alive)."""
    if isinstance(t, np.ndarray):
        return C.c_void_p(t.ctypes.data)
    return C.c_void_p(t.data_ptr())


# ------------------------------------------------------------ conversions --
def is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def to_device64(x, n=None):
    """fp64 contiguous CUDA tensor view/copy of a numpy array, list or tensor."""
    import torch
    dev = device()
    if is_torch(x):
        t = x.to(device=dev, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev)
    t = t.contiguous()
    if n is not None and t.numel() != n:
        raise DimensionError(f"expected vector of length {n}, got {tuple(t.shape)}")
    return t


def like_input(t, ref):
    """Return tensor ``t`` as the same kind of object as ``ref``."""
    if is_torch(ref):
        return t.to(ref.device) if ref.is_cuda else t.cpu()
    return t.cpu().numpy()


def device_terms(sf):
    """(Terms struct, keep-alive tuple) with the term arrays on the device."""
    import torch
    dev = device()
    key = ("dev", dev.index)
    cache = sf._device_cache
    if key not in cache:
        h = torch.from_numpy(np.ascontiguousarray(sf.h.astype(np.int8))).to(dev)
        arrs = [torch.from_numpy(np.ascontiguousarray(getattr(sf, k))).to(dev) for k in "abcde"]
        cache[key] = (h, *arrs)
    keep = cache[key]
    T = Terms(len(sf), *(C.c_void_p(a.data_ptr()) for a in keep))
    return T, keep


def host_terms(sf):
    """Terms struct over host arrays (the library copies them itself)."""
    h = np.ascontiguousarray(sf.h.astype(np.int8))
    arrs = [np.ascontiguousarray(getattr(sf, k), dtype=np.float64) for k in "abcde"]
    keep = (h, *arrs)
    T = Terms(len(sf), *(C.c_void_p(a.ctypes.data) for a in keep))
    return T, keep


# ------------------------------------------------------- simple services --
def prox_separable_dev(sf, rho_t, v_t):
    import torch
    L = lib()
    T, keep = device_terms(sf)
    out = torch.empty_like(v_t)
    check(L.gf_prox_separable(C.byref(T), ptr(rho_t), ptr(v_t), ptr(out), stream()))
    return out


def prox_base_dev(code, rho_t, v_t):
    import torch
    L = lib()
    out = torch.empty_like(v_t)
    check(L.gf_prox_base(v_t.numel(), int(code), ptr(rho_t), ptr(v_t), ptr(out), stream()))
    return out


def evaluate(sf, v) -> float:
    L = lib()
    v_t = to_device64(v)
    if v_t.dim() != 1 or v_t.numel() != len(sf):
        raise DimensionError(f"expected vector of length {len(sf)}, got shape {tuple(np.shape(v))}")
    T, keep = device_terms(sf)
    out = C.c_double()
    check(L.gf_evaluate(C.byref(T), ptr(v_t), C.byref(out), stream()))
    return float(out.value)


def conjugate(sf, w):
    """Sum of the term conjugates at w, or None when unsupported."""
    L = lib()
    w_t = to_device64(w)
    if w_t.dim() != 1 or w_t.numel() != len(sf):
        raise DimensionError(f"expected vector of length {len(sf)}, got shape {tuple(np.shape(w))}")
    T, keep = device_terms(sf)
    out = C.c_double()
    ok = C.c_int()
    check(L.gf_conjugate(C.byref(T), ptr(w_t), C.byref(out), C.byref(ok), stream()))
    return float(out.value) if ok.value else None


def conj_base(code, w):
    import torch
    L = lib()
    scalar = np.ndim(w) == 0 and not is_torch(w)
    w_t = to_device64(np.atleast_1d(np.asarray(w, float)) if scalar else w)
    out = torch.empty_like(w_t)
    check(L.gf_conj_base(w_t.numel(), int(code), ptr(w_t), ptr(out), stream()))
    if scalar:
        return float(out.item())
    return like_input(out, w)


def eval_base(code, x):
    import torch
    L = lib()
    scalar = np.ndim(x) == 0 and not is_torch(x)
    x_t = to_device64(np.atleast_1d(np.asarray(x, float)) if scalar else x)
    out = torch.empty_like(x_t)
    check(L.gf_eval_base(x_t.numel(), int(code), ptr(x_t), ptr(out), stream()))
    if scalar:
        return float(out.item())
    return like_input(out, x)


# ----------------------------------------------------- input synthesis --
_M64 = (1 << 64) - 1


def normal_fill(rng, out, count, loc=0.0, scale=1.0, ncol=None, rs=None, cs=1):
    """Write ``rng.normal(loc, scale, size=count)`` (numpy Generator on PCG64)
    into the CUDA tensor ``out``: normal j lands at flat offset
    (j // ncol) * rs + (j % ncol) * cs.  Bit-identical to numpy."""
    import torch
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ParameterError("device sampling reproduces PCG64 streams only")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    dt = GF_F32 if out.dtype == torch.float32 else GF_F64
    ncol = int(count) if ncol is None else int(ncol)
    rs = ncol if rs is None else int(rs)
    check(lib().gf_normal_fill(s >> 64, s & _M64, inc >> 64, inc & _M64, int(count), float(loc), float(scale),
                               dt, ptr(out), ncol, int(rs), int(cs), stream()))


def dense_matvec(A, x, transpose=False):
    """fp64 A @ x (or A.T @ x) over a CUDA matrix with unit column stride."""
    import torch
    L = lib()
    if A.stride(1) != 1:
        raise ParameterError("matrix must have unit column stride")
    m, n = int(A.shape[0]), int(A.shape[1])
    x_t = to_device64(x)
    y = torch.empty(n if transpose else m, dtype=torch.float64, device=A.device)
    dt = GF_F32 if A.dtype == torch.float32 else GF_F64
    check(L.gf_dense_matvec(dt, m, n, ptr(A), int(A.stride(0)), 1 if transpose else 0, ptr(x_t), ptr(y), stream()))
    return y


def rows_affine(A, s, t):
    """A_ij <- s_i * (A_ij + t_i) in place (fp64 CUDA matrix)."""
    s_t, t_t = to_device64(s), to_device64(t)
    check(lib().gf_rows_affine(int(A.shape[0]), int(A.shape[1]), ptr(A), int(A.stride(0)), ptr(s_t), ptr(t_t),
                               stream()))


def all_finite(A) -> bool:
    """Every entry of the CUDA matrix A (unit column stride) finite: one pass
    over A on the device (gf_matrix_all_finite)."""
    import torch
    dt = GF_F32 if A.dtype == torch.float32 else GF_F64
    out = C.c_int(0)
    check(lib().gf_matrix_all_finite(dt, int(A.shape[0]), int(A.shape[1]), ptr(A), int(A.stride(0)), C.byref(out),
                                     stream()))
    return bool(out.value)


def convert_matrix(src, dst):
    """dst <- src (fp64 -> dst's dtype), both CUDA, unit column stride."""
    import torch
    dt = GF_F32 if dst.dtype == torch.float32 else GF_F64
    check(lib().gf_convert_matrix(int(src.shape[0]), int(src.shape[1]), ptr(src), int(src.stride(0)), dt, ptr(dst),
                                  int(dst.stride(0)), stream()))


class Matrix:
    """Owning handle of a gf_matrix (library-side padded copy of A)."""

    def __init__(self, A, dtype: int):
        L = lib()
        self._lib = L
        src_ld = None
        if is_torch(A):
            import torch
            src = A
            if src.is_cuda and src.dim() == 2 and src.stride(1) == 1 and src.dtype in (torch.float32, torch.float64):
                src_ld = int(src.stride(0))    # row-strided device view (e.g. a padded buffer): no copy
            else:
                src = src.contiguous()
            if src.dtype not in (torch.float32, torch.float64):
                src = src.to(torch.float64)
            if not src.is_cuda:
                src = src.numpy()
        else:
            src = np.ascontiguousarray(A)
            if src.dtype not in (np.float32, np.float64):
                src = src.astype(np.float64)
        self.m, self.n = int(src.shape[0]), int(src.shape[1])
        sdt = GF_F32 if str(src.dtype).endswith("float32") else GF_F64
        h = C.c_void_p()
        check(L.gf_matrix_create(dtype, self.m, self.n, ptr(src) if self.m else None, sdt,
                                 src_ld if src_ld is not None else self.n, stream(), C.byref(h)))
        self.handle = h
        self.dtype = dtype
        self.owned = True

    def release(self):
        """Give up ownership (the handle was passed to an owning object)."""
        self.owned = False

    def download(self) -> np.ndarray:
        out = np.empty((self.m, self.n))
        check(self._lib.gf_matrix_download(self.handle, ptr(out), stream()))
        return out

    def __del__(self):
        try:
            if self.owned and self.handle:
                self._lib.gf_matrix_destroy(self.handle)
        except Exception:
            pass


# gf_sweep_fn: void (*)(int64_t k, const double* d, const double* e, int64_t m, int64_t n, void* user)
SWEEP_FN = C.CFUNCTYPE(None, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64, C.c_int64,
                       C.c_void_p)
