"""ctypes view of the C ABI (include/acg.h) of ``libacg_cuda.so``.

This is the plugin boundary a non-C++ host binds (the cgo/JNI/ctypes stub of
INTEGRATION.md); ``bench.py`` and the multi-slab / device-resident tests use it
directly. Fields live on the device between calls (no host round trip).
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ACG_LIB_OVERRIDE") or os.path.join(_HERE, "libacg_cuda.so")

F64, F32 = 0, 1
VERTICAL, HORIZONTAL = 0, 1
HOST_FULL, HOST_LOCAL = 0, 1
STANDARD, INTERLEAVED = 0, 1
MATRIX_FREE, CSR = 0, 1
EXACT, FAST = 0, 1


class AcgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"acg status {status}: {msg}")
        self.status = status


class BreakdownError(AcgError):
    """NumericalBreakdown (operator.hpp:21-24)."""


class OperatorDesc(C.Structure):
    _fields_ = [("m", C.c_int), ("n_z", C.c_int)] + [
        (n, C.POINTER(C.c_double)) for n in
        ("a_prime", "b_prime", "c_prime", "d", "cell_area", "alpha_east", "alpha_north", "alpha_diag")]


class Placement(C.Structure):
    _fields_ = [("device", C.c_int), ("slabs", C.c_int), ("comm", C.c_void_p), ("math", C.c_int)]


class ContextInfo(C.Structure):
    _fields_ = [("m", C.c_int), ("n_z", C.c_int), ("dtype", C.c_int), ("math", C.c_int),
                ("nslabs_total", C.c_int), ("nslabs_local", C.c_int), ("rank", C.c_int),
                ("i_begin", C.c_int), ("i_end", C.c_int), ("exact_tree", C.c_int),
                ("bytes_per_field_local", C.c_size_t), ("thomas_tmem", C.c_int)]


class SolverConfig(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("tau", C.c_double), ("maxiter", C.c_int),
                ("variant", C.c_int), ("backend", C.c_int), ("workers", C.c_int),
                ("record_timings", C.c_int), ("layout", C.c_int)]


class KernelTimings(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("spmv", "prec", "blas", "fused_spmv", "fused_prec",
                                          "setup", "total")]


class SolveResult(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("true_residual", C.c_double),
                ("n_residual", C.c_int), ("n_kappa", C.c_int), ("n_alpha", C.c_int),
                ("n_beta", C.c_int), ("timings", KernelTimings), ("kernel_launches", C.c_longlong),
                ("history", C.POINTER(C.c_double) * 4)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libacg_cuda.so not built at {LIB_PATH}")
    L = C.CDLL(LIB_PATH)
    vp, ip, dp = C.c_void_p, C.c_int, C.POINTER(C.c_double)
    pp = C.POINTER(C.c_void_p)
    sig = {
        "acg_last_error": (C.c_char_p, []),
        "acg_abi_version": (ip, []),
        "acg_kernel_launch_count": (C.c_longlong, []),
        "acg_device_count": (ip, [C.POINTER(C.c_int)]),
        "acg_host_alloc": (ip, [pp, C.c_size_t]),
        "acg_host_free": (ip, [vp]),
        "acg_comm_unique_id": (ip, [vp]),
        "acg_comm_create": (ip, [pp, ip, ip, vp, ip]),
        "acg_comm_destroy": (ip, [vp]),
        "acg_context_create": (ip, [pp, ip, C.POINTER(OperatorDesc), C.POINTER(Placement)]),
        "acg_context_destroy": (ip, [vp]),
        "acg_partition_plan": (ip, [ip, ip, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "acg_context_info_get": (ip, [vp, C.POINTER(ContextInfo)]),
        "acg_context_stream": (vp, [vp]),
        "acg_synchronize": (ip, [vp]),
        "acg_field_create": (ip, [pp, vp]),
        "acg_field_destroy": (ip, [vp]),
        "acg_field_upload": (ip, [vp, vp, ip, ip]),
        "acg_field_download": (ip, [vp, vp, ip, ip]),
        "acg_field_upload_async": (ip, [vp, vp, ip, ip]),
        "acg_field_download_async": (ip, [vp, vp, ip, ip]),
        "acg_field_wait": (ip, [vp]),
        "acg_field_upload_device": (ip, [vp, vp, ip, ip]),
        "acg_comm_create_ipc": (ip, [pp, ip, ip, vp, ip]),
        "acg_field_download_device": (ip, [vp, vp, ip, ip]),
        "acg_field_fill": (ip, [vp, C.c_double]),
        "acg_field_fill_random": (ip, [vp, C.c_uint64]),
        "acg_field_copy": (ip, [vp, vp]),
        "acg_apply": (ip, [vp, vp, vp]),
        "acg_precondition": (ip, [vp, vp, vp]),
        "acg_axpy": (ip, [C.c_double, vp, vp]),
        "acg_scal": (ip, [C.c_double, vp]),
        "acg_dot": (ip, [vp, vp, dp]),
        "acg_nrm2": (ip, [vp, dp]),
        "acg_true_residual": (ip, [vp, vp, vp, dp]),
        "acg_interleaved_spmv_kernel": (ip, [vp, vp, vp, vp, vp, C.c_double, C.c_double, dp]),
        "acg_interleaved_prec_kernel": (ip, [vp, vp, vp, vp, C.c_double, dp, dp]),
        "acg_solver_config_default": (None, [C.POINTER(SolverConfig)]),
        "acg_solve_result_release": (None, [C.POINTER(SolveResult)]),
        "acg_context_wait_stream": (ip, [vp, vp]),
        "acg_stream_wait_context": (ip, [vp, vp]),
        "acg_context_release_scratch": (ip, [vp]),
        "acg_solve": (ip, [vp, vp, vp, C.POINTER(SolverConfig), vp, C.POINTER(SolveResult),
                           vp, vp, vp, vp]),
        "acg_solver_create": (ip, [pp, vp, C.POINTER(SolverConfig)]),
        "acg_solver_destroy": (ip, [vp]),
        "acg_solver_start": (ip, [vp, vp, vp]),
        "acg_solver_iterate": (ip, [vp, ip]),
        "acg_solver_finish": (ip, [vp, vp, C.POINTER(SolveResult), vp, vp, vp, vp]),
        "acg_solver_time_kernels": (ip, [vp, ip]),
        "acg_solver_kernel_times": (ip, [vp, C.POINTER(C.c_int), dp, C.POINTER(C.c_int), dp]),
        "acg_apply_host": (ip, [vp, ip, vp, vp]),
        "acg_precondition_host": (ip, [vp, ip, vp, vp]),
        "acg_true_residual_host": (ip, [vp, ip, vp, vp, dp]),
        "acg_solve_host": (ip, [vp, ip, vp, vp, C.POINTER(SolverConfig), vp,
                                C.POINTER(SolveResult), vp, vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols():
    """Names of the C-ABI functions this wrapper binds (all declared in acg.h)."""
    lib()
    return [n for n in dir(_lib) if n.startswith("acg_")]


def partition_plan(m, p):
    """(i_begin[0..p], exact_tree) of the p-slab decomposition (acg_partition_plan)."""
    ib = (C.c_int * (p + 1))()
    ex = C.c_int()
    check(lib().acg_partition_plan(m, p, ib, C.byref(ex)))
    return list(ib), bool(ex.value)


def check(status):
    if status == 0:
        return
    msg = lib().acg_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise BreakdownError(status, msg)
    raise AcgError(status, msg)


def _dptr(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _vptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


class Comm:
    """NCCL communicator, one rank per GPU (acg_comm_create)."""

    def __init__(self, rank, nranks, unique_id: bytes, device):
        h = C.c_void_p()
        buf = C.create_string_buffer(unique_id, 128)
        check(lib().acg_comm_create(C.byref(h), rank, nranks, buf, device))
        self.h, self.rank, self.nranks = h, rank, nranks

    @classmethod
    def ipc(cls, rank, nranks, unique_id: bytes, device):
        """Peer-memory communicator (acg_comm_create_ipc): ranks of one node,
        CUDA IPC mailboxes, no NCCL. unique_id: same bytes on every rank."""
        self = cls.__new__(cls)
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id)[:128].ljust(128, b"\0"), 128)
        check(lib().acg_comm_create_ipc(C.byref(h), rank, nranks, buf, device))
        self.h, self.rank, self.nranks = h, rank, nranks
        return self

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().acg_comm_unique_id(buf))
        return buf.raw

    def close(self):
        if self.h:
            lib().acg_comm_destroy(self.h)
            self.h = None


class Context:
    """Device operator context (OperatorContext<T>, operator.hpp:29-67)."""

    def __init__(self, a_prime, b_prime, c_prime, d, cell_area, alpha_east, alpha_north, alpha_diag,
                 dtype=F64, slabs=1, math=EXACT, device=0, comm: Comm | None = None):
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1) for a in
                (a_prime, b_prime, c_prime, d, cell_area, alpha_east, alpha_north, alpha_diag)]
        arrs = [a if a.size else np.zeros(1) for a in arrs]
        self._keep = arrs
        m = int(round(np.sqrt(arrs[4].size)))
        n_z = arrs[0].size
        desc = OperatorDesc(m, n_z, *[_dptr(a) for a in arrs])
        pl = Placement(device, slabs, comm.h if comm else None, math)
        h = C.c_void_p()
        check(lib().acg_context_create(C.byref(h), dtype, C.byref(desc), C.byref(pl)))
        self.h, self.m, self.n_z, self.dtype = h, m, n_z, dtype
        self.np_dtype = np.float32 if dtype == F32 else np.float64
        self._children = weakref.WeakSet()  # fields/solvers released before the context

    @classmethod
    def borrow(cls, handle, owner=None):
        """View of an existing acg_context (e.g. an anisocg.OperatorContext's);
        does not destroy it. `owner` is kept alive for the view's lifetime."""
        self = cls.__new__(cls)
        self.h = C.c_void_p(handle)
        inf = ContextInfo()
        check(lib().acg_context_info_get(self.h, C.byref(inf)))
        self.m, self.n_z, self.dtype = inf.m, inf.n_z, inf.dtype
        self.np_dtype = np.float32 if inf.dtype == F32 else np.float64
        self._children = weakref.WeakSet()
        self._owner = owner
        self._borrowed = True
        return self

    @classmethod
    def from_setup(cls, profile, panel, **kw):
        """From (a', b', c', d) and (area, east, north, diag) arrays."""
        return cls(*profile, *panel, **kw)

    def info(self):
        i = ContextInfo()
        check(lib().acg_context_info_get(self.h, C.byref(i)))
        return {f: getattr(i, f) for f, _ in ContextInfo._fields_}

    def sync(self):
        check(lib().acg_synchronize(self.h))

    @property
    def stream(self):
        return lib().acg_context_stream(self.h)

    def wait_for(self, stream):
        """The context's stream waits for the work enqueued on `stream` so far."""
        check(lib().acg_context_wait_stream(self.h, C.c_void_p(stream or None)))

    def signal_to(self, stream):
        """`stream` waits for the work enqueued on the context's stream so far."""
        check(lib().acg_stream_wait_context(C.c_void_p(stream or None), self.h))

    def release_scratch(self):
        """Free cached scratch (solver work fields, pooled fields, staging)."""
        check(lib().acg_context_release_scratch(self.h))

    def field(self):
        return Field(self)

    def close(self):
        if self.h:
            for child in list(self._children):
                child.close()
            if not getattr(self, "_borrowed", False):
                lib().acg_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def is_cuda_array(a):
    """True for device arrays exposing __cuda_array_interface__ (torch, CuPy)."""
    return hasattr(a, "__cuda_array_interface__")


def array_stream(a):
    """cudaStream_t handle of the stream that produces / consumes a CUDA array:
    torch's current stream for torch tensors, else the __cuda_array_interface__
    v3 'stream' key (1 = legacy default, 2 = per-thread default; absent/None:
    the legacy default stream)."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            return torch.cuda.current_stream(a.device).cuda_stream
    except ImportError:  # pragma: no cover - torch is part of this image
        pass
    st = a.__cuda_array_interface__.get("stream")
    return int(st) if st else 0


def cuda_array_ptr(a, dtype, shape):
    """Device pointer of a C-contiguous CUDA array of `dtype` and `shape`
    (raises ValueError otherwise, like the reference's nonconformant-field check)."""
    ai = a.__cuda_array_interface__
    if np.dtype(ai["typestr"]) != np.dtype(dtype):
        raise ValueError(f"device array dtype {np.dtype(ai['typestr'])} != context dtype {np.dtype(dtype)}")
    if tuple(ai["shape"]) != tuple(shape):
        raise ValueError(f"device array shape {tuple(ai['shape'])} != expected {tuple(shape)}")
    st = ai.get("strides")
    if st is not None:
        item = np.dtype(dtype).itemsize
        want, acc = [], item
        for d in reversed(shape):
            want.append(acc)
            acc *= d
        if tuple(st) != tuple(reversed(want)):
            raise ValueError("device array must be C-contiguous")
    return int(ai["data"][0])


class Field:
    """Device field (Field3D<T> storage in the plane-major device layout)."""

    def __init__(self, ctx: Context):
        h = C.c_void_p()
        check(lib().acg_field_create(C.byref(h), ctx.h))
        self.h, self.ctx = h, ctx
        ctx._children.add(self)

    def _shape(self, layout, scope):
        m, n_z = self.ctx.m, self.ctx.n_z
        inf = self.ctx.info() if scope == HOST_LOCAL else None
        ml = inf["i_end"] - inf["i_begin"] if inf else m
        return (ml, m, n_z) if layout == VERTICAL else (m, n_z, ml)

    def upload(self, a, layout=VERTICAL, scope=HOST_FULL):
        """From a host array, or zero-PCIe from a CUDA array (torch/CuPy:
        anything with __cuda_array_interface__) on the context's device."""
        if is_cuda_array(a):
            ptr = cuda_array_ptr(a, self.ctx.np_dtype, self._shape(layout, scope))
            st = array_stream(a)
            self.ctx.wait_for(st)    # the producer's pending writes land first
            check(lib().acg_field_upload_device(self.h, C.c_void_p(ptr), layout, scope))
            self.ctx.signal_to(st)   # later work on the owner's stream (frees, reuse) waits for the read
            return self
        a = np.ascontiguousarray(a, dtype=self.ctx.np_dtype)
        check(lib().acg_field_upload(self.h, _vptr(a), layout, scope))
        return self

    def download(self, layout=VERTICAL, out=None, scope=HOST_FULL):
        """To a host array, or (out = a CUDA array) device to device."""
        if out is not None and is_cuda_array(out):
            ptr = cuda_array_ptr(out, self.ctx.np_dtype, self._shape(layout, scope))
            st = array_stream(out)
            self.ctx.wait_for(st)    # pending work on the output's memory finishes first
            check(lib().acg_field_download_device(self.h, C.c_void_p(ptr), layout, scope))
            self.ctx.signal_to(st)   # the consumer's stream sees the result
            return out
        if out is None:
            out = np.empty(self._shape(layout, scope), dtype=self.ctx.np_dtype)
        check(lib().acg_field_download(self.h, _vptr(out), layout, scope))
        return out

    def upload_async(self, host, layout=VERTICAL, scope=HOST_FULL):
        """Enqueue the upload of a page-locked host array (HostBuffer.array) on
        the context's copy stream and return at once; later calls on this
        field run after it. Keep `host` unchanged until wait()."""
        a = np.asarray(host)
        if a.dtype != self.ctx.np_dtype or not a.flags.c_contiguous:
            raise ValueError("upload_async needs a C-contiguous page-locked array of the context dtype")
        if a.shape != self._shape(layout, scope):
            raise ValueError(f"upload_async: shape {a.shape}, expected {self._shape(layout, scope)}")
        check(lib().acg_field_upload_async(self.h, _vptr(a), layout, scope))
        return self

    def download_async(self, out, layout=VERTICAL, scope=HOST_FULL):
        """Enqueue the download into a page-locked host array; `out` is
        complete after wait()."""
        if out.dtype != self.ctx.np_dtype or not out.flags.c_contiguous:
            raise ValueError("download_async needs a C-contiguous page-locked array of the context dtype")
        if out.shape != self._shape(layout, scope):
            raise ValueError(f"download_async: shape {out.shape}, expected {self._shape(layout, scope)}")
        check(lib().acg_field_download_async(self.h, _vptr(out), layout, scope))
        return out

    def wait(self):
        """Block until this field's asynchronous transfers are complete."""
        check(lib().acg_field_wait(self.h))
        return self

    def fill(self, v):
        check(lib().acg_field_fill(self.h, float(v)))
        return self

    def fill_random(self, seed):
        check(lib().acg_field_fill_random(self.h, seed))
        return self

    def copy_from(self, other):
        check(lib().acg_field_copy(self.h, other.h))
        return self

    def close(self):
        if self.h:
            lib().acg_field_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def apply(ctx, x, y):
    check(lib().acg_apply(ctx.h, x.h, y.h))


def precondition(ctx, y, x):
    check(lib().acg_precondition(ctx.h, y.h, x.h))


def dot(x, y):
    out = C.c_double()
    check(lib().acg_dot(x.h, y.h, C.byref(out)))
    return out.value


def nrm2(x):
    out = C.c_double()
    check(lib().acg_nrm2(x.h, C.byref(out)))
    return out.value


def axpy(alpha, x, y):
    check(lib().acg_axpy(alpha, x.h, y.h))


def scal(alpha, x):
    check(lib().acg_scal(alpha, x.h))


def true_residual(ctx, u, f):
    out = C.c_double()
    check(lib().acg_true_residual(ctx.h, u.h, f.h, C.byref(out)))
    return out.value


def fused_spmv(ctx, u, p, q, z, alpha, beta):
    out = C.c_double()
    check(lib().acg_interleaved_spmv_kernel(ctx.h, u.h, p.h, q.h, z.h, alpha, beta, C.byref(out)))
    return out.value


def fused_prec(ctx, r, z, q, alpha):
    rn, ka = C.c_double(), C.c_double()
    check(lib().acg_interleaved_prec_kernel(ctx.h, r.h, z.h, q.h, alpha, C.byref(rn), C.byref(ka)))
    return rn.value, ka.value


def config(epsilon=1e-5, tau=1e-20, maxiter=500, variant=INTERLEAVED, timings=False,
           backend=MATRIX_FREE, layout=VERTICAL):
    c = SolverConfig()
    lib().acg_solver_config_default(C.byref(c))
    c.epsilon, c.tau, c.maxiter, c.variant = epsilon, tau, maxiter, variant
    c.record_timings = 1 if timings else 0
    c.backend, c.layout = backend, layout
    return c


def _result(res):
    """SolveResult dict from an acg_solve_result whose histories the library
    allocated (NULL caller buffers); releases them."""
    t = res.timings
    try:
        hs = [np.ctypeslib.as_array(res.history[a], shape=(n,)).copy() if n > 0 else np.zeros(0)
              for a, n in enumerate((res.n_residual, res.n_kappa, res.n_alpha, res.n_beta))]
    finally:
        lib().acg_solve_result_release(C.byref(res))
    return {
        "iterations": res.iterations, "converged": bool(res.converged),
        "true_residual": res.true_residual,
        "residual_history": hs[0], "kappa_history": hs[1],
        "alpha_history": hs[2], "beta_history": hs[3],
        "timings": {k: getattr(t, k) for k, _ in KernelTimings._fields_},
        "kernel_launches": res.kernel_launches,
    }


def solve(ctx, f: Field, u0: Field | None = None, u_out: Field | None = None, **kw):
    cfg = config(**kw)
    res = SolveResult()
    check(lib().acg_solve(ctx.h, f.h, u0.h if u0 else None, C.byref(cfg), u_out.h if u_out else None,
                          C.byref(res), None, None, None, None))
    return _result(res)


def solve_host(ctx, f, u0=None, layout=VERTICAL, out=None, **kw):
    """Host buffers in, host buffer out (acg_solve_host)."""
    cfg = config(**kw)
    f = np.ascontiguousarray(f, dtype=ctx.np_dtype)
    u = out if out is not None else np.empty_like(f)
    res = SolveResult()
    check(lib().acg_solve_host(ctx.h, layout, _vptr(f),
                               _vptr(np.ascontiguousarray(u0, dtype=ctx.np_dtype)) if u0 is not None else None,
                               C.byref(cfg), _vptr(u), C.byref(res), None, None, None, None))
    return u, _result(res)


class Solver:
    """Step-level control of the device-resident loop (acg_solver_*)."""

    def __init__(self, ctx, **kw):
        self.cfg = config(**kw)
        h = C.c_void_p()
        check(lib().acg_solver_create(C.byref(h), ctx.h, C.byref(self.cfg)))
        self.h, self.ctx = h, ctx
        ctx._children.add(self)

    def start(self, f, u0=None):
        check(lib().acg_solver_start(self.h, f.h, u0.h if u0 else None))

    def iterate(self, n):
        check(lib().acg_solver_iterate(self.h, n))

    def time_kernels(self, on=True):
        check(lib().acg_solver_time_kernels(self.h, 1 if on else 0))

    def kernel_times(self):
        n1, n2 = C.c_int(), C.c_int()
        t1, t2 = C.c_double(), C.c_double()
        check(lib().acg_solver_kernel_times(self.h, C.byref(n1), C.byref(t1), C.byref(n2), C.byref(t2)))
        return {"fused_prec": (n1.value, t1.value), "fused_spmv": (n2.value, t2.value)}

    def finish(self, u_out=None):
        res = SolveResult()
        check(lib().acg_solver_finish(self.h, u_out.h if u_out else None, C.byref(res),
                                      None, None, None, None))
        return _result(res)

    def close(self):
        if self.h:
            lib().acg_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def launch_count():
    return lib().acg_kernel_launch_count()


class HostBuffer:
    """Pinned host memory as a numpy array (acg_host_alloc)."""

    def __init__(self, shape, dtype=np.float64):
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = C.c_void_p()
        check(lib().acg_host_alloc(C.byref(p), n))
        self.p = p
        buf = (C.c_char * n).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def close(self):
        if self.p:
            self.array = None
            lib().acg_host_free(self.p)
            self.p = None
