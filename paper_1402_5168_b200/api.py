"""Thin Python binding of include/rexp.h: setup / apply / free (+ queries).

Argument marshalling only - every step of the apply runs in librexp.so's CUDA
kernels.  There is no CPU implementation of the apply here or anywhere in the
package.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

MODELS = {"rsw": 0, "wave": 1}
STORES = {"auto": 0, "shared": 1, "pernode": 2}


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Handle:
    """Owns a rexp_handle (operator store on one device)."""

    def __init__(self, ptr, model, nrhs, device):
        self.ptr = ptr
        self.model = model
        self.nrhs = nrhs
        self.device = device
        lib = _lib.load()
        self.N = int(lib.rexp_num_nodes(ptr))
        self.num_poles = int(lib.rexp_num_poles(ptr))
        self.num_half_poles = int(lib.rexp_num_half_poles(ptr))

    # -- queries ------------------------------------------------------------
    def poles(self):
        lib = _lib.load()
        a = np.zeros(2 * self.num_poles)
        b = np.zeros(2 * self.num_poles)
        _lib.check(lib.rexp_get_poles(self.ptr, _dptr(a), _dptr(b)), "rexp_get_poles")
        return a.view(np.complex128), b.view(np.complex128)

    def accuracy(self):
        e = ctypes.c_double()
        m = ctypes.c_double()
        _lib.check(_lib.load().rexp_get_accuracy(self.ptr, ctypes.byref(e), ctypes.byref(m)), "rexp_get_accuracy")
        return e.value, m.value

    def node_coords(self):
        x = np.zeros(self.N)
        y = np.zeros(self.N)
        _lib.check(_lib.load().rexp_node_coords(self.ptr, _dptr(x), _dptr(y)), "rexp_node_coords")
        return x, y

    @property
    def store_bytes(self):
        return int(_lib.load().rexp_store_bytes(self.ptr))

    @property
    def work_bytes(self):
        return int(_lib.load().rexp_work_bytes(self.ptr))

    @property
    def launches_per_step(self):
        return int(_lib.load().rexp_launches_per_step(self.ptr))

    @property
    def leaf_solver(self):
        """'spectral' (tensor-product leaf inverse in the eigenbasis of the 1-D
        second-derivative block, pole loop in the spectral basis) or 'dense'
        (q^2 x q^2 leaf operators)."""
        v = int(_lib.load().rexp_leaf_solver(self.ptr))
        return {0: "dense", 1: "spectral"}.get(v, None)

    @property
    def stage_report(self):
        buf = ctypes.create_string_buffer(4096)
        _lib.check(_lib.load().rexp_stage_report(self.ptr, buf, 4096), "rexp_stage_report")
        return buf.value.decode()

    @property
    def partial_len(self):
        return int(_lib.load().rexp_partial_len(self.ptr))

    def close(self):
        if self.ptr:
            _lib.load().rexp_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def mesh_coords(n, p):
    """Node coordinates (x, y) of the n x n element, p x p node mesh (no setup needed)."""
    lib = _lib.load()
    N = int(lib.rexp_mesh_num_nodes(n, p))
    if N <= 0:
        raise ValueError("invalid mesh")
    x = np.zeros(N)
    y = np.zeros(N)
    _lib.check(lib.rexp_mesh_coords(n, p, _dptr(x), _dptr(y)), "rexp_mesh_coords")
    return x, y


def setup(model, n, p, tau, delta, Lambda, f=1.0, kappa=None, nrhs=1, store="auto", device=0,
          half_range=None, nthreads=0):
    """rexp_setup(L, tau, delta, Lambda): poles/weights + factorization + device store."""
    lib = _lib.load()
    prob = _lib.RexpProblem()
    prob.model = MODELS[model]
    prob.n = n
    prob.p = p
    prob.f = f
    kap = None
    if kappa is not None:
        kap = np.ascontiguousarray(kappa, dtype=np.float64)
        prob.kappa = _dptr(kap)
    opt = _lib.RexpOptions()
    lib.rexp_default_options(ctypes.byref(opt))
    opt.nrhs = nrhs
    opt.store = STORES[store]
    opt.device = device
    if half_range is not None:
        opt.half_begin, opt.half_end = half_range
    opt.nthreads = nthreads
    out = ctypes.c_void_p()
    _lib.check(lib.rexp_setup(ctypes.byref(prob), tau, delta, Lambda, ctypes.byref(opt), ctypes.byref(out)),
               "rexp_setup")
    return Handle(out, model, nrhs, device)


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(stream)


def apply(handle: Handle, u, nsteps, stream=None):
    """rexp_apply: u <- step^nsteps u, in place.

    u: a CUDA torch.complex128 tensor [nrhs, 3, N] (device path, async on the
    current torch stream) or a numpy complex128 array (host path: copies in,
    steps, copies back, synchronizes).
    """
    lib = _lib.load()
    if isinstance(u, np.ndarray):
        if u.dtype != np.complex128 or not u.flags.c_contiguous or u.size != handle.nrhs * 3 * handle.N:
            raise ValueError("host state must be C-contiguous complex128 of size nrhs*3*N")
        _lib.check(lib.rexp_apply(handle.ptr, u.ctypes.data, nsteps, 0, ctypes.c_void_p(_stream_ptr(stream))),
                   "rexp_apply")
        return u
    import torch
    if not (u.is_cuda and u.dtype == torch.complex128 and u.is_contiguous() and u.numel() == handle.nrhs * 3 * handle.N):
        raise ValueError("device state must be a contiguous CUDA complex128 tensor of size nrhs*3*N")
    _lib.check(lib.rexp_apply(handle.ptr, u.data_ptr(), nsteps, 1, ctypes.c_void_p(_stream_ptr(stream))),
               "rexp_apply")
    return u


def _check_sharded_args(handle: Handle, u, e):
    import torch
    dev = u.device if isinstance(u, torch.Tensor) else None
    if not (isinstance(u, torch.Tensor) and u.is_cuda and u.dtype == torch.complex128 and u.is_contiguous()
            and u.numel() == handle.nrhs * 3 * handle.N):
        raise ValueError("u must be a contiguous CUDA complex128 tensor of size nrhs*3*N")
    if not (isinstance(e, torch.Tensor) and e.is_cuda and e.dtype == torch.float64 and e.is_contiguous()
            and e.numel() == handle.partial_len):
        raise ValueError("e must be a contiguous CUDA float64 tensor of length partial_len")
    if e.device != dev or (handle.device >= 0 and dev.index != handle.device):
        raise ValueError("u and e must live on the handle's device")


def step_partial(handle: Handle, u, e, stream=None):
    """Pole-sharded step, part 1: this handle's pole sums into e (CUDA float64, partial_len)."""
    _check_sharded_args(handle, u, e)
    _lib.check(_lib.load().rexp_step_partial(handle.ptr, u.data_ptr(), e.data_ptr(),
                                             ctypes.c_void_p(_stream_ptr(stream))), "rexp_step_partial")


def step_finish(handle: Handle, e, u, stream=None):
    """Pole-sharded step, part 2: recover the new state from the all-reduced pole sums."""
    _check_sharded_args(handle, u, e)
    _lib.check(_lib.load().rexp_step_finish(handle.ptr, e.data_ptr(), u.data_ptr(),
                                            ctypes.c_void_p(_stream_ptr(stream))), "rexp_step_finish")


KERNEL_CLASSES = ["pre", "leaf_up", "leaf_flux", "merge_up", "root", "merge_down", "leaf_down", "pole_sum", "recover"]


def timing_begin(handle: Handle):
    _lib.check(_lib.load().rexp_timing_begin(handle.ptr), "rexp_timing_begin")


def timing_end(handle: Handle):
    """{class: (device_ms, launches)} accumulated since timing_begin (CUDA events)."""
    ms = np.zeros(len(KERNEL_CLASSES))
    cnt = np.zeros(len(KERNEL_CLASSES), dtype=np.int32)
    _lib.check(_lib.load().rexp_timing_end(handle.ptr, _dptr(ms), cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))),
               "rexp_timing_end")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


def free(handle: Handle):
    handle.close()


# -- host-only export (setup verification tests) ---------------------------
def export_level_info(handle: Handle, lev):
    info = (ctypes.c_int64 * 8)()
    _lib.check(_lib.load().rexp_export_level_info(handle.ptr, lev, info), "rexp_export_level_info")
    return list(info)


def export_num_levels(handle: Handle):
    return int(_lib.load().rexp_export_num_levels(handle.ptr))


def export_matrix(handle: Handle, half_index, lev, node, which, rows, cols):
    out = np.zeros(2 * rows * cols)
    _lib.check(_lib.load().rexp_export_matrix(handle.ptr, half_index, lev, node, which, _dptr(out)),
               "rexp_export_matrix")
    return out.view(np.complex128).reshape(cols, rows).T   # column-major -> (rows, cols)


def export_index(handle: Handle, lev, which, count):
    out = np.zeros(count, dtype=np.int32)
    _lib.check(_lib.load().rexp_export_index(handle.ptr, lev, which, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))),
               "rexp_export_index")
    return out
