"""Kernel-module shim: the reference's backend ABI, served by the GPU.

The reference dispatches its hot loop through a registry of kernel modules
(kernels.py:23-52); a module exposes ``BACKEND_NAME`` and
``assign_ivf(indptr, terms, vals, m_indptr, m_cids, m_vals, rho, labels, ctr)``
(_kernels.pyx:106-128) with 1-based ids, float64 values, labels written in
place and ``ctr[0..2] += postings touched``.  This module is that object:
registering it makes the reference's own ``assign_ivf`` / ``run`` (and its
backend-parametrised tests) execute on the B200 kernels:

    import sparse_kmeans.kernels as K
    from paper_2002_09094_b200 import backend
    K._MODULES["b200"] = backend

The call goes straight to the C entry point ivfkm_assign_ivf_host (host
buffers in, host labels out), i.e. the same ABI a cgo/JNI/ctypes binding of
the reference's FFI would use.  The reference's ``rho`` scratch is accepted
and ignored: the similarity vector lives in registers on the device.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

BACKEND_NAME = "b200"


def _arr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, C.c_void_p(a.ctypes.data)


def assign_ivf(indptr, terms, vals, m_indptr, m_cids, m_vals, rho, labels, ctr) -> None:
    lib = _lib.load()
    ip, p_ip = _arr(indptr, np.int64)
    t, p_t = _arr(terms, np.int32)
    v, p_v = _arr(vals, np.float64)
    mp, p_mp = _arr(m_indptr, np.int64)
    mc, p_mc = _arr(m_cids, np.int32)
    mv, p_mv = _arr(m_vals, np.float64)
    n = ip.size - 1
    dim = mp.size - 1
    k = int(np.asarray(rho).shape[0])
    out = np.empty(n, dtype=np.int32)
    c = np.zeros(5, dtype=np.int64)
    rc = lib.ivfkm_assign_ivf_host(n, p_ip, p_t, p_v, dim, p_mp, p_mc, p_mv, k,
                                   C.c_void_p(out.ctypes.data), C.c_void_p(c.ctypes.data))
    if rc == -6:
        from .types import CorruptionError

        raise CorruptionError("posting id outside its owner range")
    _lib.check(rc, "ivfkm_assign_ivf_host")
    labels[:] = out
    ctr[:3] += c[:3]


def assign_ivfd(x_indptr, x_oids, x_vals, m_indptr, m_terms, m_vals, rho, rho_max, labels,
                ctr) -> None:
    """_kernels.pyx:178-207: objects given as their inverted file, means
    mean-major; ``rho`` / ``rho_max`` scratch accepted and left untouched."""
    lib = _lib.load()
    xp, p_xp = _arr(x_indptr, np.int64)
    xo, p_xo = _arr(x_oids, np.int32)
    xv, p_xv = _arr(x_vals, np.float64)
    mp, p_mp = _arr(m_indptr, np.int64)
    mt, p_mt = _arr(m_terms, np.int32)
    mv, p_mv = _arr(m_vals, np.float64)
    n = int(np.asarray(rho).shape[0])
    dim = xp.size - 1
    k = mp.size - 1
    out = np.empty(n, dtype=np.int32)
    c = np.zeros(5, dtype=np.int64)
    rc = lib.ivfkm_assign_ivfd_host(n, p_xp, p_xo, p_xv, dim, p_mp, p_mt, p_mv, k,
                                    C.c_void_p(out.ctypes.data), C.c_void_p(c.ctypes.data))
    if rc == -6:
        from .types import CorruptionError

        raise CorruptionError("posting id outside its owner range")
    _lib.check(rc, "ivfkm_assign_ivfd_host")
    labels[:] = out
    ctr[:3] += c[:3]


def register(kernels_module) -> None:
    """Add this backend to a reference ``sparse_kmeans.kernels`` registry."""
    kernels_module._MODULES[BACKEND_NAME] = __import__(__name__, fromlist=["x"])
