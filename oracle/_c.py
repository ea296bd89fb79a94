"""ctypes loader for oracle/ring_c.c (TEST INFRASTRUCTURE ONLY).

The shared object is compiled on first use with plain ``gcc -O2 -fopenmp``;
``__graft_entry__.build()`` also compiles it (building the checker is not
using it).
"""
import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ring_c.c")
_SO = os.path.join(_HERE, "_ring_c.so")
_lock = threading.Lock()
_lib = None
# call counter (bench.py's cost model of an oracle compare is checked against it in tests/)
CALLS = {"ring_mul": 0}


def build(force=False):
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".%d.tmp" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            u64p = ctypes.POINTER(ctypes.c_uint64)
            i64p = ctypes.POINTER(ctypes.c_int64)
            i32p = ctypes.POINTER(ctypes.c_int32)
            L.ring_mul.argtypes = [u64p, u64p, u64p, ctypes.c_int, i64p, ctypes.c_uint64, ctypes.c_int]
            L.poly_mod_phi.argtypes = [u64p, ctypes.c_int, i64p, ctypes.c_int, ctypes.c_uint64]
            L.eval_naive.argtypes = [u64p, ctypes.c_int, i32p, ctypes.c_int, ctypes.c_int, u64p,
                                     ctypes.c_uint64, u64p]
            L.vec_mulmod.argtypes = [u64p, u64p, u64p, ctypes.c_int64, ctypes.c_uint64]
            L.vec_mulscalar.argtypes = [u64p, ctypes.c_uint64, u64p, ctypes.c_int64, ctypes.c_uint64]
            _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def ring_mul(a, b, phi, q, m):
    """Schoolbook a*b mod (q, Phi_m); a, b: uint64[n] residues in [0, q)."""
    CALLS["ring_mul"] += 1
    a = u64(a)
    b = u64(b)
    n = a.shape[0]
    out = np.empty(n, dtype=np.uint64)
    ph = np.ascontiguousarray(phi, dtype=np.int64)
    lib().ring_mul(_p(a, ctypes.c_uint64), _p(b, ctypes.c_uint64), _p(out, ctypes.c_uint64), n,
                   _p(ph, ctypes.c_int64), int(q), int(m))
    return out


def poly_mod_phi(t, phi, q):
    """Long division of t (residues mod q, any length) by monic Phi_m; returns length n."""
    n = len(phi) - 1
    t = np.array(t, dtype=np.uint64, copy=True)
    if t.shape[0] < n:
        t = np.concatenate([t, np.zeros(n - t.shape[0], dtype=np.uint64)])
    ph = np.ascontiguousarray(phi, dtype=np.int64)
    lib().poly_mod_phi(_p(t, ctypes.c_uint64), t.shape[0], _p(ph, ctypes.c_int64), n, int(q))
    return t[:n].copy()


def eval_naive(f, z, m, wpow, q):
    f = u64(f)
    z = np.ascontiguousarray(z, dtype=np.int32)
    wpow = u64(wpow)
    out = np.empty(z.shape[0], dtype=np.uint64)
    lib().eval_naive(_p(f, ctypes.c_uint64), f.shape[0], _p(z, ctypes.c_int32), z.shape[0], m,
                     _p(wpow, ctypes.c_uint64), int(q), _p(out, ctypes.c_uint64))
    return out


def vec_mulmod(a, b, q):
    a = u64(a)
    b = u64(b)
    out = np.empty_like(a)
    lib().vec_mulmod(_p(a, ctypes.c_uint64), _p(b, ctypes.c_uint64), _p(out, ctypes.c_uint64),
                     a.size, int(q))
    return out


def vec_mulscalar(a, c, q):
    a = u64(a)
    out = np.empty_like(a)
    lib().vec_mulscalar(_p(a, ctypes.c_uint64), int(c) % int(q), _p(out, ctypes.c_uint64), a.size,
                        int(q))
    return out
