"""CPU oracle for permuting sorted LCO sparse tensors (arXiv 1802.02619).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this package.
The product (``paper_1802_02619_b200``) never imports it; the two share no code.

Thin ctypes marshalling over ``oracle/oracle.cpp`` (plain C++, ``/``, ``%`` and
``std::stable_sort``).  See that file for the passages each function follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_SRC_PAR = os.path.join(_HERE, "oracle_par.cpp")
_LIB_PAR = os.path.join(_HERE, "liboracle_par.so")

_ERR = {1: "bad argument", 2: "coordinate/key out of range", 3: "product of dims > 2^63-1",
        4: "RP claim violated (region not ordered by a resting index)"}


def _compile(src, lib, extra, force):
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        tmp = lib + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", *extra, "-o", tmp,
                               src])
        os.replace(tmp, lib)
    return lib


def build(force: bool = False) -> str:
    """Compile oracle.cpp with g++ (-O2, single thread) and the all-cores variant
    oracle_par.cpp (-fopenmp).  Returns the single-thread .so path."""
    _compile(_SRC_PAR, _LIB_PAR, ["-fopenmp"], force)
    return _compile(_SRC, _LIB, [], force)


_lib = None


def _get():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        u64p = ctypes.POINTER(ctypes.c_uint64)
        for name in ("oracle_permute", "oracle_sort", "oracle_rp_permute"):
            f = getattr(_lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [ctypes.c_int, u64p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                          ctypes.c_void_p]
        _lib.oracle_shuffle.restype = ctypes.c_int
        _lib.oracle_shuffle.argtypes = [ctypes.c_int, u64p, ctypes.c_void_p, ctypes.c_uint64,
                                        ctypes.c_void_p, ctypes.c_void_p]
        _lib.oracle_linearize.restype = ctypes.c_int
        _lib.oracle_linearize.argtypes = [ctypes.c_int, u64p, u64p, u64p]
        _lib.oracle_delinearize.restype = ctypes.c_int
        _lib.oracle_delinearize.argtypes = [ctypes.c_int, u64p, ctypes.c_uint64, u64p]
        _lib.oracle_classify.restype = ctypes.c_int
        _lib.oracle_classify.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _lib.oracle_partition.restype = ctypes.c_int
        _lib.oracle_partition.argtypes = [ctypes.c_int, u64p, ctypes.c_void_p, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
                                          ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.oracle_compress.restype = ctypes.c_int
        _lib.oracle_compress.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib.oracle_add.restype = ctypes.c_int
        _lib.oracle_add.argtypes = [ctypes.c_int, u64p, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return _lib


_lib_par = None


def _get_par():
    global _lib_par
    if _lib_par is None:
        build()
        _lib_par = ctypes.CDLL(_LIB_PAR)
        f = _lib_par.oracle_permute_par
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p,
                      ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib_par.oracle_par_threads.restype = ctypes.c_int
    return _lib_par


def par_threads() -> int:
    """Threads the all-cores oracle uses (OpenMP: the process affinity mask by default)."""
    return int(_get_par().oracle_par_threads())


def _dims(dims):
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))
    return d, d.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _perm(perm, order):
    if perm is None:
        perm = range(order)
    return np.ascontiguousarray(np.asarray(perm, dtype=np.int32))


def _check(rc):
    if rc != 0:
        raise ValueError(f"oracle: {_ERR.get(rc, rc)}")


def _ptr(a):
    return None if a is None else a.ctypes.data


def linearize(dims, coords) -> int:
    d, dp = _dims(dims)
    c = np.ascontiguousarray(np.asarray(coords, dtype=np.uint64))
    out = np.zeros(1, dtype=np.uint64)
    _check(_get().oracle_linearize(len(d), dp, c.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                   out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return int(out[0])


def delinearize(dims, key: int) -> list:
    d, dp = _dims(dims)
    out = np.zeros(len(d), dtype=np.uint64)
    _check(_get().oracle_delinearize(len(d), dp, int(key),
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return [int(x) for x in out]


def shuffle(dims, perm, keys) -> np.ndarray:
    d, dp = _dims(dims)
    p = _perm(perm, len(d))
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    out = np.empty_like(k)
    _check(_get().oracle_shuffle(len(d), dp, p.ctypes.data, len(k), _ptr(k), _ptr(out)))
    return out


def classify(perm) -> list:
    """1 = rearrangement index, 0 = resting index, by NEW position."""
    p = _perm(perm, None)
    out = np.zeros(len(p), dtype=np.int32)
    _check(_get().oracle_classify(len(p), p.ctypes.data, out.ctypes.data))
    return [int(x) for x in out]


def _run(fn, dims, perm, keys, vals, idx):
    d, dp = _dims(dims)
    p = _perm(perm, len(d))
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    n = len(k)
    v = None if vals is None else np.ascontiguousarray(np.asarray(vals, dtype=np.float64))
    ix = None if idx is None else np.ascontiguousarray(np.asarray(idx, dtype=np.uint32))
    ko = np.empty(n, dtype=np.uint64)
    vo = None if v is None else np.empty(n, dtype=np.float64)
    po = np.empty(n, dtype=np.uint32)
    _check(fn(len(d), dp, p.ctypes.data, n, _ptr(k), _ptr(v), _ptr(ix), _ptr(ko), _ptr(vo),
              _ptr(po)))
    return ko, vo, po


def permute(dims, perm, keys, vals=None, idx=None):
    """LIV shuffle + std::stable_sort (the definition).  Returns (keys, vals, perm)."""
    return _run(_get().oracle_permute, dims, perm, keys, vals, idx)


def permute_par(dims, perm, keys, vals=None, idx=None):
    """The same definition on all cores (OpenMP decode / gather, __gnu_parallel::stable_sort);
    bit-identical to permute()."""
    return _run(_get_par().oracle_permute_par, dims, perm, keys, vals, idx)


def sort(dims, perm, keys, vals=None, idx=None):
    return _run(_get().oracle_sort, dims, perm, keys, vals, idx)


def rp_permute(dims, perm, keys, vals=None, idx=None):
    """The paper's RP algorithm step by step (regions, shaved keys, recursion)."""
    return _run(_get().oracle_rp_permute, dims, perm, keys, vals, idx)


def partition(dims, perm, keys, vals, idx_base, splitters):
    d, dp = _dims(dims)
    p = _perm(perm, len(d))
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    v = np.ascontiguousarray(np.asarray(vals, dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(splitters, dtype=np.uint64))
    world = len(s) + 1
    n = len(k)
    sk = np.empty(n, dtype=np.uint64)
    sv = np.empty(n, dtype=np.float64)
    si = np.empty(n, dtype=np.uint32)
    cnt = np.zeros(world, dtype=np.uint64)
    _check(_get().oracle_partition(len(d), dp, p.ctypes.data, n, _ptr(k), _ptr(v), int(idx_base),
                                   world, _ptr(s), _ptr(sk), _ptr(sv), _ptr(si), _ptr(cnt)))
    return sk, sv, si, cnt


def add(dims_b, match, keys_a, vals_a, keys_b, vals_b, sign=1.0):
    """Index-matched addition C = A + sign * permute(B, match):
    union of supports, collisions summed, explicit zeros kept, ascending keys."""
    d, dp = _dims(dims_b)
    p = _perm(match, len(d))
    ka = np.ascontiguousarray(np.asarray(keys_a, dtype=np.uint64))
    va = np.ascontiguousarray(np.asarray(vals_a, dtype=np.float64))
    kb = np.ascontiguousarray(np.asarray(keys_b, dtype=np.uint64))
    vb = np.ascontiguousarray(np.asarray(vals_b, dtype=np.float64))
    kc = np.empty(len(ka) + len(kb), dtype=np.uint64)
    vc = np.empty(len(ka) + len(kb), dtype=np.float64)
    n = np.zeros(1, dtype=np.uint64)
    _check(_get().oracle_add(len(d), dp, p.ctypes.data, len(ka), _ptr(ka), _ptr(va), len(kb),
                             _ptr(kb), _ptr(vb), ctypes.c_double(sign), _ptr(kc), _ptr(vc),
                             _ptr(n)))
    m = int(n[0])
    return kc[:m].copy(), vc[:m].copy()


def compress(keys, n_major, n_minor, doubly=False):
    """CSR/CSC (doubly=False): (ptr[n_major+1], minor); DCSR/DCSC: (ids, ptr[nz+1], minor),
    from a major-first LCO matrix (§5.2 step 2)."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    n = len(k)
    minor = np.empty(n, dtype=np.uint64)
    if not doubly:
        ptr = np.empty(int(n_major) + 1, dtype=np.uint64)
        _check(_get().oracle_compress(n, _ptr(k), int(n_major), int(n_minor), 0, _ptr(ptr), None,
                                      _ptr(minor), None))
        return ptr, minor
    ids = np.empty(max(n, 1), dtype=np.uint64)
    ptr = np.empty(n + 1, dtype=np.uint64)
    nz = np.zeros(1, dtype=np.uint64)
    _check(_get().oracle_compress(n, _ptr(k), int(n_major), int(n_minor), 1, _ptr(ptr), _ptr(ids),
                                  _ptr(minor), _ptr(nz)))
    m = int(nz[0])
    return ids[:m].copy(), ptr[:m + 1].copy(), minor
