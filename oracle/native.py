"""TEST INFRASTRUCTURE ONLY -- ctypes loader for the C oracle (cq_oracle.c).

``build()`` compiles oracle/cq_oracle.c with gcc (-O2 -fopenmp
-ffp-contract=off) into oracle/_build/liboracle.so; the built library travels
to the GPU box with the snapshot (git-ignored, not gpurun-ignored).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cq_oracle.c")
LIB = os.path.join(HERE, "_build", "liboracle.so")

_lib = None


def build(force=False) -> str:
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               SRC, "-o", LIB, "-lm"]
        subprocess.run(cmd, check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_saxpy_f64.argtypes = [ctypes.c_double, P, P, P, i64]
        L.oracle_saxpy_f32.argtypes = [ctypes.c_float, P, P, P, i64]
        L.oracle_wave5_f64.argtypes = [P, P, P, i64, i64, i64, i64, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double]
        L.oracle_wave5_f32.argtypes = [P, P, P, i64, i64, i64, i64, ctypes.c_float, ctypes.c_float,
                                       ctypes.c_float]
        L.oracle_nbody_accel.argtypes = [P, i64, i64, i64, ctypes.c_double, P]
        L.oracle_nbody_accel_idx.argtypes = [P, i64, P, i64, ctypes.c_double, P]
        L.oracle_sgemm_rows.argtypes = [P, P, i64, i64, P, i64, P, P]
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def saxpy(alpha, x, y):
    z = np.empty_like(x)
    if x.dtype == np.float32:
        lib().oracle_saxpy_f32(ctypes.c_float(alpha), _p(x), _p(y), _p(z), x.size)
    else:
        lib().oracle_saxpy_f64(ctypes.c_double(alpha), _p(x), _p(y), _p(z), x.size)
    return z


def wave_step(u, upr, c, k2=2.0, k4=4.0, rows=None, out=None):
    """One leapfrog step; returns the new field (writes ``out`` if given)."""
    h, w = u.shape
    if out is None:
        out = np.empty_like(upr)
    r0, r1 = rows if rows is not None else (0, h)
    if u.dtype == np.float32:
        lib().oracle_wave5_f32(_p(u), _p(upr), _p(out), h, w, r0, r1, ctypes.c_float(c),
                               ctypes.c_float(k2), ctypes.c_float(k4))
    else:
        lib().oracle_wave5_f64(_p(u), _p(upr), _p(out), h, w, r0, r1, ctypes.c_double(c),
                               ctypes.c_double(k2), ctypes.c_double(k4))
    return out


def wave_run(u0, up0, steps, c):
    """``steps`` ping-pong steps (workloads.wave_program); returns (u, up)."""
    u = np.ascontiguousarray(u0).copy()
    up = np.ascontiguousarray(up0).copy()
    for s in range(steps):
        if s % 2 == 0:
            wave_step(u, up, c, out=up)
        else:
            wave_step(up, u, c, out=u)
    return u, up


def nbody_accel(pos, i0, i1, eps2):
    pos = np.ascontiguousarray(pos, dtype=np.float32)
    acc = np.empty((i1 - i0, 3), np.float64)
    lib().oracle_nbody_accel(_p(pos), pos.shape[0], i0, i1, ctypes.c_double(eps2), _p(acc))
    return acc


def nbody_accel_idx(pos, idx, eps2):
    pos = np.ascontiguousarray(pos, dtype=np.float32)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    acc = np.empty((idx.size, 3), np.float64)
    lib().oracle_nbody_accel_idx(_p(pos), pos.shape[0], _p(idx), idx.size, ctypes.c_double(eps2), _p(acc))
    return acc


def sgemm_rows(a, b, rows, with_abs=True):
    """float64 C rows (and sum |a||b| per element unless ``with_abs`` is
    False, then None)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    n = b.shape[1]
    c = np.empty((rows.size, n), np.float64)
    cabs = np.empty((rows.size, n), np.float64) if with_abs else None
    lib().oracle_sgemm_rows(_p(a), _p(b), n, a.shape[1], _p(rows), rows.size, _p(c),
                            _p(cabs) if with_abs else None)
    return c, cabs
