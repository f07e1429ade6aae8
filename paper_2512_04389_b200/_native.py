"""ctypes bindings of include/lbk.h (liblbk_host.so and liblbk.so).

The shared objects are built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2512_04389_b200.build``) into ``paper_2512_04389_b200/_lib``.
There is no fallback: a missing library raises ImportError-style errors at
first use, loudly.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import errors

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
HOST_LIB = os.path.join(LIB_DIR, "liblbk_host.so")
DEV_LIB = os.environ.get("LBK_DEV_LIB") or os.path.join(LIB_DIR, "liblbk.so")  # override: experiments only

LBK_OK = 0
LBK_ERR_ZERO_PIVOT = 1
LBK_ERR_SUPPORT = 2
LBK_ERR_DIM_MISMATCH = 3
LBK_ERR_CUDA = 4
LBK_ERR_NCCL = 5
LBK_ERR_OOM = 6
LBK_ERR_PIVOT_SWAP = 7
LBK_ERR_BAD_ARG = 8

c_i64p = C.POINTER(C.c_int64)
c_i32p = C.POINTER(C.c_int32)
c_i8p = C.POINTER(C.c_int8)
c_f64p = C.POINTER(C.c_double)
c_vpp = C.POINTER(C.c_void_p)


class LbkStatus(C.Structure):
    _fields_ = [("code", C.c_int32), ("block", C.c_int32), ("col", C.c_int32),
                ("pad", C.c_int32), ("msg", C.c_char * 256)]


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctype)


_host = None
_dev = None


def _declare(lib, name, restype, argtypes):
    fn = getattr(lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    return fn


def host_lib():
    global _host
    if _host is None:
        if not os.path.exists(HOST_LIB):
            raise ImportError(f"{HOST_LIB} missing: run __graft_entry__.build() first")
        lib = C.CDLL(HOST_LIB)
        i64 = C.c_int64
        _declare(lib, "lbk_symbolic_nnz", C.c_int, [i64, c_i64p, c_i64p, c_i64p])
        _declare(lib, "lbk_symbolic_fill", C.c_int, [i64, c_i64p, c_i64p, c_i64p, c_i64p, c_i64p])
        _declare(lib, "lbk_blockptr", C.c_int, [i64, c_i64p, c_i64p, c_i64p])
        _declare(lib, "lbk_check_symmetric", C.c_int, [i64, c_i64p, c_i64p, c_i64p])
        _declare(lib, "lbk_partition_count", C.c_int, [i64, c_i64p, c_i64p, i64, c_i64p, c_i64p, c_i64p])
        _declare(lib, "lbk_partition_fill", C.c_int,
                 [i64, c_i64p, c_i64p, c_i64p, c_i64p, c_f64p, i64, c_i64p, i64, c_i64p, c_i64p, c_i64p,
                  c_f64p, c_i64p, c_i64p])
        _declare(lib, "lbk_levels_run", C.c_int,
                 [i64, i64, c_i64p, c_i64p, c_i64p, c_vpp, c_i64p, c_i64p])
        _declare(lib, "lbk_levels_fetch", C.c_int,
                 [C.c_void_p, c_i8p, c_i32p, c_i32p, c_i32p, c_i64p, c_i64p, c_i32p, c_i64p, c_i32p])
        _declare(lib, "lbk_levels_free", None, [C.c_void_p])
        _host = lib
    return _host


def check_host(rc: int, what: str) -> None:
    if rc == LBK_OK:
        return
    if rc == LBK_ERR_DIM_MISMATCH:
        raise errors.DimensionMismatch(f"{what}: filled pattern does not cover the input pattern")
    if rc == LBK_ERR_OOM:
        raise MemoryError(f"{what}: host allocation failed")
    raise errors.LuBlockError(f"{what}: native error {rc}")


def raise_status(st: LbkStatus, what: str) -> None:
    """Map a device lbk_status onto the reference exception classes."""
    code = st.code
    if code == LBK_OK:
        return
    msg = st.msg.decode(errors="replace")
    if code == LBK_ERR_ZERO_PIVOT:
        raise errors.ZeroPivot(int(st.block), int(st.col))
    if code == LBK_ERR_SUPPORT:
        raise errors.SupportViolation(msg or f"{what}: product outside filled support")
    if code == LBK_ERR_DIM_MISMATCH:
        raise errors.DimensionMismatch(msg or what)
    if code == LBK_ERR_BAD_ARG:
        raise errors.BadParams(msg or what)
    if code == LBK_ERR_OOM:
        raise MemoryError(f"{what}: {msg}")
    raise errors.DeviceError(f"{what}: code {code}: {msg}")
