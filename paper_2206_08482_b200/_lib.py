"""ctypes binding of libgmi.so (C-ABI declared in include/gmi.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
Python or CPU fallback: a missing library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgmi.so")

_lib = None

c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)

# name -> (restype, argtypes); kept in sync with include/gmi.h (tests check both ways).
PROTOTYPES: dict[str, tuple] = {
    "gmi_last_error": (C.c_char_p, []),
    "gmi_exit_code": (C.c_int, [C.c_int]),
    "gmi_version": (C.c_int, []),
    "gmi_dev_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                               C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong,
                               C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p,
                               C.c_longlong, C.c_int, C.c_void_p]),
}


class GmiError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[gmi error {code}] {msg}")
        self.code = code


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libgmi.so not built at {LIB_PATH}; run __graft_entry__.build() "
                "(no CPU fallback exists)")
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(code: int) -> None:
    if code != 0:
        msg = lib().gmi_last_error().decode(errors="replace")
        raise GmiError(code, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
