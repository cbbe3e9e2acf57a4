"""ctypes binding of the C-ABI in include/pasa_b200.h (libpasa_b200.so).

Loading the library needs no GPU; every compute entry point does.  There is no
fallback: if the library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(PKG, "_build", "libpasa_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "pasa_b200.h")

OK, EINVAL, EUNSUPPORTED, ECUDA, ENODEV = 0, -1, -2, -3, -4


class Desc(C.Structure):
    """Mirror of ``pasa_b200_desc``."""

    _fields_ = [
        ("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
        ("seq_q", C.c_int32), ("seq_kv", C.c_int32), ("head_dim", C.c_int32),
        ("s1", C.c_int32), ("s2", C.c_int32), ("causal", C.c_int32),
        ("layout", C.c_int32), ("beta", C.c_double), ("alpha", C.c_double),
    ]


_LIB = None


class Diag(C.Structure):
    """Mirror of ``pasa_b200_diag`` (device-side RunDiagnostics)."""

    _fields_ = [
        ("out_nonfinite", C.c_ulonglong), ("out_total", C.c_ulonglong),
        ("store_pos_inf", C.c_ulonglong), ("store_neg_inf", C.c_ulonglong),
        ("store_nan", C.c_ulonglong), ("store_finite_min", C.c_float),
        ("store_finite_max", C.c_float),
    ]


def exported_symbols_from_header() -> list[str]:
    """Every function the public header declares."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"PASA_B200_API\s+[\w\s\*]*?\b(pasa_b200_\w+)\s*\(", text)))


def load(path: str = SO) -> C.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} is missing: build it with `python -m paper_2503_01873_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(path)
    vp, dp = C.c_void_p, C.POINTER(Desc)
    L.pasa_b200_version.restype = C.c_int
    L.pasa_b200_last_error.restype = C.c_char_p
    L.pasa_b200_shift_entries.argtypes = [C.c_int32, C.c_double, C.c_double,
                                          C.POINTER(C.c_uint16), C.POINTER(C.c_uint16)]
    L.pasa_b200_check.argtypes = [dp]
    L.pasa_b200_workspace_size.restype = C.c_size_t
    L.pasa_b200_workspace_size.argtypes = [dp]
    L.pasa_b200_preprocess_keys.argtypes = [dp, vp, vp, vp, vp, C.c_float, vp]
    L.pasa_b200_attention_fwd.argtypes = [dp, vp, vp, vp, vp, vp, C.c_size_t, vp, vp]
    L.pasa_b200_attention_fwd_tiles.argtypes = [dp, vp, vp, vp, vp, vp, C.c_size_t, C.c_int32, C.c_int32, vp]
    L.pasa_b200_attention_fwd_prepped.argtypes = [dp, vp, vp, vp, vp, vp, vp]
    L.pasa_b200_preprocess.argtypes = [dp, vp, vp, vp, vp, vp, vp]
    L.pasa_b200_attention_host.argtypes = [dp, vp, vp, vp, vp]
    L.pasa_b200_attention_host_multi.argtypes = [dp, vp, vp, vp, vp, vp, C.c_int32]
    L.pasa_b200_flash_fp16_fwd.argtypes = [dp, vp, vp, vp, vp, vp]
    L.pasa_b200_preprocess_keys_host.argtypes = [dp, vp, vp, C.c_double, C.c_double]
    L.pasa_b200_diag_reset.argtypes = [vp, vp]
    L.pasa_b200_attention_host_diag.argtypes = [dp, vp, vp, vp, vp, C.POINTER(Diag)]
    u64, i32, f64 = C.c_uint64, C.c_int32, C.c_double
    L.pasa_b200_generate.argtypes = [i32, f64, f64, f64, u64, u64, u64, u64, vp, vp]
    L.pasa_b200_generate_resonance.argtypes = [u64, i32, i32, i32, i32, i32, f64, f64, vp, vp]
    _LIB = L
    return L


class PasaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != OK:
        msg = load().pasa_b200_last_error().decode()
        if rc == EINVAL:
            raise ValueError(msg)  # the reference's std::invalid_argument
        raise PasaError(rc, msg)
