"""NPY v1.0 tensor ingestion for real-model dumps (the ``cli``
module's load_tensor_file / save_tensor_file; absent from the reference's code).

Accepted: little-endian float16, float32, and bfloat16 stored as uint16 (with
``bf16=True``, since NPY has no bfloat16 tag); C order; exactly 4-D (B, H, S, d).
Values become the FP16 carrier with one RNE rounding (BF16 -> FP32 is exact).
Errors name the byte offset of the offending header field.
"""
from __future__ import annotations

import ast
import struct

import numpy as np

MAGIC = b"\x93NUMPY"


class NpyFormatError(ValueError):
    pass


def _parse_header(buf: bytes, path: str) -> tuple[dict, int]:
    if len(buf) < 10 or buf[:6] != MAGIC:
        raise NpyFormatError(f"{path}: bad magic at byte 0 (expected \\x93NUMPY)")
    major, minor = buf[6], buf[7]
    if major == 1:
        (hlen,) = struct.unpack_from("<H", buf, 8)
        hstart = 10
    elif major in (2, 3):
        (hlen,) = struct.unpack_from("<I", buf, 8)
        hstart = 12
    else:
        raise NpyFormatError(f"{path}: unsupported NPY version {major}.{minor} at byte 6")
    if len(buf) < hstart + hlen:
        raise NpyFormatError(f"{path}: header truncated at byte {len(buf)} (needs {hstart + hlen})")
    try:
        hdr = ast.literal_eval(buf[hstart:hstart + hlen].decode("latin1"))
    except (ValueError, SyntaxError) as e:
        raise NpyFormatError(f"{path}: unparsable header dict at byte {hstart}: {e}") from None
    if not isinstance(hdr, dict) or not {"descr", "fortran_order", "shape"} <= set(hdr):
        raise NpyFormatError(f"{path}: header at byte {hstart} lacks descr/fortran_order/shape")
    return hdr, hstart + hlen


def load_tensor_file(path: str, bf16: bool = False) -> np.ndarray:
    """Read a 4-D NPY tensor and return it as float16 (the FP16 input carrier)."""
    with open(path, "rb") as f:
        buf = f.read()
    hdr, off = _parse_header(buf, path)
    descr, shape = hdr["descr"], tuple(hdr["shape"])
    if hdr["fortran_order"]:
        raise NpyFormatError(f"{path}: Fortran-ordered arrays are not supported (header byte 10)")
    if len(shape) != 4:
        raise NpyFormatError(f"{path}: expected a 4-D (B, H, S, d) tensor, got shape {shape}")
    kinds = {"<f2": np.float16, "<f4": np.float32, "<u2": np.uint16, "|u2": np.uint16}
    if descr not in kinds:
        raise NpyFormatError(f"{path}: unsupported dtype {descr!r} (float16, float32, or "
                             "bfloat16 as uint16)")
    if kinds[descr] is np.uint16 and not bf16:
        raise NpyFormatError(f"{path}: uint16 payload needs bf16=True (--dtype bf16)")
    dt = np.dtype(kinds[descr])
    n = int(np.prod(shape))
    if len(buf) - off < n * dt.itemsize:
        raise NpyFormatError(f"{path}: payload truncated at byte {len(buf)} "
                             f"(needs {off + n * dt.itemsize})")
    a = np.frombuffer(buf, dtype=dt, count=n, offset=off).reshape(shape)
    if dt == np.uint16:  # bfloat16 bits -> float32 (exact) -> float16
        a = (a.astype(np.uint32) << 16).view(np.float32)
    return a.astype(np.float16)


def save_tensor_file(path: str, a: np.ndarray) -> None:
    """Write NPY v1.0 (float16 or float32, C order); load_tensor_file round-trips bit-exactly."""
    a = np.ascontiguousarray(a)
    if a.dtype not in (np.float16, np.float32):
        raise ValueError("save_tensor_file writes float16 or float32")
    descr = "<f2" if a.dtype == np.float16 else "<f4"
    hdr = "{'descr': '%s', 'fortran_order': False, 'shape': %s, }" % (descr, repr(tuple(a.shape)))
    pad = 64 - (10 + len(hdr) + 1) % 64
    hdr = hdr + " " * (pad % 64) + "\n"
    with open(path, "wb") as f:
        f.write(MAGIC + bytes([1, 0]) + struct.pack("<H", len(hdr)) + hdr.encode("latin1"))
        f.write(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes())
