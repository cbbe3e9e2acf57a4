"""ctypes bindings for the TEST ORACLES (test infrastructure, not product code).

* ``Oracle``   -- our C restatement, ``oracle/_build/libpasa_oracle.so``
* ``RefLib``   -- the unmodified reference compiled by ``oracle/Makefile`` into
  ``oracle/_ref/libpasa_ref_capi.so`` (built in the dev container, where
  /root/reference exists; the prebuilt .so travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference legs may import this module.  The product package
(``paper_2503_01873_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OWN_SO = os.path.join(HERE, "_build", "libpasa_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpasa_ref_capi.so")

P64, P32, P16 = 0, 1, 2
PR1 = 3  # accumulation mode of the fused path's rank-1 pre-pass (orc_preprocess_keys)
# reference PolicyId (precision.hpp:41-47)
GOLDEN_FP64, FA_FP32, FA_PARTIAL_FP16, FA_FULL_FP16, PASA_FP16 = range(5)
POLICY_PRECS = {  # (accum, store, vec) -- precision.cpp:23-38
    GOLDEN_FP64: (P64, P64, P64),
    FA_FP32: (P32, P32, P32),
    FA_PARTIAL_FP16: (P32, P16, P16),
    FA_FULL_FP16: (P16, P16, P16),
    PASA_FP16: (P32, P16, P16),
}
BETA_STAR = 0.984497  # bench.hpp:93
LOG2E = 1.4426950408889634


def build(force: bool = False) -> None:
    """Build the oracle libraries (reference part only where its sources exist)."""
    if force or not os.path.exists(OWN_SO) or (
        os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)
    ):
        subprocess.run(["make", "-C", HERE, "-j8"], check=True, capture_output=True)


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class Shape(C.Structure):
    _fields_ = [
        ("B", C.c_size_t), ("Hq", C.c_size_t), ("Hkv", C.c_size_t),
        ("S1", C.c_size_t), ("S2", C.c_size_t), ("d", C.c_size_t),
        ("s1", C.c_size_t), ("s2", C.c_size_t),
        ("causal", C.c_int), ("q_offset", C.c_size_t),
    ]


class ModelParams(C.Structure):
    _fields_ = [
        ("beta", C.c_double), ("diag", C.c_double), ("off", C.c_double),
        ("lscale", C.c_double), ("tc_mode", C.c_int), ("c0", C.c_double),
        ("xscale", C.c_double), ("rowsum", C.c_int),
    ]


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class Problem:
    """Q (B,Hq,S1,d), K/V (B,Hkv,S2,d) as float64 carriers of FP16 values."""

    q: np.ndarray
    k: np.ndarray
    v: np.ndarray
    s1: int = 128
    s2: int = 128
    causal: bool = False
    q_offset: int = 0

    def shape(self) -> Shape:
        B, Hq, S1, d = self.q.shape
        _, Hkv, S2, _ = self.k.shape
        return Shape(B, Hq, Hkv, S1, S2, d, self.s1, self.s2, int(self.causal), self.q_offset)


class Oracle:
    """Our C restatement (oracle/pasa_oracle.c)."""

    def __init__(self, path: str = OWN_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_f16_round.restype = C.c_double
        L.orc_f16_round.argtypes = [C.c_double]
        L.orc_f16_round_array.argtypes = [_dp, _dp, C.c_size_t]
        L.orc_shift_entries.argtypes = [C.c_size_t, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.orc_invariance.argtypes = [C.c_double, C.c_size_t, _dp]
        L.orc_optimal_beta.argtypes = [C.c_double, C.c_size_t, C.c_double,
                                       C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.orc_generate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                   C.c_uint64, C.c_uint64, C.c_size_t, _dp]
        L.orc_generate_resonance.argtypes = [C.c_uint64, C.c_int, C.c_size_t, C.c_size_t,
                                             C.c_size_t, C.c_size_t, C.c_double, C.c_double, _dp]
        L.orc_rmse.restype = C.c_double
        L.orc_rmse.argtypes = [_dp, _dp, C.c_size_t]
        L.orc_nan_pct.restype = C.c_double
        L.orc_nan_pct.argtypes = [_dp, C.c_size_t]
        L.orc_golden.argtypes = [C.POINTER(Shape), _dp, _dp, _dp, _dp, C.c_int]
        L.orc_flash_ref.argtypes = [C.POINTER(Shape), _dp, _dp, _dp, _dp,
                                    C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_preprocess_keys.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                          C.c_size_t, C.c_double, C.c_double, C.c_int, C.c_int,
                                          C.c_double, _dp, C.c_int]
        L.orc_pasa_ref.argtypes = [C.POINTER(Shape), _dp, _dp, _dp, _dp, C.c_double,
                                   C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int]
        L.orc_model_inflation.restype = C.c_double
        L.orc_model_inflation.argtypes = [C.c_double, C.c_size_t, C.c_double]
        L.orc_model_pasa.argtypes = [C.POINTER(Shape), _dp, _dp, _dp, _dp,
                                     C.POINTER(ModelParams), C.c_int]
        L.orc_model_fa16.argtypes = [C.POINTER(Shape), _dp, _dp, _dp, _dp, C.c_int, C.c_int]

    # -- scalars -----------------------------------------------------------
    def f16(self, x):
        x = _f64(x)
        y = np.empty_like(x)
        self.lib.orc_f16_round_array(x.reshape(-1), y.reshape(-1), x.size)
        return y

    def shift_entries(self, s2: int, beta: float, alpha: float, prec: int = P16):
        d, o = C.c_double(), C.c_double()
        rc = self.lib.orc_shift_entries(s2, beta, alpha, prec, C.byref(d), C.byref(o))
        if rc:
            raise ValueError("shifting matrix: invalid arguments")
        return d.value, o.value

    def invariance(self, beta: float, n: int):
        out = np.zeros(5)
        if self.lib.orc_invariance(beta, n, out):
            raise ValueError("invariance: invalid arguments")
        return dict(zip(["a", "b", "inva_ideal", "inva_actual", "rel_err"], out))

    def optimal_beta(self, beta0: float, n: int = 128, tol: float = 1e-8):
        b, it = C.c_double(), C.c_int()
        if self.lib.orc_optimal_beta(beta0, n, tol, C.byref(b), C.byref(it)):
            raise RuntimeError("optimal_beta failed")
        return b.value, it.value

    # -- inputs --------------------------------------------------------------
    def generate(self, kind: str, x0: float, am: float, seed: int, B: int, H: int, S: int,
                 d: int, p: float = 0.001, tensor_ids=(0, 1, 2), Hkv: int | None = None):
        """Reference-identical generator (bench.cpp:63-72); Hkv shrinks K/V heads."""
        kk = 0 if kind == "uniform" else 1
        outs = []
        for tid in tensor_ids:
            h = H if (tid == 0 or Hkv is None) else Hkv
            a = np.empty(B * h * S * d)
            if self.lib.orc_generate(kk, x0, am, p, seed, tid, 0, a.size, a):
                raise ValueError("generate: p must lie in (0,1)")
            outs.append(a.reshape(B, h, S, d))
        return outs

    def generate_resonance(self, seed: int, B: int, H: int, S: int, d: int,
                           qa: float = 70.0, ka: float = 34.0):
        outs = []
        for tid in range(3):
            a = np.empty(B * H * S * d)
            self.lib.orc_generate_resonance(seed, tid, B, H, S, d, qa, ka, a)
            outs.append(a.reshape(B, H, S, d))
        return outs

    # -- metrics ---------------------------------------------------------------
    def rmse(self, x, g) -> float:
        x, g = _f64(x).reshape(-1), _f64(g).reshape(-1)
        r = self.lib.orc_rmse(x, g, x.size)
        if r == -1.0:
            raise ZeroDivisionError("rmse: golden norm is zero")
        return r

    def nan_pct(self, x) -> float:
        x = _f64(x).reshape(-1)
        return self.lib.orc_nan_pct(x, x.size)

    # -- attention -------------------------------------------------------------
    def golden(self, pb: Problem, threads: int = 0) -> np.ndarray:
        o = np.empty(pb.q.shape)
        sh = pb.shape()
        rc = self.lib.orc_golden(C.byref(sh), _f64(pb.q), _f64(pb.k), _f64(pb.v), o, threads)
        if rc:
            raise ValueError(f"golden: rc={rc}")
        return o

    def flash_ref(self, pb: Problem, policy: int = FA_PARTIAL_FP16, m0_zero=False,
                  threads: int = 0) -> np.ndarray:
        a, s, v = POLICY_PRECS[policy]
        o = np.empty(pb.q.shape)
        sh = pb.shape()
        rc = self.lib.orc_flash_ref(C.byref(sh), _f64(pb.q), _f64(pb.k), _f64(pb.v), o,
                                    a, s, v, int(m0_zero), threads)
        if rc:
            raise ValueError(f"flash_ref: rc={rc}")
        return o

    def preprocess_keys(self, k, s2: int, diag: float, off: float, lscale: float = 1.0,
                        p_acc: int = P32, p_store: int = P16, threads: int = 0):
        k = _f64(k)
        B, H, S2, d = k.shape
        out = np.empty_like(k)
        if self.lib.orc_preprocess_keys(k, B, H, S2, d, s2, diag, off, p_acc, p_store,
                                        lscale, out, threads):
            raise ValueError("preprocess_keys: S2 % s2 != 0")
        return out

    def pasa_ref(self, pb: Problem, beta: float = BETA_STAR, policy: int = PASA_FP16,
                 m_prec: int = P16, threads: int = 0) -> np.ndarray:
        a, s, v = POLICY_PRECS[policy]
        d = pb.q.shape[-1]
        diag, off = self.shift_entries(pb.s2, beta, float(np.sqrt(d)), m_prec)
        o = np.empty(pb.q.shape)
        sh = pb.shape()
        rc = self.lib.orc_pasa_ref(C.byref(sh), _f64(pb.q), _f64(pb.k), _f64(pb.v), o, beta,
                                   diag, off, a, s, v, threads)
        if rc:
            raise ValueError(f"pasa_ref: rc={rc}")
        return o

    def model_inflation(self, vmax: float, S2: int, lscale: float = LOG2E) -> float:
        return self.lib.orc_model_inflation(vmax, S2, lscale)

    def model_pasa(self, pb: Problem, beta: float = BETA_STAR, lscale: float = LOG2E / 2,
                   tc_mode: int = 1, c0: float = -1.0, threads: int = 0,
                   xscale: float | None = None, rowsum: int | None = None) -> np.ndarray:
        """The kernel's numerics: scores stored in units of lscale
        (log2(e)/2 on the device), exp argument xscale*fl16(S' - c_j) with
        xscale = log2(e)/lscale rounded to the power of two (2 by default).
        ``rowsum``: the pseudo-average's row sum -- 1: tensor core, q.hi and q.lo added in
        FP32 (the kernel at d = 64); 2: one FP32 accumulator over [q|q].[hi|lo] (d = 128);
        0: the CUDA-core FP32 chains (d = 128 default build); None: the kernel's choice."""
        d = pb.q.shape[-1]
        if rowsum is None:  # d = 64: per-block tensor-core sums; d = 128: CUDA cores
            rowsum = 1 if 128 + d + 16 <= 256 else 0
        diag, off = self.shift_entries(pb.s2, beta, float(np.sqrt(d)), P16)
        if xscale is None:
            xscale = 2.0 if lscale == LOG2E / 2 else 1.0
        mp = ModelParams(beta, diag, off, lscale, tc_mode, c0, xscale, rowsum)
        o = np.empty(pb.q.shape)
        sh = pb.shape()
        rc = self.lib.orc_model_pasa(C.byref(sh), _f64(pb.q), _f64(pb.k), _f64(pb.v), o,
                                     C.byref(mp), threads)
        if rc:
            raise ValueError(f"model_pasa: rc={rc}")
        return o


    def model_fa16(self, pb: Problem, tc_mode: int = 1, threads: int = 0) -> np.ndarray:
        """The kernel's beta == 0 mode: naive FP16 FlashAttention (see pasa_oracle.c)."""
        o = np.empty(pb.q.shape)
        sh = pb.shape()
        rc = self.lib.orc_model_fa16(C.byref(sh), _f64(pb.q), _f64(pb.k), _f64(pb.v), o, tc_mode,
                                     threads)
        if rc:
            raise ValueError(f"model_fa16: rc={rc}")
        return o


class RefLib:
    """The reference itself through oracle/ref_capi.cpp (equal Q/K heads only)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        sz = C.c_size_t
        L.ref_pasa_attention.argtypes = [sz] * 7 + [_dp, _dp, _dp, C.c_double, C.c_int,
                                                    C.c_int, C.c_int, _dp, C.c_void_p]
        L.ref_flash_attention.argtypes = [sz] * 7 + [_dp, _dp, _dp, C.c_int, C.c_int,
                                                     C.c_int, _dp, C.c_void_p]
        L.ref_golden.argtypes = [sz] * 7 + [_dp, _dp, _dp, C.c_int, _dp]
        L.ref_generate.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                   sz, sz, sz, sz, _dp, _dp, _dp]
        L.ref_rmse.restype = C.c_double
        L.ref_rmse.argtypes = [sz, _dp, _dp]
        L.ref_nan_stats.restype = C.c_double
        L.ref_report.restype = C.c_long
        L.ref_report.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p),
                                 C.POINTER(C.c_char_p), _dp,
                                 np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS"), C.c_int,
                                 C.c_char_p, sz]
        L.ref_nan_stats.argtypes = [sz, _dp]
        L.ref_shift_entries.argtypes = [sz, C.c_double, C.c_double, C.c_int,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_preprocess_keys.argtypes = [sz, sz, _dp, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_optimal_beta.argtypes = [C.c_double, sz, C.c_double, C.POINTER(C.c_double),
                                       C.POINTER(C.c_size_t), C.POINTER(C.c_double)]
        L.ref_invariance.argtypes = [C.c_double, sz, _dp]

    def _check(self, rc):
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())

    @staticmethod
    def _dims(pb: Problem):
        B, H, S1, d = pb.q.shape
        S2 = pb.k.shape[2]
        if pb.k.shape[1] != H:
            raise ValueError("reference requires equal Q/K heads (tensor.cpp:24-26)")
        return B, H, S1, S2, d, pb.s1, pb.s2

    DIAG_FIELDS = ("store_finite_min", "store_finite_max", "store_pos_inf", "store_neg_inf",
                   "store_nan", "out_nonfinite", "out_total")

    def _diag(self, want):
        return np.zeros(7) if want else None

    def pasa(self, pb: Problem, beta: float = BETA_STAR, policy: int = PASA_FP16,
             m_prec: int = P16, threads: int = 0, diag: bool = False):
        """The reference's pasa_attention; with diag=True returns (O, RunDiagnostics dict)."""
        o = np.empty(pb.q.shape)
        dg = self._diag(diag)
        self._check(self.lib.ref_pasa_attention(*self._dims(pb), _f64(pb.q), _f64(pb.k),
                                                _f64(pb.v), beta, m_prec, policy, threads, o,
                                                dg.ctypes.data if diag else None))
        return (o, dict(zip(self.DIAG_FIELDS, dg))) if diag else o

    def flash(self, pb: Problem, policy: int = FA_PARTIAL_FP16, m0_zero=False, threads: int = 0,
              diag: bool = False):
        o = np.empty(pb.q.shape)
        dg = self._diag(diag)
        self._check(self.lib.ref_flash_attention(*self._dims(pb), _f64(pb.q), _f64(pb.k),
                                                 _f64(pb.v), policy, int(m0_zero), threads, o,
                                                 dg.ctypes.data if diag else None))
        return (o, dict(zip(self.DIAG_FIELDS, dg))) if diag else o

    def golden(self, pb: Problem, threads: int = 0):
        o = np.empty(pb.q.shape)
        self._check(self.lib.ref_golden(*self._dims(pb), _f64(pb.q), _f64(pb.k), _f64(pb.v),
                                        threads, o))
        return o

    def generate(self, kind: str, x0: float, am: float, seed: int, B: int, H: int, S: int,
                 d: int, p: float = 0.001):
        q, k, v = (np.empty((B, H, S, d)) for _ in range(3))
        self._check(self.lib.ref_generate(0 if kind == "uniform" else 1, x0, am, p, seed,
                                          B, H, S, d, q, k, v))
        return q, k, v

    def rmse(self, x, g):
        x, g = _f64(x).reshape(-1), _f64(g).reshape(-1)
        return self.lib.ref_rmse(x.size, x, g)

    def report(self, rows, json: bool = False) -> str:
        """The reference's report_csv / report_json_rows text for RunReport-like rows."""
        n = len(rows)
        enc = lambda xs: (C.c_char_p * max(n, 1))(*[x.encode() for x in xs])  # noqa: E731
        nums = np.zeros((max(n, 1), 14))
        ints = np.zeros((max(n, 1), 6), dtype=np.int64)
        for i, r in enumerate(rows):
            nums[i, :11] = [r.x0, r.am, r.p, r.beta, r.rmse, r.nan_pct, r.s_min_before,
                            r.s_max_before, r.s_min_after, r.s_max_after, r.wall_s]
            ints[i] = [r.seed, r.batch, r.heads, r.seq, r.dim, int(r.has_ranges)]
        cap = 4096 + 1024 * n
        buf = C.create_string_buffer(cap)
        m = self.lib.ref_report(n, enc([r.policy for r in rows]), enc([r.kind for r in rows]),
                                enc([r.error for r in rows]), nums, ints, int(json), buf, cap)
        if m < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return buf.value.decode()

    def nan_stats(self, x):
        x = _f64(x).reshape(-1)
        return self.lib.ref_nan_stats(x.size, x)

    def shift_entries(self, s2, beta, alpha, prec=P16):
        d, o = C.c_double(), C.c_double()
        self._check(self.lib.ref_shift_entries(s2, beta, alpha, prec, C.byref(d), C.byref(o)))
        return d.value, o.value

    def preprocess_block(self, kblock, beta, alpha, policy=PASA_FP16):
        kblock = _f64(kblock)
        s2, d = kblock.shape
        out = np.empty((d, s2))
        self._check(self.lib.ref_preprocess_keys(s2, d, kblock, beta, alpha, policy, out))
        return out

    def optimal_beta(self, beta0, n=128, tol=1e-8):
        b, it, e = C.c_double(), C.c_size_t(), C.c_double()
        self._check(self.lib.ref_optimal_beta(beta0, n, tol, C.byref(b), C.byref(it), C.byref(e)))
        return b.value, it.value, e.value

    def invariance(self, beta, n):
        out = np.zeros(5)
        self._check(self.lib.ref_invariance(beta, n, out))
        return dict(zip(["a", "b", "inva_ideal", "inva_actual", "rel_err"], out))


def ref_available() -> bool:
    return os.path.exists(REF_SO)
