"""Python mirror of the reference PASA operator API, over the C-ABI.

Same names, argument meaning and error behaviour as the reference C++ surface
(/root/reference/proj/include/pasa/*.hpp):

=====================================  =========================================
reference                              here
=====================================  =========================================
``Prec``, ``PolicyId``,                ``Prec``, ``PolicyId``, ``PrecisionPolicy``,
``PrecisionPolicy``, ``policy_for``    ``policy_for``       (precision.hpp:16-56)
``AttnOptions``, ``RunDiagnostics``    same                 (attention.hpp:16-48)
``build_shifting_matrix``              same                 (pasa.hpp:23-28)
``PasaParams::make``                   ``PasaParams.make``  (pasa.hpp:57-64)
``make_problem`` / ``AttentionProblem`` same                (tensor.hpp:41-56)
``preprocess_keys``                    same, batched on device (pasa.hpp:34-36)
``pasa_attention``                     same                 (pasa.hpp:92-99)
=====================================  =========================================

Tensors are torch fp16 tensors in BHSD layout.  CUDA tensors run in place on
their stream; host tensors go through ``pasa_b200_attention_host`` (copy in,
compute, copy out).  There is no CPU fallback: without the CUDA library or a
device every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

BETA_STAR = 0.984497  # optimal beta for s2=128, FP16 (bench.hpp:93)
LOG2E = 1.4426950408889634


class Prec(enum.IntEnum):
    FP64 = 0
    FP32 = 1
    FP16 = 2


class PolicyId(enum.IntEnum):
    GOLDEN_FP64 = 0
    FA_FP32 = 1
    FA_PARTIAL_FP16 = 2
    FA_FULL_FP16 = 3
    PASA_FP16 = 4


@dataclass(frozen=True)
class PrecisionPolicy:
    id: PolicyId = PolicyId.GOLDEN_FP64
    gemm_accum: Prec = Prec.FP64
    gemm_store: Prec = Prec.FP64
    vector_prec: Prec = Prec.FP64


def policy_for(pid: PolicyId) -> PrecisionPolicy:
    """precision.cpp:23-38."""
    table = {
        PolicyId.GOLDEN_FP64: (Prec.FP64, Prec.FP64, Prec.FP64),
        PolicyId.FA_FP32: (Prec.FP32, Prec.FP32, Prec.FP32),
        PolicyId.FA_PARTIAL_FP16: (Prec.FP32, Prec.FP16, Prec.FP16),
        PolicyId.FA_FULL_FP16: (Prec.FP16, Prec.FP16, Prec.FP16),
        PolicyId.PASA_FP16: (Prec.FP32, Prec.FP16, Prec.FP16),
    }
    return PrecisionPolicy(pid, *table[PolicyId(pid)])


class M0Mode(enum.IntEnum):
    NEG_INF = 0
    ZERO = 1


@dataclass
class AttnOptions:
    """attention.hpp:21-25, plus the causal-mask extension (SPEC.md:189 has none)."""

    m0: M0Mode = M0Mode.NEG_INF  # ignored by PASA, as in the reference (pasa.cpp:141-147)
    threads: int = 0             # accepted for API parity; the GPU ignores it
    diagnose: bool = False
    causal: bool = False
    check_finite: bool = True    # make_problem's finiteness rule (tensor.cpp:39-46)


@dataclass
class RunDiagnostics:
    """attention.hpp:30-48: store statistics (the scores the tensor core stored, in the
    reference's units) and output counters, filled by the device; no FP64 side channel."""

    store_finite_min: float = math.inf
    store_finite_max: float = -math.inf
    store_pos_inf: int = 0
    store_neg_inf: int = 0
    store_nan: int = 0
    out_nonfinite: int = 0
    out_total: int = 0
    has_fp64_ranges: bool = False

    @staticmethod
    def from_c(d: "_lib.Diag") -> "RunDiagnostics":
        """From the C-ABI's pasa_b200_diag (device RunDiagnostics, copied to the host)."""
        return RunDiagnostics(float(d.store_finite_min), float(d.store_finite_max),
                              int(d.store_pos_inf), int(d.store_neg_inf), int(d.store_nan),
                              int(d.out_nonfinite), int(d.out_total))

    def merge(self, o: "RunDiagnostics") -> None:
        self.store_finite_min = min(self.store_finite_min, o.store_finite_min)
        self.store_finite_max = max(self.store_finite_max, o.store_finite_max)
        self.store_pos_inf += o.store_pos_inf
        self.store_neg_inf += o.store_neg_inf
        self.store_nan += o.store_nan
        self.out_nonfinite += o.out_nonfinite
        self.out_total += o.out_total
        self.has_fp64_ranges = self.has_fp64_ranges or o.has_fp64_ranges


def _f16_bits_to_float(u: int) -> float:
    return float(np.array([u], dtype=np.uint16).view(np.float16)[0])


def shift_entries(s2: int, beta: float, alpha: float) -> tuple[float, float]:
    """(diag, off) of M at FP16 (pasa.cpp:26-27), computed by the C-ABI."""
    d, o = C.c_uint16(), C.c_uint16()
    _lib.check(_lib.load().pasa_b200_shift_entries(s2, beta, alpha, C.byref(d), C.byref(o)))
    return _f16_bits_to_float(d.value), _f16_bits_to_float(o.value)


class SingularMatrixError(ValueError):
    """pasa.hpp:19-21 (a std::domain_error there)."""


def shifting_matrix_inverse(s: int, lam: float) -> np.ndarray:
    """Theorem 2.1's closed-form inverse of (I - lam J): I + lam / (1 - lam s) J, FP64
    (pasa.cpp:37-51); SingularMatrixError exactly when lam s == 1 (beta == 1)."""
    denom = 1.0 - lam * float(s)
    if denom == 0.0:
        raise SingularMatrixError("shifting matrix is singular: lambda * s == 1 (beta == 1)")
    m = np.full((s, s), lam / denom)
    m[np.diag_indices(s)] += 1.0
    return m


def build_shifting_matrix(s2: int, beta: float, alpha: float, prec: Prec = Prec.FP16) -> np.ndarray:
    """M = I/alpha - beta*J/(alpha*s2), each entry rounded once (pasa.cpp:16-35)."""
    if prec != Prec.FP16:
        n = float(s2)
        diag, off = (1.0 - beta / n) / alpha, -beta / (alpha * n)
        if prec == Prec.FP32:
            diag, off = float(np.float32(diag)), float(np.float32(off))
    else:
        diag, off = shift_entries(s2, beta, alpha)
    m = np.full((s2, s2), off)
    np.fill_diagonal(m, diag)
    return m


@dataclass
class PasaParams:
    """pasa.hpp:57-64; ``m`` is materialised lazily (only its 2 entries matter)."""

    beta: float = 0.0
    alpha: float = 1.0
    s2: int = 0
    prec: Prec = Prec.FP16
    _m: np.ndarray | None = field(default=None, repr=False)

    @staticmethod
    def make(s2: int, beta: float, alpha: float, prec: Prec = Prec.FP16) -> "PasaParams":
        if beta < 0.0 or beta >= 1.0:  # pasa.cpp:98-101
            raise ValueError("pasa params: beta must lie in [0, 1); beta == 1 has no recovery")
        return PasaParams(beta=beta, alpha=alpha, s2=s2, prec=prec)

    @property
    def m(self) -> np.ndarray:
        if self._m is None:
            self._m = build_shifting_matrix(self.s2, self.beta, self.alpha, self.prec)
        return self._m


@dataclass
class AttentionProblem:
    """tensor.hpp:41-51: Q (B,Hq,S1,d), K/V (B,Hkv,S2,d), block sizes, alpha = sqrt(d)."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    s1: int
    s2: int
    alpha: float

    def seq_q(self) -> int:
        return self.q.shape[2]

    def seq_kv(self) -> int:
        return self.k.shape[2]

    def q_blocks(self) -> int:
        return self.seq_q() // self.s1

    def kv_blocks(self) -> int:
        return self.seq_kv() // self.s2


def _as_f16(t) -> torch.Tensor:
    if isinstance(t, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(t))
    if t.dtype != torch.float16:
        t = t.to(torch.float16)
    return t.contiguous()


def make_problem(q, k, v, s1: int, s2: int, check_finite: bool = True) -> AttentionProblem:
    """Validation rules of tensor.cpp:19-55 (GQA: Hkv may divide Hq)."""
    q, k, v = _as_f16(q), _as_f16(k), _as_f16(v)
    if q.dim() != 4 or q.numel() == 0:
        raise ValueError("problem: empty query tensor")
    B, Hq, S1, d = q.shape
    if k.dim() != 4 or k.shape[0] != B or k.shape[3] != d or k.shape[1] == 0 or Hq % k.shape[1]:
        raise ValueError("problem: K shape does not match Q")
    if tuple(v.shape) != tuple(k.shape):
        raise ValueError("problem: V shape does not match K")
    S2 = k.shape[2]
    if s1 == 0 or s2 == 0 or S1 % s1 or S2 % s2:
        raise ValueError(
            f"problem: sequence lengths must be nonzero multiples of the block sizes (S1={S1}, "
            f"s1={s1}, S2={S2}, s2={s2}); ragged inputs are rejected, use truncation explicitly")
    if check_finite:
        for t in (q, k, v):
            if not bool(torch.isfinite(t).all()):
                raise ValueError("problem: input tensors must be finite in the input precision")
    return AttentionProblem(q, k, v, s1, s2, math.sqrt(float(d)))


_LAYOUTS = {"bhsd": 0, "bshd": 1}


def _desc(q: torch.Tensor, k: torch.Tensor, s1: int, s2: int, beta: float, alpha: float,
          causal: bool, layout: str = "bhsd") -> _lib.Desc:
    """``layout`` "bhsd" (the reference's Tensor4D order) or "bshd" (tensors (B, S, H, d))."""
    if layout not in _LAYOUTS:
        raise ValueError(f"layout must be one of {sorted(_LAYOUTS)}")
    if layout == "bshd":
        B, S1, Hq, d = q.shape
        S2, Hkv = k.shape[1], k.shape[2]
    else:
        B, Hq, S1, d = q.shape
        Hkv, S2 = k.shape[1], k.shape[2]
    return _lib.Desc(B, Hq, Hkv, S1, S2, d, s1, s2, int(causal), _LAYOUTS[layout], beta, alpha)


def _check_device_tensors(fn: str, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                          out: torch.Tensor | None) -> None:
    """The C-ABI takes raw fp16 device pointers: reject what it would misread."""
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError(f"{fn} expects CUDA tensors; use pasa_attention for host data")
    for name, t in (("q", q), ("k", k), ("v", v), ("out", out)):
        if t is None:
            continue
        if t.dtype != torch.float16:
            raise ValueError(f"{fn}: {name} must be float16, got {t.dtype}")
        if t.device != q.device:
            raise ValueError(f"{fn}: {name} is on {t.device}, q on {q.device}")
    if out is not None and (tuple(out.shape) != tuple(q.shape) or not out.is_contiguous()):
        raise ValueError(f"{fn}: out must be a contiguous tensor of q's shape {tuple(q.shape)}")


_WS: "OrderedDict[tuple[int, int], torch.Tensor]" = OrderedDict()
_WS_MAX = 8  # cached workspaces (least recently used dropped first)


def workspace_for(desc: _lib.Desc, device: torch.device,
                  stream: "torch.cuda.Stream | None" = None) -> torch.Tensor:
    """The cached K'/V' workspace of (device, stream), grown to the largest request.

    Each stream gets its own buffer, allocated while that stream is current, so torch's
    caching allocator only hands its memory out again in that stream's order: two calls on
    different streams never share a workspace, and a buffer replaced by a larger one cannot
    be reused while a kernel on its stream may still read it.  At most _WS_MAX buffers are
    kept (a dropped one is freed in its stream's order, like any tensor the launches
    recorded on that stream); release_workspaces() drops them all."""
    n = _lib.load().pasa_b200_workspace_size(C.byref(desc))
    idx = device.index if device.index is not None else torch.cuda.current_device()
    s = stream if stream is not None else torch.cuda.current_stream(idx)
    key = (idx, s.cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < n:
        with torch.cuda.device(idx), torch.cuda.stream(s):
            ws = torch.empty(n, dtype=torch.uint8, device=device)
        _WS[key] = ws
    _WS.move_to_end(key)
    while len(_WS) > _WS_MAX:
        _WS.popitem(last=False)
    return ws[:n]


def release_workspaces() -> None:
    """Drop every cached K'/V' workspace (freed in the order of the streams that used them)."""
    _WS.clear()


def _launch_stream(dev: torch.device, stream: "torch.cuda.Stream | None"):
    """(launch stream, current stream).  A launch on another stream first waits for the
    current one, where the inputs (and any contiguous copies made here) were produced."""
    cur = torch.cuda.current_stream(dev)
    s = stream if stream is not None else cur
    if s != cur:
        s.wait_stream(cur)
    return s, cur


def _hold_for(s: "torch.cuda.Stream", cur: "torch.cuda.Stream", *tensors) -> None:
    """Keep tensors allocated on other streams alive until the launch stream is done with
    them (torch's allocator otherwise only tracks their allocation stream)."""
    if s == cur:
        return
    for t in tensors:
        if t is not None:
            t.record_stream(s)


def pasa_attention_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, beta: float = BETA_STAR,
                       causal: bool = False, s1: int = 128, s2: int = 128,
                       out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                       stream: torch.cuda.Stream | None = None,
                       diag: "RunDiagnostics | None" = None, layout: str = "bhsd",
                       q_tiles: tuple[int, int] | None = None) -> torch.Tensor:
    """Device entry point: fp16 CUDA tensors (BHSD, or BSHD with ``layout="bshd"``),
    asynchronous on ``stream`` (default: the current stream; another stream first waits
    for the current one, and everything it reads or writes stays allocated until it is
    done).  ``diag`` (optional) is merged with the device RunDiagnostics of this call (the
    diagnostic kernel instantiation; synchronises the stream).  ``q_tiles=(t0, n)``
    computes only the query rows of 128-row tiles [t0, t0 + n) of every (b, h)
    (pasa_b200_attention_fwd_tiles: bit-identical to those rows of the whole call; the
    other rows of ``out`` are left as they were)."""
    L = _lib.load()
    _check_device_tensors("pasa_attention_fwd", q, k, v, out)
    if workspace is not None and (not workspace.is_cuda or workspace.device != q.device):
        raise ValueError("pasa_attention_fwd: workspace must be on q's device")
    q, k, v = (t if t.is_contiguous() else t.contiguous() for t in (q, k, v))
    desc = _desc(q, k, s1, s2, beta, math.sqrt(float(q.shape[-1])), causal, layout)
    _lib.check(L.pasa_b200_check(C.byref(desc)))
    with torch.cuda.device(q.device):  # the library launches on the current device
        s, cur = _launch_stream(q.device, stream)
        with torch.cuda.stream(s):  # out / workspace / diag are allocated in s's order
            if out is None:
                out = torch.empty_like(q)
            if workspace is None:
                workspace = workspace_for(desc, q.device, s)
            dbuf = None
            if diag is not None:
                dbuf = torch.empty(C.sizeof(_lib.Diag), dtype=torch.uint8, device=q.device)
                _lib.check(L.pasa_b200_diag_reset(dbuf.data_ptr(), s.cuda_stream))
            if q_tiles is not None:
                if diag is not None:
                    raise ValueError("pasa_attention_fwd: diag is not supported with q_tiles")
                _lib.check(L.pasa_b200_attention_fwd_tiles(
                    C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                    workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                    int(q_tiles[0]), int(q_tiles[1]), s.cuda_stream))
            else:
                _lib.check(L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(),
                                                     v.data_ptr(), out.data_ptr(), workspace.data_ptr(),
                                                     workspace.numel() * workspace.element_size(),
                                                     dbuf.data_ptr() if dbuf is not None else None,
                                                     s.cuda_stream))
        _hold_for(s, cur, q, k, v, out, workspace)
    if dbuf is not None:
        s.synchronize()
        host = _lib.Diag.from_buffer_copy(bytes(dbuf.cpu().numpy()))
        diag.merge(RunDiagnostics.from_c(host))
    return out


def flash_fp16_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal: bool = False,
                   s1: int = 128, s2: int = 128, out: torch.Tensor | None = None,
                   stream: torch.cuda.Stream | None = None, layout: str = "bhsd") -> torch.Tensor:
    """The naive FP16 FlashAttention baseline on the same pipeline (FA_PARTIAL_FP16
    semantics of flash_attention, attention.cpp:92-180): scale after the FP16 score
    store, so inputs whose |QK^T| exceeds 65504 produce NaN -- the failure PASA removes.
    Stream semantics as pasa_attention_fwd."""
    L = _lib.load()
    _check_device_tensors("flash_fp16_fwd", q, k, v, out)
    q, k, v = (t if t.is_contiguous() else t.contiguous() for t in (q, k, v))
    desc = _desc(q, k, s1, s2, 0.0, math.sqrt(float(q.shape[-1])), causal, layout)
    _lib.check(L.pasa_b200_check(C.byref(desc)))
    with torch.cuda.device(q.device):
        s, cur = _launch_stream(q.device, stream)
        with torch.cuda.stream(s):
            if out is None:
                out = torch.empty_like(q)
            _lib.check(L.pasa_b200_flash_fp16_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(),
                                                  v.data_ptr(), out.data_ptr(), s.cuda_stream))
        _hold_for(s, cur, q, k, v, out)
    return out


def flash_attention(problem: AttentionProblem, policy: PrecisionPolicy | PolicyId,
                    opts: AttnOptions | None = None,
                    diag: RunDiagnostics | None = None) -> torch.Tensor:
    """attention.hpp:57-60 on the B200: the FA_PARTIAL_FP16 policy only (the
    reference's partial-FP16 FlashAttention); FP64/FP32 policies are CPU-oracle features.
    ``diag`` gets the stored-score statistics and output counters (attention.cpp:125)."""
    opts = opts or AttnOptions()
    pol = policy if isinstance(policy, PrecisionPolicy) else policy_for(policy)
    if (pol.gemm_accum, pol.gemm_store, pol.vector_prec) != (Prec.FP32, Prec.FP16, Prec.FP16):
        raise ValueError(f"flash_attention on B200 implements FA_PARTIAL_FP16 only, got {pol.id.name}")
    if opts.m0 != M0Mode.NEG_INF:
        raise ValueError("flash_attention on B200 implements m0 = -inf only")
    q, k, v = problem.q, problem.k, problem.v
    if not q.is_cuda:
        raise ValueError("flash_attention on B200 expects CUDA tensors")
    if diag is not None:  # beta = 0 through the diagnostic instantiation
        return pasa_attention_fwd(q, k, v, 0.0, opts.causal, problem.s1, problem.s2, diag=diag)
    return flash_fp16_fwd(q, k, v, opts.causal, problem.s1, problem.s2)


def preprocess_keys(k: torch.Tensor, params: PasaParams, lscale: float = 1.0,
                    v: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Batched K'_j = K_j^T M on device (pasa.cpp:53-56, loop :231-240).

    Returns (kp, vmax) with kp in the K-major layout kp[b,h,j*s2+c,t] = K'_j[t][c];
    ``lscale=1`` reproduces the reference's bits."""
    L = _lib.load()
    _check_device_tensors("preprocess_keys", k, k, k if v is None else v, None)
    k = k.contiguous()
    v = v.contiguous() if v is not None else None
    B, H, S2, d = k.shape
    desc = _lib.Desc(B, H, H, S2, S2, d, params.s2, params.s2, 0, 0, params.beta, params.alpha)
    kp = torch.empty_like(k)
    vmax = torch.zeros(B * H, dtype=torch.float32, device=k.device)
    with torch.cuda.device(k.device):
        st = torch.cuda.current_stream(k.device).cuda_stream
        _lib.check(L.pasa_b200_preprocess_keys(C.byref(desc), k.data_ptr(),
                                               v.data_ptr() if v is not None else None,
                                               kp.data_ptr(), vmax.data_ptr(), lscale, st))
    return kp, vmax


def pasa_attention(problem: AttentionProblem, params: PasaParams,
                   policy: PrecisionPolicy | PolicyId = PolicyId.PASA_FP16,
                   opts: AttnOptions | None = None,
                   diag: RunDiagnostics | None = None) -> torch.Tensor:
    """pasa.hpp:95-99 on the B200.  Only the PASA_FP16 policy runs on the device;
    any other policy raises (the FP64/FP32 policies live in the CPU oracle)."""
    opts = opts or AttnOptions()
    pol = policy if isinstance(policy, PrecisionPolicy) else policy_for(policy)
    if params.s2 != problem.s2:
        raise ValueError("pasa: params.s2 does not match the problem")
    if params.alpha != problem.alpha:
        raise ValueError("pasa: params.alpha does not match sqrt(d)")
    if params.beta == 1.0:
        raise ValueError("pasa: beta == 1 has no recovery")
    if params.beta == 0.0:  # degrades to the blocked FP16 attention (pasa.cpp:212-221)
        return flash_attention(problem, pol, opts, diag)
    if pol.id != PolicyId.PASA_FP16:
        raise ValueError(f"pasa_attention on B200 implements PASA_FP16 only, got {pol.id.name}")
    q, k, v = problem.q, problem.k, problem.v
    if q.is_cuda:
        out = pasa_attention_fwd(q, k, v, params.beta, opts.causal, problem.s1, problem.s2,
                                 diag=diag)
    else:
        L = _lib.load()
        desc = _desc(q, k, problem.s1, problem.s2, params.beta, problem.alpha, opts.causal)
        out = torch.empty_like(q)
        qn, kn, vn = (t.contiguous().view(torch.int16) for t in (q, k, v))
        if diag is None:
            _lib.check(L.pasa_b200_attention_host(C.byref(desc), qn.data_ptr(), kn.data_ptr(),
                                                  vn.data_ptr(), out.view(torch.int16).data_ptr()))
        else:
            hd = _lib.Diag()
            _lib.check(L.pasa_b200_attention_host_diag(C.byref(desc), qn.data_ptr(), kn.data_ptr(),
                                                       vn.data_ptr(),
                                                       out.view(torch.int16).data_ptr(),
                                                       C.byref(hd)))
            diag.merge(RunDiagnostics.from_c(hd))
    return out
