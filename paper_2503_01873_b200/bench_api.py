"""The reference's benchmark surface on the B200.

Mirrors ``pasa/bench.hpp`` (names, fields, error behaviour, report schema):

=====================================  ==============================================
reference                              here
=====================================  ==============================================
``DistKind``, ``DistributionSpec``     same                       (bench.hpp:24-36)
``generate``                           same, on the device        (bench.cpp:28-72)
``golden_attention``                   same, FP64 on the device   (attention.cpp:66-90)
``rmse``, ``nan_stats``                same, FP64 on the device   (bench.cpp:74-100)
``range_report``, ``RangeReport``      same, FP64 on the device   (bench.cpp:102-168)
``sweep``, ``SweepOptions``,           same                       (bench.cpp:170-247)
``RunReport``
``report_csv``, ``report_json_rows``,  same text                  (bench.cpp:249-331)
``range_csv``
=====================================  ==============================================

Inputs come from the device generator (``pasa_b200_generate``): the uniform
kind is bit-identical to the reference, the hybrid kind agrees except within
an ulp of an FP16 rounding boundary, so a sweep here and the reference's
``sweep`` run on the same tensors.  The golden, RMSE and range reports are
checkers, computed with FP64 cuBLAS/torch on the device (the reference's are
FP64 on the CPU); only the PASA_FP16 and FA_PARTIAL_FP16 policies are
offloaded -- a cell asking for another policy records the error, like the
reference's never-aborting sweep (bench.cpp:228-238).
"""
from __future__ import annotations

import enum
import json
import math
import time
from dataclasses import dataclass, field

import torch

from . import _lib
from .api import (BETA_STAR, AttnOptions, M0Mode, PasaParams, PolicyId, Prec, flash_attention,
                  make_problem, pasa_attention, policy_for)


class ZeroNormError(ValueError):
    """bench.hpp:20-22 (a std::domain_error)."""


class DistKind(enum.IntEnum):
    UNIFORM = 0
    HYBRID = 1

    def __str__(self) -> str:  # to_string(DistKind), bench.cpp:102-104
        return "uniform" if self == DistKind.UNIFORM else "hybrid"


@dataclass
class DistributionSpec:
    """bench.hpp:28-35; ``heads_kv`` (GQA) is an extension (K/V get their own head count)."""

    kind: DistKind = DistKind.UNIFORM
    x0: float = 0.0
    am: float = 0.0
    p: float = 0.001
    seed: int = 0
    batch: int = 1
    heads: int = 1
    seq: int = 128
    dim: int = 64
    heads_kv: int | None = None


@dataclass
class GeneratedInputs:
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def generate_tensor(kind: DistKind, x0: float, am: float, p: float, seed: int, tensor_id: int,
                    shape: tuple[int, ...], device: str | torch.device = "cuda",
                    start: int = 0) -> torch.Tensor:
    """Elements [start, start + numel) of tensor ``tensor_id`` (gen_tensor, bench.cpp:50-56)."""
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError("generate_tensor runs on the device; pass a CUDA device")
    out = torch.empty(shape, dtype=torch.float16, device=device)
    _lib.check(_lib.load().pasa_b200_generate(int(kind), x0, am, p, seed, tensor_id, start,
                                              out.numel(), out.data_ptr(), _stream(device)))
    return out


def generate(spec: DistributionSpec, device: str | torch.device = "cuda") -> GeneratedInputs:
    """bench.cpp:58-72: Q, K, V = tensors 0, 1, 2 of the spec, FP16, on the device."""
    if spec.kind == DistKind.HYBRID and not (0.0 < spec.p < 1.0):
        raise ValueError("generate: p must lie in (0, 1)")
    hkv = spec.heads if spec.heads_kv is None else spec.heads_kv
    shp = lambda h: (spec.batch, h, spec.seq, spec.dim)  # noqa: E731
    q = generate_tensor(spec.kind, spec.x0, spec.am, spec.p, spec.seed, 0, shp(spec.heads), device)
    k = generate_tensor(spec.kind, spec.x0, spec.am, spec.p, spec.seed, 1, shp(hkv), device)
    v = generate_tensor(spec.kind, spec.x0, spec.am, spec.p, spec.seed, 2, shp(hkv), device)
    return GeneratedInputs(q, k, v)


def generate_resonance(seed: int, batch: int, heads: int, seq: int, dim: int, qa: float = 70.0,
                       ka: float = 34.0, device: str | torch.device = "cuda") -> GeneratedInputs:
    """SURVEY.md 8d config 3 (SVD d = 64): Q/K share a head-dim cosine with a 180-degree
    lag, so the pre-scale scores sit near -8e4 (the oracle's orc_generate_resonance)."""
    device = torch.device(device)
    outs = []
    for tid in range(3):
        t = torch.empty((batch, heads, seq, dim), dtype=torch.float16, device=device)
        _lib.check(_lib.load().pasa_b200_generate_resonance(seed, tid, batch, heads, seq, dim, qa,
                                                            ka, t.data_ptr(), _stream(device)))
        outs.append(t)
    return GeneratedInputs(*outs)


# ----------------------------------------------------------------------------- golden + metrics
def golden_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, causal: bool = False,
                     dtype: torch.dtype = torch.float64, max_chunk_bytes: int = 1 << 30,
                     rows: slice | None = None) -> torch.Tensor:
    """attention.cpp:66-90 on the device: S = Q K^T, S /= sqrt(d), row softmax with max
    subtraction, O = P V -- unblocked, in ``dtype`` (FP64 like the reference by default;
    FP32 for the 128K sweeps).  Chunked over query rows so N = 128K fits.  ``rows``
    restricts the query rows (a sampled golden); causal keeps col <= row + S2 - S1."""
    B, Hq, S1, d = q.shape
    S2 = k.shape[2]
    r0, r1 = (0, S1) if rows is None else (rows.start or 0, rows.stop if rows.stop is not None else S1)
    out = torch.empty((B, Hq, r1 - r0, d), dtype=dtype, device=q.device)
    elt = torch.finfo(dtype).bits // 8
    chunk = max(1, min(r1 - r0, max_chunk_bytes // (3 * S2 * elt)))
    old_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for b in range(B):
            for h in range(Hq):
                kh = k[b, h // (Hq // k.shape[1])].to(dtype)
                vh = v[b, h // (Hq // k.shape[1])].to(dtype)
                for i in range(r0, r1, chunk):
                    j = min(r1, i + chunk)
                    s = (q[b, h, i:j].to(dtype) @ kh.T) / math.sqrt(float(d))
                    if causal:  # bottom-right aligned: row r sees keys <= r + S2 - S1
                        ri = torch.arange(i, j, device=q.device)[:, None] + (S2 - S1)
                        cj = torch.arange(S2, device=q.device)[None, :]
                        s.masked_fill_(cj > ri, float("-inf"))
                    s = torch.softmax(s, dim=-1)
                    out[b, h, i - r0:j - r0] = s @ vh
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old_tf32
    return out


def golden_rmse(computed: torch.Tensor, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                causal: bool = False, dtype: torch.dtype = torch.float32,
                max_chunk_bytes: int = 1 << 30) -> float:
    """rmse(computed, golden_attention(q, k, v)) streamed over (b, h, row chunks) so the
    golden is never materialised: full-output RMSE at N = 128K."""
    B, Hq, S1, d = q.shape
    S2 = k.shape[2]
    if not bool(torch.isfinite(computed).all()):
        return math.nan
    elt = torch.finfo(dtype).bits // 8
    chunk = max(1, min(S1, max_chunk_bytes // (3 * S2 * elt)))
    err = nrm = 0.0
    for b in range(B):
        for h in range(Hq):
            for i in range(0, S1, chunk):
                j = min(S1, i + chunk)
                g = golden_attention(q[b:b + 1, h:h + 1], k[b:b + 1, h // (Hq // k.shape[1]):][:, :1],
                                     v[b:b + 1, h // (Hq // k.shape[1]):][:, :1], causal, dtype,
                                     max_chunk_bytes, slice(i, j)).to(torch.float64)
                c = computed[b, h, i:j].to(torch.float64)
                err += float(((c - g[0, 0]) ** 2).sum())
                nrm += float((g * g).sum())
    if nrm == 0.0:
        raise ZeroNormError("rmse: golden norm is zero, metric undefined")
    return math.sqrt(err) / math.sqrt(nrm)


def rmse(computed: torch.Tensor, golden: torch.Tensor) -> float:
    """bench.cpp:74-90: ||c - g||_2 / ||g||_2 in FP64; NaN if ``computed`` holds a NaN/INF;
    ZeroNormError if the golden norm is zero."""
    if computed.shape != golden.shape:
        raise ValueError("rmse: shapes disagree")
    c = computed.to(torch.float64)
    if not bool(torch.isfinite(c).all()):
        return math.nan
    g = golden.to(device=c.device, dtype=torch.float64)
    g2 = float((g * g).sum())
    if g2 == 0.0:
        raise ZeroNormError("rmse: golden norm is zero, metric undefined")
    return math.sqrt(float(((c - g) ** 2).sum())) / math.sqrt(g2)


def nan_stats(t: torch.Tensor) -> float:
    """bench.cpp:92-100: percentage of NaN or INF elements."""
    if t.numel() == 0:
        return 0.0
    return 100.0 * float((~torch.isfinite(t)).sum()) / t.numel()


# ----------------------------------------------------------------------------- range report
@dataclass
class RangeEntry:
    """bench.hpp:53-60."""

    batch: int = 0
    head: int = 0
    k_before_min: float = math.inf
    k_before_max: float = -math.inf
    k_after_min: float = math.inf
    k_after_max: float = -math.inf
    s_before_min: float = math.inf
    s_before_max: float = -math.inf
    s_after_min: float = math.inf
    s_after_max: float = -math.inf


F16_MAX = 65504.0


@dataclass
class RangeReport:
    per_head: list[RangeEntry] = field(default_factory=list)
    total: RangeEntry = field(default_factory=RangeEntry)

    def overflow_predicted(self, alpha: float) -> bool:
        """bench.cpp:102-106."""
        peak = max(abs(self.total.s_before_min), abs(self.total.s_before_max))
        return peak * alpha > F16_MAX


def range_report(q: torch.Tensor, k: torch.Tensor, params: PasaParams, s2: int) -> RangeReport:
    """bench.cpp:108-168 on the device in FP64: ranges of K and K'^T = K_j^T M (FP64
    products of the FP16 M), of S = Q K^T / alpha and of S' = Q K'."""
    B, Hq, S1, d = q.shape
    S2 = k.shape[2]
    m = torch.as_tensor(params.m, dtype=torch.float64, device=q.device)
    rep = RangeReport()
    old_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for b in range(B):
            for h in range(Hq):
                kh = k[b, h // (Hq // k.shape[1])].to(torch.float64)
                qh = q[b, h].to(torch.float64)
                kp = (kh.view(S2 // s2, s2, d).transpose(1, 2) @ m)  # (nkv, d, s2)
                kp = kp.transpose(0, 1).reshape(d, S2)
                e = RangeEntry(b, h)
                e.k_before_min, e.k_before_max = float(kh.min()), float(kh.max())
                e.k_after_min, e.k_after_max = float(kp.min()), float(kp.max())
                s = (qh @ kh.T) / params.alpha
                e.s_before_min, e.s_before_max = float(s.min()), float(s.max())
                ss = qh @ kp
                e.s_after_min, e.s_after_max = float(ss.min()), float(ss.max())
                rep.per_head.append(e)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old_tf32
    t = rep.total
    for e in rep.per_head:
        for f in ("k_before", "k_after", "s_before", "s_after"):
            setattr(t, f + "_min", min(getattr(t, f + "_min"), getattr(e, f + "_min")))
            setattr(t, f + "_max", max(getattr(t, f + "_max"), getattr(e, f + "_max")))
    return rep


# ----------------------------------------------------------------------------- sweep
@dataclass
class SweepOptions:
    """bench.hpp:91-98 (+ causal, an extension)."""

    policies: list[PolicyId] = field(default_factory=list)
    beta: float = BETA_STAR
    s1: int = 128
    s2: int = 128
    diagnose: bool = False
    m0: M0Mode = M0Mode.NEG_INF
    threads: int = 0
    causal: bool = False


@dataclass
class RunReport:
    """bench.hpp:73-89; mirrors the CSV schema exactly."""

    policy: str = ""
    kind: str = ""
    x0: float = 0.0
    am: float = 0.0
    p: float = 0.0
    seed: int = 0
    batch: int = 0
    heads: int = 0
    seq: int = 0
    dim: int = 0
    beta: float = 0.0
    rmse: float = 0.0
    nan_pct: float = 0.0
    has_ranges: bool = False
    s_min_before: float = 0.0
    s_max_before: float = 0.0
    s_min_after: float = 0.0
    s_max_after: float = 0.0
    wall_s: float = 0.0
    error: str = ""


def sweep(specs: list[DistributionSpec], opts: SweepOptions,
          device: str | torch.device = "cuda") -> list[RunReport]:
    """bench.cpp:170-247: per spec, generate once, share the golden, run every policy on
    the identical inputs; a failing cell records its error and never aborts the sweep."""
    device = torch.device(device)
    rows: list[RunReport] = []
    for spec in specs:
        base = RunReport(kind=str(DistKind(spec.kind)), x0=spec.x0, am=spec.am, p=spec.p,
                         seed=spec.seed, batch=spec.batch, heads=spec.heads, seq=spec.seq,
                         dim=spec.dim, beta=opts.beta)
        cell_error = ""
        try:
            gi = generate(spec, device)
            problem = make_problem(gi.q, gi.k, gi.v, opts.s1, opts.s2)
            params = PasaParams.make(opts.s2, opts.beta, problem.alpha, Prec.FP16)
            golden = golden_attention(problem.q, problem.k, problem.v, opts.causal)
            ranges = range_report(problem.q, problem.k, params, opts.s2) if opts.diagnose else None
        except Exception as ex:  # noqa: BLE001 -- the reference catches std::exception
            cell_error = str(ex)
        for pid in opts.policies:
            row = RunReport(**{**base.__dict__, "policy": PolicyId(pid).name})
            if cell_error:
                row.error, row.rmse, row.nan_pct = cell_error, math.nan, math.nan
                rows.append(row)
                continue
            try:
                policy = policy_for(pid)
                aopts = AttnOptions(m0=opts.m0, threads=opts.threads, causal=opts.causal)
                torch.cuda.synchronize(device)
                t0 = time.perf_counter()
                if pid == PolicyId.PASA_FP16:
                    out = pasa_attention(problem, params, policy, aopts)
                else:
                    out = flash_attention(problem, policy, aopts)
                torch.cuda.synchronize(device)
                row.wall_s = time.perf_counter() - t0
                row.nan_pct = nan_stats(out)
                row.rmse = rmse(out, golden)
                if ranges is not None:
                    row.has_ranges = True
                    t = ranges.total
                    row.s_min_before, row.s_max_before = t.s_before_min, t.s_before_max
                    row.s_min_after, row.s_max_after = t.s_after_min, t.s_after_max
            except Exception as ex:  # noqa: BLE001
                row.error, row.rmse = str(ex), math.nan
            rows.append(row)
    return rows


# ----------------------------------------------------------------------------- reports
REPORT_CSV_HEADER = ("policy,kind,x0,Am,p,seed,B,N,S,d,beta,rmse,nan_pct,s_min_before,"
                     "s_max_before,s_min_after,s_max_after,wall_s")  # bench.hpp:105-107


def fmt_double(v: float, spec: str = "%.10g") -> str:
    """bench.cpp:74-80 (fmt_double): printf formatting, "nan" for NaN."""
    if math.isnan(v):
        return "nan"
    return spec % v


def report_csv(rows: list[RunReport]) -> str:
    """bench.cpp:249-277."""
    out = REPORT_CSV_HEADER + "\n"
    for r in rows:
        f = [r.policy, r.kind, fmt_double(r.x0), fmt_double(r.am),
             fmt_double(r.p) if r.kind == "hybrid" else "", str(r.seed), str(r.batch),
             str(r.heads), str(r.seq), str(r.dim), fmt_double(r.beta), fmt_double(r.rmse),
             fmt_double(r.nan_pct)]
        for v in (r.s_min_before, r.s_max_before, r.s_min_after, r.s_max_after):
            f.append(fmt_double(v) if r.has_ranges else "")
        f.append(fmt_double(r.wall_s, "%.4g"))
        out += ",".join(f) + "\n"
    return out


def _num(v: float):
    return None if isinstance(v, float) and (math.isnan(v) or math.isinf(v)) else v


def report_json_rows(rows: list[RunReport]) -> str:
    """bench.cpp:279-316: an array of objects with the CSV's fields (keys sorted, as the
    reference's nlohmann::json object orders them; NaN serialises as null)."""
    arr = []
    for r in rows:
        o = {"policy": r.policy, "kind": r.kind, "x0": r.x0, "Am": r.am,
             "p": r.p if r.kind == "hybrid" else None, "seed": r.seed, "B": r.batch,
             "N": r.heads, "S": r.seq, "d": r.dim, "beta": r.beta, "rmse": _num(r.rmse),
             "nan_pct": _num(r.nan_pct), "wall_s": r.wall_s}
        for key in ("s_min_before", "s_max_before", "s_min_after", "s_max_after"):
            o[key] = _num(getattr(r, key)) if r.has_ranges else None
        if r.error:
            o["error"] = r.error
        arr.append(o)
    return json.dumps(arr, indent=2, sort_keys=True)


def range_csv(report: RangeReport) -> str:
    """bench.cpp:318-331."""
    out = ("batch,head,k_min_before,k_max_before,k_min_after,k_max_after,"
           "s_min_before,s_max_before,s_min_after,s_max_after\n")
    for e in report.per_head:
        vals = (e.k_before_min, e.k_before_max, e.k_after_min, e.k_after_max, e.s_before_min,
                e.s_before_max, e.s_after_min, e.s_after_max)
        out += f"{e.batch},{e.head}," + ",".join(fmt_double(v, "%.7g") for v in vals) + "\n"
    return out


def runs_from_json(text: str) -> list[RunReport]:
    """Inverse of report_json_rows (the CLI's ``report`` subcommand)."""
    rows = []
    for o in json.loads(text):
        has = o.get("s_min_before") is not None
        nan = lambda x: math.nan if x is None else x  # noqa: E731
        rows.append(RunReport(
            policy=o["policy"], kind=o["kind"], x0=o["x0"], am=o["Am"],
            p=o["p"] if o["p"] is not None else 0.0, seed=o["seed"], batch=o["B"],
            heads=o["N"], seq=o["S"], dim=o["d"], beta=o["beta"], rmse=nan(o["rmse"]),
            nan_pct=nan(o["nan_pct"]), has_ranges=has,
            s_min_before=nan(o["s_min_before"]) if has else 0.0,
            s_max_before=nan(o["s_max_before"]) if has else 0.0,
            s_min_after=nan(o["s_min_after"]) if has else 0.0,
            s_max_after=nan(o["s_max_after"]) if has else 0.0,
            wall_s=o["wall_s"], error=o.get("error", "")))
    return rows
