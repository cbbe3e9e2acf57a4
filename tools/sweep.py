"""Throughput + accuracy sweep over the BASELINE.json configurations (tool).

    python tools/sweep.py [--out profiles/r01_sweep.json] [--quick]

For each configuration: fused-kernel TFLOP/s (CUDA events, L2 flushed between
launches), step TFLOP/s (pre-pass + fused), RMSE of sampled rows against a
torch FP32 attention and the non-finite count of the whole output.
Configs (BASELINE.json):
  configs[1] Qwen2-7B attn 28/4 GQA d=128 causal, N in {8K, 16K, 32K}
  configs[2] SVD spatial d=64 (50 x 5 heads, N = 9216) with resonance Q/K
  configs[3] long sweep d=128, H=32 (B=1) N in {4K .. 128K}, non-causal
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_01873_b200 import _lib  # noqa: E402
from paper_2503_01873_b200.api import LOG2E  # noqa: E402

BETA = 0.984497


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        return 1590.0


def gen(kind, B, Hq, Hkv, S, d, dev, seed):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    if kind == "resonance":
        c = torch.arange(d, device=dev, dtype=torch.float32)
        h = torch.arange(Hq, device=dev, dtype=torch.float32)[:, None, None]
        s = torch.arange(S, device=dev, dtype=torch.float32)[None, :, None]
        wave = torch.cos(2 * math.pi * 3 * c / d + 0.3 * h)
        q = 70 * wave + (2 * torch.rand(B, Hq, S, d, device=dev, generator=g) - 1)
        k = -34 * (1 + 0.1 * torch.sin(2 * math.pi * s / 512)) * wave[:Hkv] + (
            2 * torch.rand(B, Hkv, S, d, device=dev, generator=g) - 1)
        v = 2 * torch.rand(B, Hkv, S, d, device=dev, generator=g) - 1
        return q.half(), k.half(), v.half()

    def hybrid(shape):
        core = torch.randn(shape, device=dev, generator=g)
        gate = torch.rand(shape, device=dev, generator=g) < 0.001
        return core + gate * (10.0 * torch.randn(shape, device=dev, generator=g))
    return hybrid((B, Hq, S, d)).half(), hybrid((B, Hkv, S, d)).half(), hybrid((B, Hkv, S, d)).half()


def ref_rows(q, k, v, r0, causal):
    qf, kf, vf = q.float(), k.float(), v.float()
    s = (qf @ kf.transpose(-1, -2)) / math.sqrt(q.shape[-1])
    if causal:
        rows = torch.arange(r0, r0 + q.shape[2], device=q.device)[:, None]
        s = s.masked_fill(torch.arange(k.shape[2], device=q.device)[None] > rows, float("-inf"))
    return torch.softmax(s, -1) @ vf


def run(L, name, kind, B, Hq, Hkv, S, d, causal, iters, dev):
    q, k, v = gen(kind, B, Hq, Hkv, S, d, dev, 7)
    desc = _lib.Desc(B, Hq, Hkv, S, S, d, 128, 128, int(causal), 0, BETA, math.sqrt(d))
    _lib.check(L.pasa_b200_check(C.byref(desc)))
    kp = torch.empty_like(k)
    vp = torch.empty_like(v)
    vmax = torch.zeros(B * Hkv, device=dev)
    o = torch.empty_like(q)
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def launch(ev=None):
        if ev:
            ev[0].record()
        _lib.check(L.pasa_b200_preprocess(C.byref(desc), k.data_ptr(), v.data_ptr(), kp.data_ptr(),
                                          vp.data_ptr(), vmax.data_ptr(), st))
        if ev:
            ev[1].record()
        _lib.check(L.pasa_b200_attention_fwd_prepped(C.byref(desc), q.data_ptr(), kp.data_ptr(),
                                                     vp.data_ptr(), vmax.data_ptr(), o.data_ptr(), st))
        if ev:
            ev[2].record()
    for _ in range(3):
        launch()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(iters)]
    for e in evs:
        flush.zero_()
        launch(e)
    torch.cuda.synchronize()
    step = sum(e[0].elapsed_time(e[2]) for e in evs) / iters
    fwd = sum(e[1].elapsed_time(e[2]) for e in evs) / iters
    flops = 4.0 * B * Hq * S * S * d * (0.5 if causal else 1.0)
    # accuracy: last 256 rows of a few heads vs torch FP32
    g = Hq // Hkv
    r0 = S - 256
    err = nrm = 0.0
    for b in range(min(B, 2)):
        for h in sorted({0, Hq // 2, Hq - 1}):
            ref = ref_rows(q[b:b + 1, h:h + 1, r0:], k[b:b + 1, h // g:h // g + 1],
                           v[b:b + 1, h // g:h // g + 1], r0, causal)
            got = o[b:b + 1, h:h + 1, r0:].float()
            err += float(((got - ref) ** 2).sum())
            nrm += float((ref ** 2).sum())
    res = {"config": name, "B": B, "Hq": Hq, "Hkv": Hkv, "N": S, "d": d, "causal": causal,
           "data": kind, "fwd_ms": fwd, "step_ms": step,
           "fwd_tflops": flops / fwd / 1e9, "step_tflops": flops / step / 1e9,
           "fwd_frac_of_measured_peak": flops / fwd / 1e9 / peak(),
           "rmse_vs_fp32_sampled": math.sqrt(err / nrm),
           "nonfinite": int((~torch.isfinite(o)).sum().item())}
    print(json.dumps(res), flush=True)
    del q, k, v, kp, vp, o, flush
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    L = _lib.load()
    dev = torch.device("cuda:0")
    it = 5 if a.quick else 10
    rows = []
    for S in (8192, 16384, 32768):
        rows.append(run(L, "qwen2-7b (configs[1])", "hybrid", 1, 28, 4, S, 128, True, it, dev))
    rows.append(run(L, "svd-spatial d=64 (configs[2])", "resonance", 50, 5, 5, 9216, 64, False, it, dev))
    for S in (4096, 8192, 16384, 32768, 65536, 131072):
        if a.quick and S > 32768:
            break
        rows.append(run(L, "long sweep H=32 d=128 (configs[3])", "hybrid", 1, 32, 32, S, 128, False,
                        max(2, it // (S // 16384 + 1)), dev))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
