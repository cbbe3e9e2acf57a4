"""Throughput + accuracy sweep over the BASELINE.json configurations (tool).

    python tools/sweep.py [--out gpurun_out/sweep.json] [--quick]

For each configuration: fused-kernel TFLOP/s (CUDA events, L2 flushed between
launches), step TFLOP/s (pre-pass + fused), RMSE of the WHOLE output against the
device FP32 golden (bench_api.golden_rmse, streamed), RMSE of sampled rows against
the FP64 golden, and the non-finite count.  Inputs come from the device
generators, identical to the reference's generate().
Configs (BASELINE.json):
  configs[1] Qwen2-7B attn 28/4 GQA d=128 causal, N in {8K, 16K, 32K} (uniform(30, 0.5), the
             bench's headline data)
  configs[2] SVD spatial d=64 (50 x 5 heads, N = 9216) and temporal (9216 x 5 heads,
             N = 25 frames, the packed kernel) with resonance Q/K
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
from paper_2503_01873_b200 import bench_api as ba  # noqa: E402
from bench import ClockSampler  # noqa: E402

BETA = 0.984497


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
    except Exception:
        return 1590.0


def gen(kind, B, Hq, Hkv, S, d, dev, seed):
    """Reference-identical inputs from the device generators (bench.cpp:28-72)."""
    if kind == "resonance":
        gi = ba.generate_resonance(seed, B, Hq, S, d, device=dev)
        return gi.q, gi.k[:, :Hkv].contiguous(), gi.v[:, :Hkv].contiguous()
    if kind == "uniform30":  # Appendix E cell 1, the bench's headline data
        gi = ba.generate(ba.DistributionSpec(ba.DistKind.UNIFORM, 30.0, 0.5, 0.001, seed, B, Hq, S, d,
                                             Hkv), dev)
        return gi.q, gi.k, gi.v
    gi = ba.generate(ba.DistributionSpec(ba.DistKind.HYBRID, 0.0, 10.0, 0.001, seed, B, Hq, S, d,
                                         Hkv), dev)
    return gi.q, gi.k, gi.v


def run(L, name, kind, B, Hq, Hkv, S, d, causal, iters, dev, full_rmse=True):
    q, k, v = gen(kind, B, Hq, Hkv, S, d, dev, 7)
    sb = min(128, S)  # short sequences (one KV block) run on the packed kernel
    desc = _lib.Desc(B, Hq, Hkv, S, S, d, sb, sb, int(causal), 0, BETA, math.sqrt(d))
    _lib.check(L.pasa_b200_check(C.byref(desc)))
    kp = torch.empty_like(k)
    vp = torch.empty_like(v)
    vmax = torch.zeros(B * Hkv, device=dev)
    o = torch.empty_like(q)
    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    packed = S <= 64 and not causal and Hq == Hkv  # one KV block: the packed kernel
    ws = torch.empty(L.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)

    def launch(ev=None):
        if packed:  # the public entry point: pre-pass fused into the packed kernel
            if ev:
                ev[0].record()
                ev[1].record()
            _lib.check(L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                 o.data_ptr(), ws.data_ptr(), ws.numel(), None, st))
            if ev:
                ev[2].record()
            return
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
    torch.cuda.synchronize()
    with ClockSampler(dev.index or 0) as cs:  # nvidia-smi during the timed launches
        for e in evs:
            flush.zero_()
            launch(e)
        torch.cuda.synchronize()
    step = sum(e[0].elapsed_time(e[2]) for e in evs) / iters
    fwd = sum(e[1].elapsed_time(e[2]) for e in evs) / iters
    flops = 4.0 * B * Hq * S * S * d * (0.5 if causal else 1.0)
    # accuracy: every row vs the device FP32 golden (streamed), and the last 256 rows of a
    # few heads vs the FP64 golden (the reference's golden_attention precision)
    full = ba.golden_rmse(o, q, k, v, causal, torch.float32) if full_rmse else None
    err = nrm = 0.0
    r0 = max(0, S - 256)
    for b in range(min(B, 2)):
        for h in sorted({0, Hq // 2, Hq - 1}):
            g = ba.golden_attention(q[b:b + 1, h:h + 1], k[b:b + 1, h // (Hq // Hkv):][:, :1],
                                    v[b:b + 1, h // (Hq // Hkv):][:, :1], causal,
                                    rows=slice(r0, S))
            got = o[b:b + 1, h:h + 1, r0:].double()
            err += float(((got - g) ** 2).sum())
            nrm += float((g ** 2).sum())
    res = {"config": name, "B": B, "Hq": Hq, "Hkv": Hkv, "N": S, "d": d, "causal": causal,
           "data": kind, "fwd_ms": fwd, "step_ms": step,
           "fwd_tflops": flops / fwd / 1e9, "step_tflops": flops / step / 1e9,
           "fwd_frac_of_measured_peak": flops / fwd / 1e9 / peak(),
           "rmse_vs_fp32_full": full, "rmse_vs_fp64_sampled": math.sqrt(err / nrm),
           "nonfinite": int((~torch.isfinite(o)).sum().item()), "clocks": cs.summary()}
    print(json.dumps(res), flush=True)
    del q, k, v, kp, vp, o, flush, ws
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="", help="comma list of row groups: qwen,svd,long (default all)")
    a = ap.parse_args()
    L = _lib.load()
    dev = torch.device("cuda:0")
    it = 5 if a.quick else 10
    rows = []
    only = set(a.only.split(",")) if a.only else {"qwen", "svd", "long"}
    for S in ((8192, 16384, 32768) if "qwen" in only else ()):
        rows.append(run(L, "qwen2-7b (configs[1])", "uniform30", 1, 28, 4, S, 128, True, it, dev))
    if "svd" in only:
        rows.append(run(L, "svd-spatial d=64 (configs[2])", "resonance", 50, 5, 5, 9216, 64, False, it, dev))
        rows.append(run(L, "svd-temporal d=64 (configs[2])", "resonance", 9216, 5, 5, 25, 64, False, it, dev))
    for S in ((4096, 8192, 16384, 32768, 65536, 131072) if "long" in only else ()):
        if a.quick and S > 32768:
            break
        rows.append(run(L, "long sweep H=32 d=128 (configs[3])", "hybrid", 1, 32, 32, S, 128, False,
                        max(2, it // (S // 16384 + 1)), dev))
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
