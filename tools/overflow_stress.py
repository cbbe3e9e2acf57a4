"""BASELINE configs[4]: the overflow stress grid on B200 and the reference (tool).

    python tools/overflow_stress.py [--out profiles/r01_overflow_stress.json] [--heads 16]

Cells: the paper's mean-bias / amplitude sweeps (Appendix D presets paper-uniform and
paper-hybrid; Appendix E's six overflow cells are among them) at the paper
shape (1, H, 1280, 128), seed 0, inputs from the device generator (the reference's
generate()).  Per cell: the B200 PASA kernel and the B200 naive FP16 FlashAttention
(beta = 0, FA_PARTIAL_FP16) -- RMSE against the FP64 golden and non-finite % -- and the
reference's own pasa_attention (PASA_FP16, oracle/_ref, all host cores) on the identical
FP16 inputs: RMSE(ref, FP64), RMSE(B200, ref).  The reference is test infrastructure here
(the checker), never the thing measured."""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2503_01873_b200 import bench_api as ba  # noqa: E402
from paper_2503_01873_b200 import flash_fp16_fwd, pasa_attention_fwd  # noqa: E402
from paper_2503_01873_b200.__main__ import PRESETS  # noqa: E402

BETA = 0.984497


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "overflow_stress.json"))
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--seq", type=int, default=1280)
    ap.add_argument("--no-ref", action="store_true")
    a = ap.parse_args()
    from oracle.oracle import Problem, RefLib
    ref = None if a.no_ref else RefLib()
    dev = torch.device("cuda:0")
    cells = PRESETS["paper-uniform"] + PRESETS["paper-hybrid"]
    rows = []
    for kind, x0, am in cells:
        dk = ba.DistKind.UNIFORM if kind == "uniform" else ba.DistKind.HYBRID
        gi = ba.generate(ba.DistributionSpec(dk, float(x0), float(am), 0.001, 0, 1, a.heads, a.seq, 128), dev)
        gold = ba.golden_attention(gi.q, gi.k, gi.v, causal=False)
        o = pasa_attention_fwd(gi.q, gi.k, gi.v, BETA)
        of = flash_fp16_fwd(gi.q, gi.k, gi.v)
        row = {"kind": kind, "x0": x0, "am": am, "B": 1, "H": a.heads, "N": a.seq, "d": 128,
               "b200_pasa_rmse_vs_fp64": ba.rmse(o, gold), "b200_pasa_nonfinite_pct": ba.nan_stats(o),
               "b200_fa16_rmse_vs_fp64": ba.rmse(of, gold), "b200_fa16_nonfinite_pct": ba.nan_stats(of)}
        if ref is not None:
            q, k, v = (t.double().cpu().numpy() for t in (gi.q, gi.k, gi.v))
            t0 = time.perf_counter()
            ro = ref.pasa(Problem(q, k, v), BETA)
            row["ref_wall_s"] = time.perf_counter() - t0
            rt = torch.from_numpy(ro)
            g64 = gold.cpu().double()
            row["ref_pasa_rmse_vs_fp64"] = ba.rmse(rt, g64)
            row["ref_pasa_nonfinite_pct"] = ba.nan_stats(rt)
            finite = torch.isfinite(rt).all().item()
            row["b200_vs_ref_rmse"] = ba.rmse(o.cpu().double(), rt) if finite else math.nan
            row["b200_vs_ref_maxabs_rel"] = (float((o.cpu().double() - rt).abs().max() / rt.abs().max())
                                             if finite else math.nan)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del gi, gold, o, of
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
