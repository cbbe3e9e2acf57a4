"""Kernel vs CPU model vs reference at growing N on sampled query rows (tool)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Problem
from paper_2503_01873_b200 import pasa_attention_fwd
orc = Oracle()
dev = torch.device("cuda:0")
for S in (1024, 4096, 8192, 16384, 32768):
    for vs in (1.0, 0.05):
        q, k, v = orc.generate("hybrid", 0.0, 10.0, 3, 1, 1, S, 128)
        v = orc.f16(v * vs)
        qs = np.ascontiguousarray(q[:, :, S - 128:])
        pb = Problem(qs, k, v)
        qt, kt, vt = (torch.from_numpy(x).half().to(dev) for x in (qs, k, v))
        o = pasa_attention_fwd(qt, kt, vt).double().cpu().numpy()
        g = orc.golden(pb); m = orc.model_pasa(pb)
        vmax = np.abs(v).max()
        print(f"S={S:6d} vscale={vs}: c0={orc.model_inflation(vmax, S):.0f} kernel={orc.rmse(o, g):.3e} "
              f"model={orc.rmse(m, g):.3e} kernel-vs-model={orc.rmse(o, m):.3e}", flush=True)
