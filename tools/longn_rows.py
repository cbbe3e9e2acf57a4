"""Per-row kernel-vs-model error at N = 32K, c0 = 7 (tool)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Problem
from paper_2503_01873_b200 import pasa_attention_fwd
orc = Oracle(); dev = torch.device("cuda:0")
S = 32768
q, k, v = orc.generate("hybrid", 0.0, 10.0, 3, 1, 1, S, 128)
qs = np.ascontiguousarray(q[:, :, S - 128:])
pb = Problem(qs, k, v)
qt, kt, vt = (torch.from_numpy(x).half().to(dev) for x in (qs, k, v))
o = pasa_attention_fwd(qt, kt, vt).double().cpu().numpy()[0, 0]
g = orc.golden(pb)[0, 0]; m = orc.model_pasa(pb)[0, 0]
ek = np.sqrt(((o - g) ** 2).sum(1) / (g ** 2).sum(1))
em = np.sqrt(((m - g) ** 2).sum(1) / (g ** 2).sum(1))
ratio = (np.abs(o).sum(1) / np.abs(g).sum(1))
print("rows kernel err: min/median/max", ek.min(), np.median(ek), ek.max())
print("rows model  err: min/median/max", em.min(), np.median(em), em.max())
print("kernel/gold magnitude ratio: min/median/max", ratio.min(), np.median(ratio), ratio.max())
mr = (np.abs(m).sum(1) / np.abs(g).sum(1)); print("model/gold magnitude ratio", mr.min(), np.median(mr), mr.max())
worst = np.argsort(-ek)[:5]
print("worst rows", worst, ek[worst], em[worst])
# fit o ~ a * g per row
a = (o * g).sum(1) / (g * g).sum(1)
print("kernel scale factor vs gold per row: min/median/max", a.min(), np.median(a), a.max())
