"""How does the tcgen05 F16 accumulator round?  Compare the tensor core's
F16-accumulated A.B^T (K = 128, 8 MMAs of K = 16) against CPU models:
RNE / truncation after every K=16 chunk, and FP32 then one RNE (tool)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = C.CDLL(os.path.join(ROOT, "tests", "cuda", "_build", "libumma_probe.so"))
lib.probe_umma.argtypes = [C.c_void_p] * 4 + [C.c_int] * 3
dev = torch.device("cuda:0")


def f16(x):
    return np.asarray(x, np.float64).astype(np.float16).astype(np.float64)


def trunc16(x):
    h = np.asarray(x, np.float64).astype(np.float16)  # RNE
    hv = h.astype(np.float64)
    # step toward zero if RNE rounded away from zero
    away = np.abs(hv) > np.abs(x)
    nxt = np.nextafter(h, np.float16(0)).astype(np.float64)
    return np.where(away, nxt, hv)


for trial, (scale, pos) in enumerate([(1.0, False), (1.0, True), (8.0, True)]):
    torch.manual_seed(trial)
    a = torch.randn(128, 128, device=dev) * scale
    b = torch.randn(128, 128, device=dev)
    if pos:
        a = a.abs()
        b = b.abs()
    a, b = a.half(), b.half()
    out = torch.zeros(128, 128, device=dev)
    assert lib.probe_umma(a.data_ptr(), b.data_ptr(), None, out.data_ptr(), 128, 0, 0) == 0
    torch.cuda.synchronize()
    got = out.cpu().double().numpy()
    A = a.cpu().double().numpy()
    B = b.cpu().double().numpy()
    prods = A[:, None, :] * B[None, :, :]  # (128, 128, K) exact
    exact = prods.sum(-1)
    models = {}
    acc_r = np.zeros((128, 128))
    acc_t = np.zeros((128, 128))
    for c in range(8):
        chunk = prods[:, :, 16 * c:16 * c + 16].sum(-1)
        acc_r = f16(acc_r + chunk)
        acc_t = trunc16(acc_t + chunk)
    models["rne_per_chunk"] = acc_r
    models["trunc_per_chunk"] = acc_t
    models["fp32_then_rne"] = f16(exact)
    print(f"trial {trial} scale {scale} positive {pos}: mean(got-exact)={np.mean(got - exact):+.3e}")
    for k, m in models.items():
        print(f"   {k:16s} match {np.mean(m == got) * 100:6.2f}%  mean(model-exact) {np.mean(m - exact):+.3e}")
