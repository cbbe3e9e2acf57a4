"""Per-block row state of the fused kernel (PASA_TRACE build) vs a NumPy mirror
of the CPU model for the same row (debugging tool)."""
import ctypes as C, math, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Problem, BETA_STAR
from paper_2503_01873_b200 import _lib
L = _lib.load(os.path.join(ROOT, "paper_2503_01873_b200", "_build", "libpasa_b200_trace.so"))
L.pasa_b200_debug_set_trace.argtypes = [C.c_void_p]
orc = Oracle(); dev = torch.device("cuda:0")
S, ROW = int(sys.argv[1]) if len(sys.argv) > 1 else 32768, 2
q, k, v = orc.generate("hybrid", 0.0, 10.0, 3, 1, 1, S, 128)
qs = np.ascontiguousarray(q[:, :, S - 128:])
qt, kt, vt = (torch.from_numpy(x).half().to(dev) for x in (qs, k, v))
o = torch.empty_like(qt)
d = _lib.Desc(1, 1, 1, 128, S, 128, 128, 128, 0, 0, BETA_STAR, math.sqrt(128.0))
ws = torch.empty(L.pasa_b200_workspace_size(C.byref(d)), dtype=torch.uint8, device=dev)
tr = torch.zeros(4 * 3 * 32 * 10 + 512 * 4, dtype=torch.int64, device=dev)
L.pasa_b200_debug_set_trace(tr.data_ptr())
_lib.check(L.pasa_b200_attention_fwd(C.byref(d), qt.data_ptr(), kt.data_ptr(), vt.data_ptr(), o.data_ptr(), ws.data_ptr(), ws.numel(), None, None))
torch.cuda.synchronize()
st = tr[4 * 3 * 32 * 10:].cpu().numpy().view(np.float32).reshape(512, 8)
# ---- NumPy mirror of orc_model_pasa for one row (float32 scalars, fp16 elements)
f16 = lambda x: np.float16(x).astype(np.float64)
diag, off = orc.shift_entries(128, BETA_STAR, math.sqrt(128.0))
kp = orc.preprocess_keys(k, 128, diag, off, lscale=1.4426950408889634 / 2)[0, 0]   # (S, 128)
qr = qs[0, 0, ROW]
vh = v[0, 0]
vmax = np.abs(v).max(); c0 = orc.model_inflation(vmax, S)
inva = np.float32(BETA_STAR / (1 - BETA_STAR))
def tc_dot_rows(a, B):  # F16 accumulation, RNE per 16-chunk, exact chunk sums
    acc = np.zeros(B.shape[0])
    for c0_ in range(0, a.shape[0], 16):
        acc = (acc + B[:, c0_:c0_ + 16] @ a[c0_:c0_ + 16]).astype(np.float16).astype(np.float64)
    return acc
m = l = fbar = np.float32(0)
print(f"c0={c0} vmax={vmax}")
print(" j   | kernel mloc    model   | kernel mnew   model  | kernel cj model | kernel ep  model | kernel lsum   model  | kernel l  model")
for j in range(S // 128):
    Sp = tc_dot_rows(qr, kp[j * 128:(j + 1) * 128])
    mloc = np.float32(Sp.max())
    ch = [2 * ((c // 2) % 4) + (c % 2) for c in range(128)]
    sacc = np.zeros((2, 8), np.float32)
    for c in range(128): sacc[int(c >= 64), ch[c]] += np.float32(Sp[c])
    sh_ = [((sacc[h, 0] + sacc[h, 1]) + (sacc[h, 2] + sacc[h, 3])) + ((sacc[h, 4] + sacc[h, 5]) + (sacc[h, 6] + sacc[h, 7])) for h in range(2)]
    ssum = np.float32(sh_[0] + sh_[1]); sbar = np.float32(ssum * np.float32(1 / 128))
    jc = j + 1
    fnew = sbar if jc == 1 else np.float32(fbar + np.float32(np.float32(sbar - fbar) * np.float32(1.0 / jc)))
    dmc = np.float32(inva * np.float32(sbar - fnew)); dmp = np.float32(0) if jc == 1 else np.float32(inva * np.float32(fbar - fnew))
    cand = np.float32(mloc + dmc); mprev = np.float32(m + dmp)
    mnew = cand if jc == 1 else max(mprev, cand)
    cj = f16(np.float32(mnew - dmc))
    ep = 0.0 if jc == 1 else f16(2.0 ** float(np.float32(mprev - mnew)))
    P = np.array([f16(2.0 ** f16(x - cj)) for x in Sp])
    lacc = np.zeros((2, 8), np.float32)
    for c in range(128): lacc[int(c >= 64), ch[c]] += np.float32(P[c])
    lsum0 = ((lacc[0, 0] + lacc[0, 1]) + (lacc[0, 2] + lacc[0, 3])) + ((lacc[0, 4] + lacc[0, 5]) + (lacc[0, 6] + lacc[0, 7]))
    l = lsum0 if jc == 1 else np.float32(np.float32(np.float32(ep) * l) + lsum0)
    k_ = st[j]
    bad = abs(k_[3] - mnew) > 1e-3 * max(1, abs(mnew)) or abs(k_[7] - l) > 1e-3 * abs(l) + 1e-12
    if j < 6 or bad or j % 32 == 0:
        print(f"{j:4d} | {k_[0]:10.4f} {mloc:10.4f} | {k_[3]:10.4f} {mnew:10.4f} | {k_[4]:7.3f} {cj:7.3f} | {k_[5]:.4e} {ep:.4e} | {k_[6]:.4e} {lsum0:.4e} | {k_[7]:.4e} {l:.4e} {'<<<' if bad else ''}")
    m, fbar = mnew, fnew
