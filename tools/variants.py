"""Time variant builds of the fused kernel on the bench workload (tool).
    python tools/variants.py libvar_a.so libvar_b.so ..."""
import ctypes as C, math, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib
dev = torch.device("cuda:0")
def run(so, B, Hq, Hkv, S, D, causal, iters=10):
    L = C.CDLL(os.path.join(ROOT, "paper_2503_01873_b200", "_build", so))
    L.pasa_b200_preprocess.argtypes = [C.POINTER(_lib.Desc)] + [C.c_void_p] * 6
    L.pasa_b200_attention_fwd_prepped.argtypes = [C.POINTER(_lib.Desc)] + [C.c_void_p] * 6
    g = torch.Generator(device=dev); g.manual_seed(0)
    q = torch.randn(B, Hq, S, D, device=dev, generator=g).half()
    k = torch.randn(B, Hkv, S, D, device=dev, generator=g).half()
    v = torch.randn(B, Hkv, S, D, device=dev, generator=g).half()
    kp, vp, o = torch.empty_like(k), torch.empty_like(v), torch.empty_like(q)
    vmax = torch.zeros(B * Hkv, device=dev)
    d = _lib.Desc(B, Hq, Hkv, S, S, D, 128, 128, int(causal), 0, 0.984497, math.sqrt(D))
    st = torch.cuda.current_stream().cuda_stream
    assert L.pasa_b200_preprocess(C.byref(d), k.data_ptr(), v.data_ptr(), kp.data_ptr(), vp.data_ptr(), vmax.data_ptr(), st) == 0
    ts = []
    for i in range(iters + 3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.pasa_b200_attention_fwd_prepped(C.byref(d), q.data_ptr(), kp.data_ptr(), vp.data_ptr(), vmax.data_ptr(), o.data_ptr(), st) == 0
        e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    fl = 4.0 * B * Hq * S * S * D * (0.5 if causal else 1.0)
    return fl / statistics.median(ts) / 1e9
for so in sys.argv[1:]:
    a = run(so, 1, 28, 4, 16384, 128, True)
    b = run(so, 1, 32, 32, 16384, 128, False)
    c = run(so, 8, 8, 8, 8192, 64, False)
    print(f"{so:28s} qwen16k-causal {a:7.1f}  H32-16k {b:7.1f}  d64-8k {c:7.1f}", flush=True)
