"""Timeline of the packed short-sequence kernel (PASA_TRACE build; profiling tool).
    python -m paper_2503_01873_b200.build --trace && python tools/trace_packed.py [B]
CTA 0, first tiles: softmax (wait S', exp + P store, next tile's pre-pass, wait T, read T,
epilogue) and MMA issuer (S' issued, P ready, PV issued) in clock64 cycles."""
import ctypes as C, math, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 9216
    L = _lib.load(os.path.join(ROOT, "paper_2503_01873_b200", "_build", "libpasa_b200_trace.so"))
    L.pasa_b200_debug_set_trace.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    q = torch.randn(B, 5, 25, 64, device=dev).half()
    k, v = torch.randn_like(q), torch.randn_like(q)
    desc = _lib.Desc(B, 5, 5, 25, 25, 64, 25, 25, 0, 0, 0.984497, 8.0)
    ws = torch.empty(L.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)
    o = torch.empty_like(q)
    tr = torch.zeros(2 * 64 * 8, dtype=torch.int64, device=dev)
    for it in range(3):
        L.pasa_b200_debug_set_trace(tr.data_ptr() if it == 2 else None)
        _lib.check(L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             o.data_ptr(), ws.data_ptr(), ws.numel(), None,
                                             torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(2, 64, 8)
    base = t[t > 0].min()
    print(" it | sm: waitS  exp+P  prep  waitT  ldT   epi | mma: S'->Pready  Pready->PVdone | period |"
          " prep(it+1): in_full wait, K/V pass, V scale + c0")
    for i in range(1, 20):
        a, m = t[0, i] - base, t[1, i] - base
        nxt = t[0, i + 1, 0] - base
        print(f"{i:3d} | {a[1]-a[0]:6d} {a[2]-a[1]:6d} {a[3]-a[2]:6d} {a[4]-a[3]:6d} {a[5]-a[4]:5d} "
              f"{nxt - a[5]:5d} | {m[1]-m[0]:8d} {m[2]-m[1]:8d} | {nxt - a[0]:6d} | "
              f"{t[0, i + 1, 6] - t[0, i, 2]:6d} {t[0, i + 1, 7] - t[0, i + 1, 6]:6d} {t[0, i, 3] - t[0, i + 1, 7]:6d}")


if __name__ == "__main__":
    main()
