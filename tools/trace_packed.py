"""Timeline of the packed short-sequence kernel (PASA_TRACE build; profiling tool).
    python -m paper_2503_01873_b200.build --trace && python tools/trace_packed.py [B]
CTA 0, tiles 1..24, in clock64 cycles: the TMA producer (Q/K, V issued), the pre-pass
warpgroup (stage landed, K' written, done), the MMA issuer (S' issued, P ready, PV committed)
and the softmax warpgroup (S' ready, P stored, T ready, T read, O stored)."""
import ctypes as C, os, sys
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
    tr = torch.zeros(2 * 64 * 16, dtype=torch.int64, device=dev)
    for it in range(3):
        L.pasa_b200_debug_set_trace(tr.data_ptr() if it == 2 else None)
        _lib.check(L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             o.data_ptr(), ws.data_ptr(), ws.numel(), None,
                                             torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(2, 64, 16)
    sm, ct = t[0], t[1]
    base = sm[1, 0]
    print("absolute cycles from tile 1's softmax start (k = 1000 cycles)")
    print(" it |   QKiss   Viss | landed  Kdone   prep | S'iss  Prdy  PVcom | S'rdy  Pst  Trdy  Trd  Ost |"
          " load  prep  S'lat  exp  PV  epi | period")
    f = lambda x: f"{(x - base) / 1000:6.2f}"
    for i in range(1, 25):
        period = sm[i + 1, 1] - sm[i, 1]
        print(f"{i:3d} | {f(ct[i,3])} {f(ct[i,4])} | {f(sm[i,6])} {f(ct[i,8])} {f(ct[i,6])} | "
              f"{f(ct[i,0])} {f(ct[i,1])} {f(ct[i,2])} | {f(sm[i,1])} {f(sm[i,2])} {f(sm[i,4])} {f(sm[i,5])} "
              f"{f(sm[i,3])} | {sm[i,6]-ct[i,4]:5d} {ct[i,6]-sm[i,6]:5d} {sm[i,1]-ct[i,0]:5d} "
              f"{sm[i,2]-sm[i,1]:5d} {ct[i,2]-ct[i,1]:4d} {sm[i,3]-sm[i,5]:4d} | {period:5d} | "
              f"prep: K side {ct[i,8]-sm[i,6]:5d} (K landed {sm[i,6]-ct[i,3]:5d} after issue) | V landed "
              f"{ct[i,9]-ct[i,4]:5d} after issue, V side {ct[i,10]-ct[i,9]:5d} c0 {ct[i,11]-ct[i,10]:5d}")


if __name__ == "__main__":
    main()
