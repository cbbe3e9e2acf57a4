"""Interleaved A/B of the packed short-sequence kernel between library builds (tool).
    python tools/packed_ab.py LIB.so [LIB2.so ...] [--B 9216] [--rounds 7]
The SVD temporal shape (B x 5 heads x 25 frames, d = 64) through the public entry point
pasa_b200_attention_fwd (pre-pass fused in the packed kernel); CUDA events, 20 launches per
sample, median over rounds; reports whether outputs are bit-identical to the first library."""
import argparse, ctypes as C, math, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--B", type=int, default=9216)
    ap.add_argument("--N", type=int, default=25)
    ap.add_argument("--rounds", type=int, default=7)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    q = torch.randn(a.B, 5, a.N, 64, device=dev).half()
    k, v = torch.randn_like(q), torch.randn_like(q)
    desc = _lib.Desc(a.B, 5, 5, a.N, a.N, 64, a.N, a.N, 0, 0, 0.984497, 8.0)
    libs = []
    for path in a.libs:
        L = C.CDLL(os.path.abspath(path))
        L.pasa_b200_workspace_size.restype = C.c_size_t
        L.pasa_b200_workspace_size.argtypes = [C.POINTER(_lib.Desc)]
        L.pasa_b200_attention_fwd.argtypes = [C.POINTER(_lib.Desc)] + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p, C.c_void_p]
        ws = torch.empty(L.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)
        libs.append((path, L, ws, torch.empty_like(q)))
    st = torch.cuda.current_stream().cuda_stream

    def run(L, ws, o):
        rc = L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                       ws.data_ptr(), ws.numel(), None, st)
        assert rc == 0, rc

    times = {p: [] for p, *_ in libs}
    for r in range(a.rounds):
        for path, L, ws, o in libs:
            for _ in range(3):
                run(L, ws, o)
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(20):
                run(L, ws, o)
            e1.record()
            torch.cuda.synchronize()
            times[path].append(e0.elapsed_time(e1) / 20)
    base = libs[0][3]
    byts = 4 * q.numel() * 2
    for path, L, ws, o in libs:
        ms = statistics.median(times[path])
        same = "" if torch.equal(o, base) else "  (DIFF)"
        print(f"{os.path.basename(path):28s} {ms * 1e3:8.1f} us  {byts / ms / 1e6:6.0f} GB/s{same}")


if __name__ == "__main__":
    main()
