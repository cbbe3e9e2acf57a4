"""PCIe bound of the host entry point (tool).
    python tools/pcie_probe.py [--seq 16384]
Times, with pinned host buffers of the bench workload's sizes (Qwen2-7B attention,
28/4 heads, d = 128): the H2D copy of Q, K, V alone, the D2H copy of O alone, both on
two streams at once, and pasa_b200_attention_host -- so the e2e number can be read
against the copy-only time it cannot beat."""
import argparse, ctypes as C, math, os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    S, HQ, HKV, D = a.seq, 28, 4, 128
    dev = torch.device("cuda:0")
    qh = torch.randn(1, HQ, S, D).half().pin_memory()
    kh = torch.randn(1, HKV, S, D).half().pin_memory()
    vh = torch.randn(1, HKV, S, D).half().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    qd, kd, vd, od = (torch.empty(x.shape, dtype=x.dtype, device=dev) for x in (qh, kh, vh, oh))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    bin_, bout = (qh.numel() + kh.numel() + vh.numel()) * 2, oh.numel() * 2

    def h2d():
        with torch.cuda.stream(s1):
            qd.copy_(qh, non_blocking=True); kd.copy_(kh, non_blocking=True); vd.copy_(vh, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            oh.copy_(od, non_blocking=True)

    def t(fn):
        best = 1e9
        for _ in range(a.reps):
            torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best
    def chunked():  # the host pipeline's copy pattern without compute: per head, 4.2 MB
        with torch.cuda.stream(s1):
            for hk in range(HKV):
                kd[:, hk].copy_(kh[:, hk], non_blocking=True); vd[:, hk].copy_(vh[:, hk], non_blocking=True)
                for g in range(HQ // HKV):
                    qd[:, hk * (HQ // HKV) + g].copy_(qh[:, hk * (HQ // HKV) + g], non_blocking=True)
        with torch.cuda.stream(s2):
            for hq in range(HQ):
                oh[:, hq].copy_(od[:, hq], non_blocking=True)
    sin = [torch.cuda.Stream() for _ in range(3)]
    sout = [torch.cuda.Stream() for _ in range(2)]

    def chunked_multi(n_in, n_out):  # the same chunks spread round-robin over several streams
        c = 0
        for hk in range(HKV):
            for src, dst in [(kh[:, hk], kd[:, hk]), (vh[:, hk], vd[:, hk])] + \
                    [(qh[:, hk * (HQ // HKV) + g], qd[:, hk * (HQ // HKV) + g]) for g in range(HQ // HKV)]:
                with torch.cuda.stream(sin[c % n_in]):
                    dst.copy_(src, non_blocking=True)
                c += 1
        for hq in range(HQ):
            with torch.cuda.stream(sout[hq % n_out]):
                oh[:, hq].copy_(od[:, hq], non_blocking=True)
    th, td, tb, tc = t(h2d), t(d2h), t(lambda: (h2d(), d2h())), t(chunked)
    for n_in, n_out in [(1, 1), (2, 1), (2, 2), (3, 2)]:
        tm = t(lambda: chunked_multi(n_in, n_out))
        print(f"chunked over {n_in} H2D + {n_out} D2H streams: {tm*1e3:.3f} ms")
    L = _lib.load()
    desc = _lib.Desc(1, HQ, HKV, S, S, D, 128, 128, 1, 0, 0.984497, math.sqrt(D))
    te = t(lambda: _lib.check(L.pasa_b200_attention_host(C.byref(desc), qh.data_ptr(), kh.data_ptr(),
                                                          vh.data_ptr(), oh.data_ptr())))
    fl = 4.0 * HQ * S * S * D * 0.5
    print(f"H2D {bin_/1e6:.0f} MB: {th*1e3:.3f} ms = {bin_/th/1e9:.1f} GB/s")
    print(f"D2H {bout/1e6:.0f} MB: {td*1e3:.3f} ms = {bout/td/1e9:.1f} GB/s")
    print(f"both at once: {tb*1e3:.3f} ms (H2D {bin_/tb/1e9:.1f} GB/s effective)")
    print(f"both at once in per-head chunks (no compute): {tc*1e3:.3f} ms")
    print(f"pasa_b200_attention_host: {te*1e3:.3f} ms = {fl/te/1e12:.1f} TFLOP/s; copy-only bound "
          f"{fl/tb/1e12:.1f} TFLOP/s; e2e / bound = {tb/te:.2f}")


if __name__ == "__main__":
    main()
