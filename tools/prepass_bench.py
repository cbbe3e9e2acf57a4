"""Time the fused path's pre-pass (pasa_b200_preprocess: max|V| + K', then V') of
library builds against each other (tool).
    python tools/prepass_bench.py [--rounds R] a.so b.so ...
Interleaved round-robin, L2 flushed before every call (as in bench.py), median per
build and shape; prints µs and the algorithmic HBM rate (K, V read twice for V, K', V'
written: 5 B Hkv S2 d 2 bytes)."""
import argparse, ctypes as C, math, os, statistics, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib  # noqa: E402
dev = torch.device("cuda:0")
SHAPES = [("qwen16k", 1, 28, 4, 16384, 128), ("H32-4k", 1, 32, 32, 4096, 128),
          ("H32-16k", 1, 32, 32, 16384, 128), ("svd-d64", 50, 5, 5, 9216, 64)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=7)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    libs = []
    for so in a.libs:
        L = C.CDLL(so if os.path.isabs(so) else os.path.join(ROOT, "paper_2503_01873_b200", "_build", so))
        libs.append(L)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    res = {(i, s[0]): [] for i in range(len(libs)) for s in SHAPES}
    bufs = {}
    for name, B, Hq, Hkv, S, D in SHAPES:
        k = torch.randn(B, Hkv, S, D, device=dev).half() * 8
        v = torch.randn(B, Hkv, S, D, device=dev).half() * 8
        bufs[name] = (_lib.Desc(B, Hq, Hkv, S, S, D, 128, 128, 0, 0, 0.984497, math.sqrt(D)), k, v,
                      torch.empty_like(k), torch.empty_like(v), torch.zeros(B * Hkv, device=dev))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(a.rounds):
        for i, L in enumerate(libs):
            for name, *_ in SHAPES:
                d, k, v, kp, vp, vm = bufs[name]
                for _rep in range(5):
                    flush.zero_()
                    e0.record()
                    assert L.pasa_b200_preprocess(C.byref(d), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                                  C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()),
                                                  C.c_void_p(vm.data_ptr()), C.c_void_p(st)) == 0
                    e1.record()
                    torch.cuda.synchronize()
                    res[(i, name)].append(e0.elapsed_time(e1) * 1e3)
    for i, so in enumerate(a.libs):
        row = []
        for name, B, Hq, Hkv, S, D in SHAPES:
            us = statistics.median(res[(i, name)])
            gbs = 5 * B * Hkv * S * D * 2 / (us * 1e-6) / 1e9
            row.append(f"{name} {us:7.1f} us {gbs:6.0f} GB/s")
        print(f"{os.path.basename(so):14s} " + "  ".join(row))


if __name__ == "__main__":
    main()
