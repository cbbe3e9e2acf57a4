"""Run the fused forward once on one BASELINE shape, for an ncu capture (tool).
    python tools/ncu_once.py --shape svd|qwen16k|temporal
Inputs from the device generator; a pre-pass launch, then three forward launches
(capture with `-k regex:pasa_fwd -s 2 -c 1`; temporal: `-k regex:packed -s 2 -c 1`)."""
import argparse, ctypes as C, math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib  # noqa: E402
from paper_2503_01873_b200 import bench_api as ba  # noqa: E402

SHAPES = {"svd": (50, 5, 5, 9216, 64, False), "qwen16k": (1, 28, 4, 16384, 128, True),
          "temporal": (9216, 5, 5, 25, 64, False)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="svd", choices=sorted(SHAPES))
    a = ap.parse_args()
    B, HQ, HKV, S, D, causal = SHAPES[a.shape]
    dev = torch.device("cuda:0")
    if a.shape == "qwen16k":  # the bench's headline data: uniform(30, 0.5)
        gi = ba.generate(ba.DistributionSpec(ba.DistKind.UNIFORM, 30.0, 0.5, 0.001, 7, B, HQ, S, D, HKV), dev)
    else:  # SVD: the resonance inputs (BASELINE configs[2])
        gi = ba.generate_resonance(7, B, HQ, S, D, device=dev)
    if a.shape == "temporal":  # the public entry point: the packed kernel with its pre-pass
        desc = _lib.Desc(B, HQ, HKV, S, S, D, S, S, 0, 0, 0.984497, math.sqrt(D))
        L = _lib.load()
        ws = torch.empty(L.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)
        o = torch.empty_like(gi.q)
        for _ in range(3):
            _lib.check(L.pasa_b200_attention_fwd(C.byref(desc), gi.q.data_ptr(), gi.k.data_ptr(),
                                                 gi.v.data_ptr(), o.data_ptr(), ws.data_ptr(), ws.numel(),
                                                 None, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        print("ok", a.shape, bool(torch.isfinite(o).all()))
        return
    L = _lib.load()
    desc = _lib.Desc(B, HQ, HKV, S, S, D, 128, 128, int(causal), 0, 0.984497, math.sqrt(D))
    kp, vp, o = torch.empty_like(gi.k), torch.empty_like(gi.v), torch.empty_like(gi.q)
    vmax = torch.zeros(B * HKV, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.pasa_b200_preprocess(C.byref(desc), C.c_void_p(gi.k.data_ptr()), C.c_void_p(gi.v.data_ptr()),
                                      C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()),
                                      C.c_void_p(vmax.data_ptr()), C.c_void_p(st)))
    for _ in range(3):
        _lib.check(L.pasa_b200_attention_fwd_prepped(C.byref(desc), C.c_void_p(gi.q.data_ptr()),
                                                     C.c_void_p(kp.data_ptr()), C.c_void_p(vp.data_ptr()),
                                                     C.c_void_p(vmax.data_ptr()), C.c_void_p(o.data_ptr()),
                                                     C.c_void_p(st)))
    torch.cuda.synchronize()
    print("ok", a.shape, bool(torch.isfinite(o).all()))


if __name__ == "__main__":
    main()
