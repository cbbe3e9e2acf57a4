"""Timeline of the fused kernel from the PASA_TRACE build (profiling tool).

    python -m paper_2503_01873_b200.build --trace
    python tools/trace_fwd.py [--seq 16384] [--out gpurun_out/trace.json]

Runs the bench workload (Qwen2-7B attention, causal) through
libpasa_b200_trace.so and prints, for the traced CTAs, the per-block phase
durations (clock64 cycles) of each softmax warpgroup and the MMA issuer.
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CTAS, ROLES, ITERS, EVENTS = 4, 3, 32, 10


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=16384)
    ap.add_argument("--hq", type=int, default=28)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--causal", type=int, default=1)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--beta", type=float, default=0.984497, help="0 = the naive FP16 FA mode")
    ap.add_argument("--lib", default="libpasa_b200_trace.so",
                    help="trace build in paper_2503_01873_b200/_build (tools/build_variant.py NAME -DPASA_TRACE ...)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "trace.json"))
    a = ap.parse_args()
    from paper_2503_01873_b200 import _lib
    lib = _lib.load(os.path.join(ROOT, "paper_2503_01873_b200", "_build", a.lib))
    lib.pasa_b200_debug_set_trace.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    S, D = a.seq, a.d
    q = torch.randn(1, a.hq, S, D, device=dev).half()
    k = torch.randn(1, a.hkv, S, D, device=dev).half()
    v = torch.randn(1, a.hkv, S, D, device=dev).half()
    o = torch.empty_like(q)
    desc = _lib.Desc(1, a.hq, a.hkv, S, S, D, 128, 128, a.causal, 0, a.beta, math.sqrt(D))
    ws = torch.empty(lib.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)
    tr = torch.zeros(CTAS * ROLES * ITERS * EVENTS + 512 * 8 + 64, dtype=torch.int64, device=dev)  # + the PASA_STATE row-state area
    st = torch.cuda.current_stream().cuda_stream
    for it in range(3):
        lib.pasa_b200_debug_set_trace(tr.data_ptr() if it == 2 else None)
        _lib.check(lib.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(),
                                               v.data_ptr(), o.data_ptr(), ws.data_ptr(),
                                               ws.numel(), None, st))
    torch.cuda.synchronize()
    n = CTAS * ROLES * ITERS * EVENTS
    t = tr[:n].cpu().numpy().reshape(CTAS, ROLES, ITERS, EVENTS).astype(np.int64)
    pro = tr[n:].cpu().numpy().view(np.float32)[512 * 8:512 * 8 + CTAS * 4].reshape(CTAS, 2, 2)
    print("prologue cycles [cta][tile] (start -> G in TMEM, G -> stored):", pro.astype(int).tolist())
    res = {}
    for c in range(CTAS):
        base = t[c][t[c] > 0].min() if (t[c] > 0).any() else 0
        rel = np.where(t[c] > 0, t[c] - base, -1)
        res[c] = rel.tolist()
        print(f"=== CTA y={c}")
        print(" j | WG0: waitS  ldS p1+sc ppwait exp  stP  waitT  ldT  O   | WG1: waitS  ldS p1+sc ppwait exp  stP  waitT  ldT  O | period0 period1 | part0: WG0 WG1")
        for j in range(1, ITERS - 1):
            row = []
            for w in range(2):
                e = rel[w, j]
                if e[0] < 0:
                    row.append("   -" * 9)
                    continue
                nxt = rel[w, j + 1][0]
                row.append(" ".join(f"{x:5d}" for x in [e[1] - e[0], e[2] - e[1], e[3] - e[2],
                                                         e[8] - e[3], e[7] - e[8], e[4] - e[7], e[5] - e[4],
                                                         e[6] - e[5], (nxt - e[6]) if nxt > 0 else -1]))
            per = [rel[w, j + 1][0] - rel[w, j][0] if rel[w, j + 1][0] > 0 else -1 for w in range(2)]
            p0 = [rel[w, j][9] - rel[w, j][8] if rel[w, j][9] > 0 else -1 for w in range(2)]
            print(f"{j:2d} | {row[0]} | {row[1]} | {per[0]:6d} {per[1]:6d} | {p0[0]:5d} {p0[1]:5d}")
        m = rel[2]
        print(" MMA: j | t0: waitP issuePV issueS | t1: waitP issuePV issueS")
        for j in range(1, 12):
            e = m[j]
            print(f"   {j:2d} | {e[1]-e[0]:5d} {e[2]-e[1]:5d} {e[3]-e[2]:5d} | {e[5]-e[4]:5d} {e[6]-e[5]:5d} {e[7]-e[6]:5d} | gap t0->t1 {e[4]-e[3]:5d}")
        if c == 0:
            break
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(res, open(a.out, "w"))


if __name__ == "__main__":
    main()
