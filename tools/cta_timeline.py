"""Per-CTA lifetimes of the fused forward (PASA_TRACE_CTA build; profiling tool).
    python tools/build_variant.py trcta -DPASA_TRACE_CTA
    python tools/cta_timeline.py --lib trcta.so [--seq 8192]
Prints the kernel span, the SMs' busy fraction, the mean gap between consecutive CTAs on
one SM (the per-CTA fill/drain the hardware scheduler cannot hide) and the tail."""
import argparse, ctypes as C, math, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="trcta.so")
    ap.add_argument("--seq", type=int, nargs="+", default=[8192, 16384])
    ap.add_argument("--hq", type=int, default=28)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--causal", type=int, default=1)
    a = ap.parse_args()
    L = _lib.load(os.path.join(ROOT, "paper_2503_01873_b200", "_build", a.lib))
    L.pasa_b200_debug_set_trace.argtypes = [C.c_void_p]
    dev = torch.device("cuda:0")
    for S in a.seq:
        D = 128
        q = torch.randn(1, a.hq, S, D, device=dev).half()
        k = torch.randn(1, a.hkv, S, D, device=dev).half()
        v = torch.randn_like(k)
        o = torch.empty_like(q)
        desc = _lib.Desc(1, a.hq, a.hkv, S, S, D, 128, 128, a.causal, 0, 0.984497, math.sqrt(D))
        ws = torch.empty(L.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)
        ncta = a.hkv * ((a.hq // a.hkv) * (S // 128) + 1) // 2
        tr = torch.zeros(4 * ncta + 64, dtype=torch.int64, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        for it in range(3):
            L.pasa_b200_debug_set_trace(tr.data_ptr() if it == 2 else None)
            _lib.check(L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                 o.data_ptr(), ws.data_ptr(), ws.numel(), None, st))
        torch.cuda.synchronize()
        e = tr[:4 * ncta].cpu().numpy().reshape(ncta, 4)
        e = e[e[:, 1] > 0]
        t0, t1 = e[:, 0].min(), e[:, 1].max()
        span = (t1 - t0) / 1e3
        busy = (e[:, 1] - e[:, 0]).sum() / 1e3
        nsm = len(np.unique(e[:, 2]))
        gaps, ends = [], []
        for sm in np.unique(e[:, 2]):
            r = e[e[:, 2] == sm]
            r = r[np.argsort(r[:, 0])]
            gaps += list((r[1:, 0] - r[:-1, 1]) / 1e3)
            ends.append((r[-1, 1] - t0) / 1e3)
        life = (e[:, 1] - e[:, 0]) / 1e3
        per_blk = life / np.maximum(e[:, 3], 1)
        print(f"S={S}: {len(e)} CTAs on {nsm} SMs, kernel span {span:.1f} us, SM busy {busy / (nsm * span):.3f}, "
              f"mean gap between CTAs on an SM {np.mean(gaps):.2f} us, last SM done at {min(ends):.1f}..{max(ends):.1f} us, "
              f"CTA life {life.mean():.1f} us mean ({np.median(per_blk):.3f} us per block, "
              f"fit: {np.polyfit(e[:, 3], life, 1)[1]:.2f} us fixed + {np.polyfit(e[:, 3], life, 1)[0]:.3f} us/block)")


if __name__ == "__main__":
    main()
