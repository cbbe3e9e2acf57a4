"""RMSE vs the FP64 golden of variant builds on one BASELINE shape (tool).
    python tools/ab_accuracy.py a.so b.so ...   (libraries in paper_2503_01873_b200/_build)
Inputs: the bench's headline data (uniform(30, 0.5)) and the Qwen-like bias data at
Qwen2-7B 16K causal; sampled rows: the last 256 of heads 0, 1, 7, 27."""
import ctypes as C, math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2503_01873_b200 import _lib  # noqa: E402
from paper_2503_01873_b200 import bench_api as ba  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    S, HQ, HKV, D = 16384, 28, 4, 128
    for data in ("headline", "qwen_bias", "hybrid0"):
        if data == "hybrid0":
            gi = ba.generate(ba.DistributionSpec(ba.DistKind.HYBRID, 0.0, 10.0, 0.001, 3, 1, HQ, S, D, HKV), dev)
            q, k, v = gi.q, gi.k, gi.v
        else:
            q, k, v = bench.make_inputs(torch, dev, 1, S, bench.SEED, data)
        gold = {h: ba.golden_attention(q[:, h:h + 1], k[:, h // 7:h // 7 + 1], v[:, h // 7:h // 7 + 1],
                                       causal=True, rows=slice(S - 256, S)) for h in (0, 1, 7, 27)}
        for so in sys.argv[1:]:
            L = C.CDLL(os.path.join(ROOT, "paper_2503_01873_b200", "_build", so))
            L.pasa_b200_attention_fwd.argtypes = [C.POINTER(_lib.Desc)] + [C.c_void_p] * 5 + [C.c_size_t, C.c_void_p, C.c_void_p]
            L.pasa_b200_workspace_size.restype = C.c_size_t
            L.pasa_b200_workspace_size.argtypes = [C.POINTER(_lib.Desc)]
            desc = _lib.Desc(1, HQ, HKV, S, S, D, 128, 128, 1, 0, bench.BETA, math.sqrt(D))
            ws = torch.empty(L.pasa_b200_workspace_size(C.byref(desc)), dtype=torch.uint8, device=dev)
            o = torch.empty_like(q)
            assert L.pasa_b200_attention_fwd(C.byref(desc), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             o.data_ptr(), ws.data_ptr(), ws.numel(), None,
                                             torch.cuda.current_stream().cuda_stream) == 0
            torch.cuda.synchronize()
            e = n = 0.0
            for h, g in gold.items():
                e += float(((o[:, h:h + 1, S - 256:].double() - g) ** 2).sum())
                n += float((g ** 2).sum())
            print(f"{data:10s} {so:12s} rmse vs FP64 {math.sqrt(e / n):.3e}  nonfinite {int((~torch.isfinite(o)).sum())}",
                  flush=True)


if __name__ == "__main__":
    main()
