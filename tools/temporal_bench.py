"""SVD temporal attention (BASELINE configs[2], N = 25 frames, d = 64) throughput (tool).
    python tools/temporal_bench.py [B ...]   (default 1024 9216)
Short sequences run on the packed kernel (csrc/pasa_fwd_packed.cu); the step is the key
pre-pass + the forward, CUDA events, inputs from the resonance generator."""
import math, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import pasa_attention_fwd  # noqa: E402
from paper_2503_01873_b200 import bench_api as ba  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    bs = [int(x) for x in sys.argv[1:]] or [1024, 9216]
    for B in bs:  # 9216 = the spatial token count of the SVD shape
        q = torch.randn(B, 5, 25, 64, device=dev).half()
        k, v = torch.randn_like(q), torch.randn_like(q)
        for _ in range(2):
            o = pasa_attention_fwd(q, k, v, 0.984497, s1=25, s2=25)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            o = pasa_attention_fwd(q, k, v, 0.984497, s1=25, s2=25)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = 4 * B * 5 * 25 * 25 * 64
        byts = 4 * q.numel() * 2
        g = ba.golden_attention(q[:64], k[:64], v[:64])
        print(f"temporal B={B} H=5 N=25 d=64: {ms:.3f} ms per step, {fl / ms / 1e9:.2f} TFLOP/s, "
              f"{byts / ms / 1e6:.0f} GB/s of Q/K/V/O, rmse vs FP64 (64 seqs) {ba.rmse(o[:64], g):.2e}")


if __name__ == "__main__":
    main()
