"""Does the tcgen05 kind::f16 MMA flush FP16 subnormal inputs? (tool)"""
import ctypes as C, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = C.CDLL(os.path.join(ROOT, "tests", "cuda", "_build", "libumma_probe.so"))
lib.probe_umma.argtypes = [C.c_void_p] * 4 + [C.c_int] * 3
dev = torch.device("cuda:0")
for val in (2.0 ** -14, 2.0 ** -15, 2.0 ** -20, 2.0 ** -24):
    for acc in (0, 1):
        a = torch.full((128, 128), val, device=dev).half()   # P-like operand (SS path)
        b = torch.ones(128, 128, device=dev).half()
        out = torch.zeros(128, 128, device=dev)
        lib.probe_umma(a.data_ptr(), b.data_ptr(), None, out.data_ptr(), 128, 0, acc)
        p = torch.full((128, 128), val, device=dev).half()   # TS path: P staged in TMEM
        v = torch.ones(128, 128, device=dev).half()
        out2 = torch.zeros(128, 128, device=dev)
        lib.probe_umma(None, v.data_ptr(), p.data_ptr(), out2.data_ptr(), 128, 1, acc)
        torch.cuda.synchronize()
        print(f"val=2^{torch.log2(torch.tensor(val)).item():.0f} f32acc={acc}: SS sum={out[0,0].item():.4e} "
              f"TS sum={out2[0,0].item():.4e} exact={128*val:.4e}")
