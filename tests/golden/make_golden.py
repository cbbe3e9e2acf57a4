"""Regenerate the golden fixtures from the UNMODIFIED reference.

Run in the dev container (needs /root/reference and ``make -C oracle``):

    python tests/golden/make_golden.py

Every fixture is produced by the reference's own public API through
oracle/ref_capi.cpp: ``pasa::generate`` for the inputs (bench.cpp:63-72),
``pasa::pasa_attention`` (PASA_FP16, pasa.cpp:196-293), ``pasa::flash_attention``
(FA_PARTIAL_FP16 and FA_FP32, attention.cpp:92-180), ``pasa::golden_attention``
(attention.cpp:66-90) and ``pasa::preprocess_keys`` (pasa.cpp:53-56).  The
fixtures pin the oracle restatement (tests/test_oracle.py) on machines where
the reference itself is absent (the GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import (BETA_STAR, FA_FP32, FA_PARTIAL_FP16, PASA_FP16, Problem,  # noqa: E402
                           RefLib, build)

CELLS = [
    # name, kind, x0, Am, seed, (B, H, S, d), s1, s2
    ("uniform_x30_a0.5", "uniform", 30.0, 0.5, 0, (1, 2, 256, 128), 128, 128),
    ("uniform_x20_a20", "uniform", 20.0, 20.0, 1, (1, 2, 256, 128), 128, 128),
    ("hybrid_x30_a10", "hybrid", 30.0, 10.0, 0, (1, 2, 256, 128), 128, 128),
    ("hybrid_x0_a10_d64", "hybrid", 0.0, 10.0, 2, (1, 2, 256, 64), 64, 128),
    ("uniform_x5_a1_s2_64", "uniform", 5.0, 1.0, 3, (1, 1, 256, 64), 128, 64),
]


def main() -> None:
    build()
    ref = RefLib()
    for name, kind, x0, am, seed, (B, H, S, d), s1, s2 in CELLS:
        q, k, v = ref.generate(kind, x0, am, seed, B, H, S, d)
        pb = Problem(q, k, v, s1=s1, s2=s2)
        alpha = float(np.sqrt(d))
        diag, off = ref.shift_entries(s2, BETA_STAR, alpha)
        kp0 = ref.preprocess_block(k[0, 0, :s2], BETA_STAR, alpha)  # d x s2
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            meta=np.array([B, H, S, d, s1, s2, seed], dtype=np.int64),
            dist=np.array([x0, am, 0.0 if kind == "uniform" else 1.0]),
            beta=np.array(BETA_STAR), shift=np.array([diag, off]),
            q=q.astype(np.float16), k=k.astype(np.float16), v=v.astype(np.float16),
            kp_block0=kp0.astype(np.float16),
            pasa=ref.pasa(pb, policy=PASA_FP16).astype(np.float16),
            fa_partial=ref.flash(pb, policy=FA_PARTIAL_FP16).astype(np.float16),
            fa_fp32=ref.flash(pb, policy=FA_FP32).astype(np.float32),
            golden=ref.golden(pb).astype(np.float32),
        )
        print("wrote", name)


if __name__ == "__main__":
    main()
