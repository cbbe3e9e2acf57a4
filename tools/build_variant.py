"""Build a variant of libpasa_b200.so with extra -D flags on pasa_fwd.cu (tool).
    python tools/build_variant.py NAME [--src other_pasa_fwd.cu] -DPASA_POLY_EVERY=2 ...
writes paper_2503_01873_b200/_build/NAME.so (for tools/variants.py); --src builds the
fused kernel from another copy of pasa_fwd.cu (e.g. the previous commit's, for A/B runs)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import build as B  # noqa: E402
name, flags = sys.argv[1], sys.argv[2:]
src_fwd = os.path.join(B.CSRC, "pasa_fwd.cu")
if flags[:1] == ["--src"]:
    src_fwd, flags = os.path.abspath(flags[1]), flags[2:]
B.build()
out = os.path.join(B.OUT, "var_" + name)
os.makedirs(out, exist_ok=True)
objs = []
for src in B.SOURCES:
    o = os.path.join(B.OUT, src.replace(".cu", ".o"))
    if src == "pasa_fwd.cu":
        o = os.path.join(out, "pasa_fwd.o")
        subprocess.run([B.NVCC, *B.ARCH, *[f for f in B.FLAGS if f not in ("-Xptxas", "-v")], *flags,
                        f"-I{B.CSRC}", "-c", src_fwd, "-o", o], check=True)
    objs.append(o)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o",
                os.path.join(B.OUT, name + ".so"), *objs], check=True)
print(os.path.join(B.OUT, name + ".so"))
