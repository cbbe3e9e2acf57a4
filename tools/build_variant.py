"""Build a variant of libpasa_b200.so with extra -D flags on pasa_fwd.cu and pasa_fwd_packed.cu (tool).
    python tools/build_variant.py NAME [--rev GIT_REV] -DPASA_POLY_EVERY=2 ...
writes paper_2503_01873_b200/_build/NAME.so (for tools/variants.py).  --rev builds
every CUDA source (and header) of the library as of another commit (e.g. HEAD for an
A/B run of uncommitted changes against the last commit)."""
import os, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_01873_b200 import build as B  # noqa: E402
name, flags = sys.argv[1], sys.argv[2:]
rev = None
if flags[:1] == ["--rev"]:
    rev, flags = flags[1], flags[2:]
out = os.path.join(B.OUT, "var_" + name)
os.makedirs(out, exist_ok=True)
csrc, inc = B.CSRC, os.path.join(ROOT, "include")
if rev:
    tmp = tempfile.mkdtemp(prefix="pasa_rev_")
    csrc, inc = os.path.join(tmp, "pkg", "csrc"), os.path.join(tmp, "include")  # ../../include
    os.makedirs(csrc), os.makedirs(inc)
    for f in B.SOURCES + B.HEADERS:
        rel = f"paper_2503_01873_b200/csrc/{f}"
        open(os.path.join(csrc, f), "wb").write(
            subprocess.run(["git", "-C", ROOT, "show", f"{rev}:{rel}"], check=True, capture_output=True).stdout)
    open(os.path.join(inc, "pasa_b200.h"), "wb").write(
        subprocess.run(["git", "-C", ROOT, "show", f"{rev}:include/pasa_b200.h"], check=True,
                       capture_output=True).stdout)
else:
    B.build()
flags_base = [f for f in B.FLAGS if f not in ("-Xptxas", "-v") and not f.startswith("-I")]
objs = []
for src in B.SOURCES:
    o = os.path.join(B.OUT, src.replace(".cu", ".o"))
    # flags the launcher must see too: the trace hook, the prologue row sum's scratch
    shared = [f for f in flags if f in ("-DPASA_TRACE", "-DPASA_TRACE_CTA") or f.startswith("-DPASA_PRO_SUM")]
    kern = src in ("pasa_fwd.cu", "pasa_fwd_packed.cu")
    if rev or (kern and flags) or src == "pasa_fwd.cu" or (shared and src == "capi.cu"):
        o = os.path.join(out, src.replace(".cu", ".o"))
        subprocess.run([B.NVCC, *B.ARCH, *flags_base, f"-I{inc}", f"-I{csrc}",
                        *(flags if kern else shared),
                        "-c", os.path.join(csrc, src), "-o", o], check=True)
    objs.append(o)
subprocess.run([B.NVCC, *B.ARCH, "-shared", "-cudart", "static", "-o",
                os.path.join(B.OUT, name + ".so"), *objs], check=True)
print(os.path.join(B.OUT, name + ".so"))
