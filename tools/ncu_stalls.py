"""Warp-state samples of an ncu --set full report by opcode and top instructions (tool).
    python tools/ncu_stalls.py gpurun_out/ncu_fwd128.ncu-rep > profiles/r02_ncu_pasa_fwd_stalls.txt"""
import csv, subprocess, sys
from collections import defaultdict


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, data = rows[1], rows[2:]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iall, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    tot = sum(float(r[iall] or 0) for r in data)
    by, ex = defaultdict(float), defaultdict(float)
    for r in data:
        toks = r[isrc].split()
        op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
        by[op] += float(r[iall] or 0)
        ex[op] += float(r[iex] or 0)
    print(f"# {rows[0][1][:110]}")
    print(f"# warp-state samples (all warps, issued or not): {tot:.0f}; by opcode (share, instructions executed)")
    for op, v in sorted(by.items(), key=lambda x: -x[1])[:20]:
        print(f"{op:12s} {100 * v / tot:5.1f} %  {ex[op]:.3g}")
    print("# top 20 instructions by samples (waits show up at the branch after the try-wait)")
    for r in sorted(data, key=lambda r: -float(r[iall] or 0))[:20]:
        print(f"{r[ia][-6:]}  {100 * float(r[iall]) / tot:5.2f} %  {r[isrc][:90]}")


if __name__ == "__main__":
    main()
