"""Copy one measurement run (gpurun_out/) into profiles/ (tool).
    python tools/write_profiles.py [TAG]      (TAG: the round, default r02)
Expects gpurun_out/{bench.json, bench_ref.json, sweep.json, overflow.json, launches.csv,
ncu_fwd128.ncu-rep, ncu_fwd64.ncu-rep, ncu_packed.ncu-rep} from tools/refresh_profiles.sh.
Writes profiles/TAG_* and profiles/roofline_traffic.json (DRAM bytes per launch, read by
bench.py)."""
import csv, json, os, re, shutil, statistics, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
METRICS = re.compile(
    r"^(dram__bytes_read\.sum|dram__bytes_write\.sum|gpu__time_duration\.sum|"
    r"l1tex__throughput\.avg\.pct_of_peak_sustained_elapsed|launch__block_size|launch__grid_size|"
    r"launch__registers_per_thread|launch__shared_mem_per_block_dynamic|sm__cycles_elapsed\.avg\.per_second|"
    r"sm__inst_executed_pipe_(alu|fma|xu)\.avg\.pct_of_peak_sustained_active|"
    r"sm__issue_active\.avg\.pct_of_peak_sustained_elapsed|"
    r"sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_elapsed|"
    r"smsp__average_warps_issue_stalled_.*_per_issue_active\.ratio|smsp__inst_executed\.sum)$")


def ncu_summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return "\n".join(f"{h:90s} {u:15s} {v}" for h, u, v in zip(hdr, units, vals) if METRICS.match(h)) + "\n"


def last_json(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    out = []
    for r in csv.reader(open(os.path.join(G, "launches.csv"))):
        if r and r[0] == "ID":
            hdr = r
            continue
        if out is not None and len(r) > 3 and "hdr" in locals() and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"]) * {"ns": 1, "us": 1e3, "ms": 1e6}.get(d["Metric Unit"], 1)
                out.append((int(d["ID"]), d["Kernel Name"], int(v)))
    with open(os.path.join(P, f"{tag}_ncu_launches.csv"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 60 (cold-cache, serialised): "
                "PASA_BENCH_NO_SWEEP=1 PASA_BENCH_NO_CPU=1 python bench.py --steps 2 --warmup 3\n")
        w = csv.writer(f)
        w.writerow(["id", "kernel", "duration_ns"])
        w.writerows(out)
    mean = lambda key: statistics.mean(o[2] for o in out if key in o[1]) / 1e3  # noqa: E731
    k, v, fw = mean("kprep_rank1"), mean("vscale"), mean("pasa_fwd_kernel")
    s128 = ncu_summary(os.path.join(G, "ncu_fwd128.ncu-rep"))
    open(os.path.join(P, f"{tag}_ncu_pasa_fwd_summary.txt"), "w").write(
        f"# ncu --set full --clock-control none --import-source on -k regex:pasa_fwd -s 2 -c 1 (B200, {tag})\n"
        "# command: python tools/ncu_once.py --shape qwen16k  (pre-pass, then three forward launches; the third is captured)\n"
        "# kernel: pasa_fwd_kernel<128, causal, PASA, no-diag> on Qwen2-7B attention (Hq=28, Hkv=4, N=16384), uniform(30, 0.5) inputs\n"
        + s128 + f"\n# per-step launch shares (profiles/{tag}_ncu_launches.csv, device steps of bench.py, cold & serialised): "
        f"kprep_rank1 {k:.1f} us, vscale {v:.1f} us, pasa_fwd {fw:.0f} us ({100 * fw / (k + v + fw):.1f} %)\n")
    s64 = ncu_summary(os.path.join(G, "ncu_fwd64.ncu-rep"))
    open(os.path.join(P, f"{tag}_ncu_pasa_fwd_d64_summary.txt"), "w").write(
        f"# ncu --set full --clock-control none --import-source on -k regex:pasa_fwd -s 2 -c 1 (B200, {tag})\n"
        "# command: python tools/ncu_once.py --shape svd  (B=50, H=5, N=9216, d=64, non-causal, resonance Q/K; BASELINE configs[2])\n"
        "# kernel: pasa_fwd_kernel<64, non-causal, PASA, no-diag>: S' row sums from the tensor core (pseudo-average GEMM), one MMA issuer per tile\n"
        + s64 + "# xu (MUFU) is the busiest pipe at d = 64: half the MMA work per exponential of d = 128\n")
    sp = ncu_summary(os.path.join(G, "ncu_packed.ncu-rep"))
    open(os.path.join(P, f"{tag}_ncu_packed_summary.txt"), "w").write(
        f"# ncu --set full --clock-control none --import-source on -k regex:packed -s 2 -c 1 (B200, {tag})\n"
        "# command: python tools/ncu_once.py --shape temporal  (B=9216, H=5, N=25, d=64: the SVD temporal attention)\n"
        "# kernel: pasa_fwd_packed_kernel<64, PASA, W = 32> with the pre-pass fused (self_prep): reads Q, K, V, writes O\n"
        + sp + "# memory-bound: algorithmic bytes 4 x 147.5 MB per launch\n")
    num = lambda key: float(re.search(re.escape(key) + r"\s+\S+\s+([\d.]+)", s128).group(1))  # noqa: E731
    rd, wr = num("dram__bytes_read.sum") * 1e6, num("dram__bytes_write.sum") * 1e6
    json.dump({"kernel": "pasa_fwd_kernel<128,true> (Qwen2-7B attn, N=16384, Hq=28, Hkv=4, causal)",
               "source": f"ncu --set full --clock-control none, {tag} (profiles/{tag}_ncu_pasa_fwd_summary.txt)",
               "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
               "algorithmic_bytes_per_launch": 268435456,
               "note": "write < O bytes: the tail of O is still in L2 (write-back) when the kernel ends"},
              open(os.path.join(P, "roofline_traffic.json"), "w"), indent=1)
    open(os.path.join(P, f"{tag}_bench_16k.json"), "w").write(json.dumps(last_json(os.path.join(G, "bench.json")), indent=1) + "\n")
    open(os.path.join(P, f"{tag}_bench_reference_arm.json"), "w").write(
        json.dumps(last_json(os.path.join(G, "bench_ref.json")), indent=1) + "\n")
    shutil.copy(os.path.join(G, "sweep.json"), os.path.join(P, f"{tag}_sweep.json"))
    if os.path.exists(os.path.join(G, "overflow.json")):
        shutil.copy(os.path.join(G, "overflow.json"), os.path.join(P, f"{tag}_overflow_stress.json"))
    print(f"profiles written; pasa_fwd {fw:.0f} us of {k + v + fw:.0f} us per step")


if __name__ == "__main__":
    main()
