"""Regenerate DESIGN.md's headline paragraph and sweep table from profiles/ (tool).
    python tools/design_numbers.py"""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "DESIGN.md")
s = open(P).read()
i = s.index("Headline (one B200, `profiles/r01_bench_16k.json`")
j = s.index("The SVD temporal row")
sw = json.load(open(os.path.join(ROOT, "profiles", "r01_sweep.json")))
b = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_16k.json")))
ncu = open(os.path.join(ROOT, "profiles", "r01_ncu_pasa_fwd_summary.txt")).read()
num = lambda k: float(re.search(k + r"\s+\S+\s+([\d.]+)", ncu).group(1))  # noqa: E731
tensor, issue = num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"), num(
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed")
dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
rows = [f"| {r['config']} | {r['B']}×{r['Hq']}/{r['Hkv']} | {r['N']} | {r['d']} | "
        f"{'yes' if r['causal'] else 'no'} | {r['fwd_tflops']:.0f} | {r['step_tflops']:.0f} | "
        f"{100 * r['fwd_frac_of_measured_peak']:.1f} % | {r['rmse_vs_fp32_full']:.1e} | "
        f"{r['rmse_vs_fp64_sampled']:.1e} | {r['nonfinite']} |" for r in sw]
a, fa = b["roofline"]["achieved"], b["fa16_baseline"]["fwd_kernel_tflops"]
new = f"""Headline (one B200, `profiles/r01_bench_16k.json`; `python bench.py` defaults, clocks at
{b['clocks']['sm_mhz']:.0f} MHz, no throttle reason): Qwen2-7B attention (28 q / 4 kv heads,
d = 128, causal), N = 16384 → **fused kernel {a:.0f} TFLOP/s =
{100 * b['roofline']['frac']:.1f} % of the measured 1679.9 TFLOP/s dense-FP16 peak**
({100 * b['roofline']['frac_of_sustained']:.0f} % of the sustained 1416), {b['value']:.0f} TFLOP/s per step
(rank-1 key pre-pass + V scale + forward; the forward is 98.8 % of the step).  N = 8192:
{b['sweep']['8192']['fwd_kernel_tflops']:.0f} ({100 * b['sweep']['8192']['fwd_kernel_tflops'] / 1679.9:.1f} %), N = 32768:
{b['sweep']['32768']['fwd_kernel_tflops']:.0f} ({100 * b['sweep']['32768']['fwd_kernel_tflops'] / 1679.9:.1f} %).  The naive FP16 FlashAttention on the *same*
pipeline (β = 0) runs at {fa:.0f} TFLOP/s{(f", so PASA's shift and recovery cost ≈ {100 * (fa / a - 1):.0f} %" if fa > a else f" in the same run, {100 * (1 - fa / a):.0f} % below PASA (the two modes time within run-to-run noise of each other; this FA16 timing synchronises every launch)")}
— and on the Qwen-like biased inputs that baseline returns
{b['fa16_baseline']['nonfinite_outputs'] / 1e6:.1f} M non-finite outputs while PASA returns 0 (on uniform(30, 0.5): FA16 100 % NaN,
PASA RMSE {b['accuracy_uniform30']['rmse_vs_fp64']:.1e}).  End-to-end through the host C-ABI with pinned buffers
(copy-in, compute and copy-out pipelined over query-head pieces): {b['e2e']['value']:.0f} TFLOP/s; the reference's own CPU
PASA on the box's {b['cpu_baseline']['cores']} host cores: {b['cpu_baseline']['value']:.3f} TFLOP/s.  ncu
(`profiles/r01_ncu_pasa_fwd_summary.txt`): tensor pipe active {tensor:.0f} % of the kernel's cycles,
issue active {issue:.0f} %, DRAM {dram:.0f} MB per launch.

### Sequence-length sweep (BASELINE configs; `tools/sweep.py` → `profiles/r01_sweep.json`)

Inputs from the device generator (identical to the reference's `generate`); RMSE of the
**whole output** against the device FP32 golden (`bench_api.golden_rmse`) and of sampled
rows against the FP64 golden.  The sweep runs configurations back to back, so the long
ones run at power-capped clocks (compare the 16K line with the bench's short run).

| config | B×Hq/Hkv | N | d | causal | fwd TFLOP/s | step TFLOP/s | of measured peak | RMSE vs FP32 (all rows) | RMSE vs FP64 (sampled) | non-finite |
|---|---|---|---|---|---|---|---|---|---|---|
""" + "\n".join(rows) + "\n\n"
open(P, "w").write(s[:i] + new + s[j:])
print("updated")
