#!/usr/bin/env python
"""PASA forward throughput on B200 -- the driver's bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE.json configs[1], the metric's configuration that fits one
GPU): Qwen2-7B attention, 28 query heads / 4 KV heads (GQA), d = 128, causal,
N = 16384 per sequence, one sequence per GPU (weak scaling: N GPUs process N
independent sequences; no collective on the data path).  A step is one pass
of the path over one batch: the key pre-pass kernel (K' = K^T M, pasa.cpp:53-56)
plus the fused PASA forward kernel (pasa.cpp:196-293).  FLOPs follow the FA
convention, 4 * B * Hq * S1 * S2 * d, halved for causal.

Inputs are synthetic, generated on the device with the reference's own
counter-based generator (bench.cpp:28-72; identical values): Appendix E's
uniform(30, 0.5) cell -- every pre-scale score is about
128 * 30^2 = 1.15e5 > 65504, so the naive FP16 FlashAttention returns 100 % NaN
on it, while the softmax itself is not degenerate (score spread ~9 in S/alpha).
A second block (``qwen_bias``) times and checks the Qwen-like channel-bias data
(hybrid(0, 10) + large K/Q channel offsets), whose
softmax is nearly one-hot.  Inputs (Q + K + V + O ~ 300 MB) exceed L2 and L2 is
also flushed (256 MiB write) between timed steps, outside the timed events.

``--impl reference`` times the reference's own CPU implementation
(oracle/_ref, compiled from /root/reference sources; pasa::pasa_attention,
PASA_FP16) on the host cores with a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PASA attn fwd TFLOPS (% FP16 peak) vs seqlen at 1/2/4/8 B200; RMSE vs FP32"
UNIT = "TFLOP/s"
BETA = 0.984497
HQ, HKV, D = 28, 4, 128
SEQ = 16384
SWEEP = (8192, 32768)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["bf16_tflops"]), float(m.get("bf16_tflops_sustained", 0.0)), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def causal_flops(B, H, S, d):
    return 4.0 * B * H * S * S * d / 2.0


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()  # the timed region starts only once samples flow
            while not self.lines and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.n0 = len(self.lines)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[max(0, getattr(self, "n0", 1) - 1):]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- inputs
HEADLINE = ("uniform", 30.0, 0.5)         # Appendix E cell 1: naive FP16 FA 100 % NaN
CHANS = (7, 23, 71, 101)                  # Qwen-like outlier channels
KBIAS = (400.0, -250.0, 300.0, -150.0)
QBIAS = (-140.0, 150.0, -160.0, 120.0)
SEED = 1234
DATA_DESC = ("synthetic: uniform(30, 0.5) (Appendix E, PAPER.md:596) via the reference's "
             "generator, device-generated")


def make_inputs(torch, dev, B, S, seed, data="headline"):
    """The bench tensors on the device.  ``headline``: the reference's uniform(30, 0.5)
    (bench.cpp:28-72, device generator: identical values).  ``qwen_bias``: hybrid(0, 10,
    p=0.001) plus the Qwen-like K/Q channel bias (scores ~ -1.6e5, nearly one-hot)."""
    from paper_2503_01873_b200 import bench_api as ba
    if data == "headline":
        gi = ba.generate(ba.DistributionSpec(ba.DistKind.UNIFORM, HEADLINE[1], HEADLINE[2], 0.001,
                                             seed, B, HQ, S, D, HKV), dev)
        return gi.q, gi.k, gi.v
    gi = ba.generate(ba.DistributionSpec(ba.DistKind.HYBRID, 0.0, 10.0, 0.001, seed, B, HQ, S, D,
                                         HKV), dev)
    q, k = gi.q.float(), gi.k.float()
    for c, kb, qb in zip(CHANS, KBIAS, QBIAS):
        k[..., c] += kb
        q[..., c] += qb
    return q.half(), k.half(), gi.v


# ----------------------------------------------------------------------------- reference arm
def reference_sample(threads_hint: int, S: int, seed: int = SEED):
    """One bounded sample of the bench workload for the CPU reference: the last nb query
    blocks of query head 0 against all S keys of KV head 0 -- the same values the B200
    arm generates (flat indices [0, S*d) of tensors 0/1/2 of the headline spec)."""
    import numpy as np

    from oracle.oracle import Oracle
    orc = Oracle()
    nb = min(max(1, threads_hint), S // 128)
    outs = []
    for tid in range(3):
        a = np.empty(S * D)
        orc.lib.orc_generate(0, HEADLINE[1], HEADLINE[2], 0.001, seed, tid, 0, a.size, a)
        outs.append(a.reshape(1, 1, S, D))
    q, k, v = outs
    return np.ascontiguousarray(q[:, :, S - nb * 128:]), k, v, nb


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def time_reference_step(ref, q, k, v, threads):
    """The thread count goes to the reference explicitly (AttnOptions::threads,
    parallel.hpp:20-32): under torchrun OMP_NUM_THREADS=1 would otherwise pin it to one."""
    from oracle.oracle import PASA_FP16, Problem
    pb = Problem(q, k, v)
    t0 = time.perf_counter()
    o = ref.pasa(pb, BETA, PASA_FP16, threads=threads)
    dt = time.perf_counter() - t0
    return dt, o


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import ref_available, RefLib
    cfg = {"workload": f"qwen2-7b-attn: B=1 Hq={HQ} Hkv={HKV} d={D} N={SEQ} causal",
           "parallelism": "openmp-host"}
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    ref = RefLib()
    cores = cpu_cores()
    q, k, v, nb = reference_sample(cores, SEQ)
    flops = 4.0 * nb * 128 * SEQ * D  # non-causal rows: the work the reference performs
    for _ in range(args.warmup):
        time_reference_step(ref, q, k, v, cores)
    times = [time_reference_step(ref, q, k, v, cores)[0] for _ in range(args.steps)]
    tot = sum(times)
    val = flops * len(times) / tot / 1e12
    sample = (f"pasa::pasa_attention PASA_FP16 (oracle/_ref), 1 head x {nb} query blocks "
              f"x {SEQ} keys, d={D}, beta={BETA}; the reference has no causal mask or GQA "
              f"(SPEC.md:189, tensor.cpp:24-26), so each sampled row runs over all keys and "
              f"its performed FLOPs (4*rows*S2*d) are counted")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f16 (emulated on f64 carriers)",
            "data": DATA_DESC + " (the B200 arm's values for head 0, on the host)",
            "config": cfg,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2503_01873_b200 import _lib
    from paper_2503_01873_b200.api import LOG2E

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L = _lib.load()
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def setup(S, data="headline"):
        q, k, v = make_inputs(torch, dev, 1, S, seed=SEED + rank, data=data)
        desc = _lib.Desc(1, HQ, HKV, S, S, D, 128, 128, 1, 0, BETA, math.sqrt(D))
        _lib.check(L.pasa_b200_check(C.byref(desc)))
        kp = torch.empty_like(k)
        vp = torch.empty_like(v)
        vmax = torch.zeros(HKV, dtype=torch.float32, device=dev)
        o = torch.empty_like(q)
        return q, k, v, kp, vp, vmax, o, desc

    def launch(bufs, evs=None):
        q, k, v, kp, vp, vmax, o, desc = bufs
        if evs:
            evs[0].record(stream)
        _lib.check(L.pasa_b200_preprocess(C.byref(desc), k.data_ptr(), v.data_ptr(), kp.data_ptr(),
                                          vp.data_ptr(), vmax.data_ptr(), sh))
        if evs:
            evs[1].record(stream)
        _lib.check(L.pasa_b200_attention_fwd_prepped(C.byref(desc), q.data_ptr(), kp.data_ptr(),
                                                     vp.data_ptr(), vmax.data_ptr(), o.data_ptr(), sh))
        if evs:
            evs[2].record(stream)

    def timed(S, steps, warmup, sampler=None, data="headline"):
        bufs = setup(S, data)
        for _ in range(warmup):
            launch(bufs)
        barrier()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        ctx = sampler if sampler is not None else _Null()
        with ctx:
            barrier()
            for i in range(steps):
                flush.zero_()  # L2 flush, outside the timed events
                launch(bufs, evs[i])
            barrier()
        step_ms = [e[0].elapsed_time(e[2]) for e in evs]
        fwd_ms = [e[1].elapsed_time(e[2]) for e in evs]
        return bufs, step_ms, fwd_ms

    # ---------------- headline
    sampler = ClockSampler(local)
    bufs, step_ms, fwd_ms = timed(SEQ, args.steps, args.warmup, sampler)
    tot_s = max_over_ranks(sum(step_ms) / 1e3)
    flops_rank = causal_flops(1, HQ, SEQ, D)
    value = flops_rank * world * args.steps / tot_s / 1e12
    fwd_avg_ms = max_over_ranks(statistics.mean(fwd_ms))
    achieved = flops_rank / (fwd_avg_ms / 1e3) / 1e12
    peak_burst, peak_sust, peak_kind = peaks()

    # ---------------- numerics on the measured output: RMSE vs FP64, non-finite count
    q, k, v, kp, vp, vmax, o, desc = bufs
    nonfinite = int((~torch.isfinite(o)).sum().item())
    from paper_2503_01873_b200 import bench_api as ba
    from paper_2503_01873_b200 import flash_fp16_fwd, pasa_attention_fwd
    rows = 256
    r0 = SEQ - rows
    hs = [0, 1, 7, 27]  # heads in different KV groups

    def rmse_rows(q_, k_, v_, o_):
        errs, norms = 0.0, 0.0
        for h in hs:
            g = ba.golden_attention(q_[:, h:h + 1], k_[:, h // 7:h // 7 + 1], v_[:, h // 7:h // 7 + 1],
                                    causal=True, rows=slice(r0, SEQ))
            errs += float(((o_[:, h:h + 1, r0:].double() - g) ** 2).sum())
            norms += float((g ** 2).sum())
        return math.sqrt(errs / norms)
    rmse_fp32 = rmse_rows(q, k, v, o)

    # The Qwen-like channel-bias data: outlier keys on the bias
    # channels win each row by ~235 in S/alpha, so the softmax is nearly one-hot there; its
    # own kernel time, non-finite counts and RMSE are reported beside the headline.
    qb_bufs, _, qb_fwd = timed(SEQ, max(3, args.steps // 3), 2, data="qwen_bias")
    qq, qk, qv, _, _, _, qo, _ = qb_bufs
    qo_fa = flash_fp16_fwd(qq, qk, qv, causal=True)
    qwen_bias = {"fwd_kernel_tflops": causal_flops(1, HQ, SEQ, D) /
                 (max_over_ranks(statistics.mean(qb_fwd)) / 1e3) / 1e12,
                 "rmse_vs_fp64": rmse_rows(qq, qk, qv, qo),
                 "nonfinite": int((~torch.isfinite(qo)).sum()),
                 "fa16_nonfinite_pct": ba.nan_stats(qo_fa),
                 "data": "hybrid(0, 10, p=0.001) + K channels 7/23/71/101 biased +400/-250/+300/-150, "
                         "Q -140/+150/-160/+120 (pre-scale scores ~ -1.6e5; nearly one-hot softmax)"}
    del qb_bufs, qq, qk, qv, qo, qo_fa

    # ---------------- seqlen sweep (same config, other N)
    sweep = {}
    for S in SWEEP:
        if os.environ.get("PASA_BENCH_NO_SWEEP"):
            break
        _, sm, fm = timed(S, max(3, args.steps // 3), 2)
        ts = max_over_ranks(sum(sm) / 1e3)
        sweep[str(S)] = {"tflops": causal_flops(1, HQ, S, D) * world * len(sm) / ts / 1e12,
                         "fwd_kernel_tflops": causal_flops(1, HQ, S, D) / (max_over_ranks(statistics.mean(fm)) / 1e3) / 1e12}
        del _
    sweep[str(SEQ)] = {"tflops": value, "fwd_kernel_tflops": achieved}

    # ---------------- the naive FP16 FA (beta = 0) on the same pipeline and inputs
    fa_ms = []
    o_fa = torch.empty_like(o)
    desc0 = _lib.Desc(1, HQ, HKV, SEQ, SEQ, D, 128, 128, 1, 0, 0.0, math.sqrt(D))
    for i in range(args.warmup + max(3, args.steps // 3)):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(L.pasa_b200_flash_fp16_fwd(C.byref(desc0), q.data_ptr(), k.data_ptr(),
                                              v.data_ptr(), o_fa.data_ptr(), sh))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if i >= args.warmup:
            fa_ms.append(e0.elapsed_time(e1))
    fa_tflops = flops_rank / (max_over_ranks(statistics.mean(fa_ms)) / 1e3) / 1e12
    fa16 = {"fwd_kernel_tflops": fa_tflops, "pasa_over_fa16_time": fa_tflops / achieved,
            "nonfinite_outputs": int((~torch.isfinite(o_fa)).sum().item()),
            "nonfinite_pct": ba.nan_stats(o_fa),
            "note": "beta = 0: scale after the FP16 score store (attention.cpp:134-136); "
                    "|QK^T| ~ 1.15e5 overflows FP16 there, PASA has 0 non-finite outputs"}
    del o_fa

    # ---------------- e2e through the public host entry point (pinned buffers)
    qh = q.cpu().pin_memory()
    kh = k.cpu().pin_memory()
    vh = v.cpu().pin_memory()
    oh = torch.empty_like(qh).pin_memory()
    e2e_times = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        _lib.check(L.pasa_b200_attention_host(C.byref(desc), qh.data_ptr(), kh.data_ptr(),
                                              vh.data_ptr(), oh.data_ptr()))
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_s = max_over_ranks(sum(e2e_times))
    e2e_val = flops_rank * world * len(e2e_times) / e2e_s / 1e12
    assert torch.equal(oh, o.cpu()), "host entry point disagrees with the device path"
    bytes_in = (q.numel() + k.numel() + v.numel()) * 2
    bytes_out = o.numel() * 2
    # the e2e roofline: the same copies alone (H2D on one stream, D2H on another, at once)
    s_a, s_b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    copy_s = []
    for i in range(4):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        with torch.cuda.stream(s_a):
            for hst, dst in ((qh, q), (kh, k), (vh, v)):
                dst.copy_(hst, non_blocking=True)
        with torch.cuda.stream(s_b):
            oh.copy_(o, non_blocking=True)
        torch.cuda.synchronize(dev)
        if i:
            copy_s.append(time.perf_counter() - t0)
    copy_ms = max_over_ranks(min(copy_s)) * 1e3
    e2e_ms = e2e_s / len(e2e_times) * 1e3
    pcie = {"copy_only_ms": copy_ms, "e2e_ms": e2e_ms, "frac_of_copy_bound": copy_ms / e2e_ms,
            "h2d_GBps_concurrent": bytes_in / copy_ms / 1e6,
            "note": "H2D of Q, K, V and D2H of O alone, concurrently on two streams: the time "
                    "the host entry point cannot beat"}
    oh.copy_(o)  # restore (the copy above overwrote oh with the same values)

    # ---------------- CPU baseline (rank 0, N = 1 only)
    cpu_base = None
    parity = None
    if world == 1 and rank == 0 and not os.environ.get("PASA_BENCH_NO_CPU"):
        from oracle.oracle import ref_available, RefLib
        if ref_available():
            cores = cpu_cores()
            qs, ks, vs, nb = reference_sample(8 * cores, SEQ)  # ~10 s of reference work
            dt, o_ref = time_reference_step(RefLib(), qs, ks, vs, cores)
            cpu_base = {"value": 4.0 * nb * 128 * SEQ * D / dt / 1e12, "unit": UNIT,
                        "cores": cores, "kind": "reference",
                        "sample": f"pasa::pasa_attention (oracle/_ref) 1 head x {nb} query blocks "
                                  f"x {SEQ} keys, non-causal rows, {dt:.1f} s"}
            # parity on the identical sample: the B200 kernel (non-causal, like the
            # reference), the reference and the FP64 golden on the same rows
            from paper_2503_01873_b200 import pasa_attention_fwd
            qt, kt, vt = (torch.from_numpy(x).half().to(dev) for x in (qs, ks, vs))
            o_new = pasa_attention_fwd(qt, kt, vt, BETA).double()
            gold = ba.golden_attention(qt, kt, vt)
            o_rt = torch.from_numpy(o_ref).to(dev)
            parity = {"rows": nb * 128, "keys": SEQ, "head": 0,
                      "rmse_b200_vs_fp64": ba.rmse(o_new, gold),
                      "rmse_reference_vs_fp64": ba.rmse(o_rt, gold),
                      "rmse_b200_vs_reference": ba.rmse(o_new, o_rt),
                      "maxabs_rel_b200_vs_reference": float((o_new - o_rt).abs().max() /
                                                            o_rt.abs().max()),
                      "nan_pct_b200": ba.nan_stats(o_new), "nan_pct_reference": ba.nan_stats(o_rt),
                      "note": "identical FP16 inputs (the headline data's head 0, last query "
                              "blocks, all keys, no causal mask: the reference has none)"}

    traffic = None
    prof = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    clocks = sampler.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16",
        "data": DATA_DESC,
        "config": {"workload": f"qwen2-7b-attn: B=1/gpu Hq={HQ} Hkv={HKV} d={D} N={SEQ} causal",
                   "global_batch": world, "seq_len": SEQ, "heads_q": HQ, "heads_kv": HKV,
                   "head_dim": D, "causal": True, "beta": BETA, "s1": 128, "s2": 128,
                   "parallelism": f"shard-by-sequence x{world} (no collective)",
                   "l2": "inputs > L2 and 256 MiB flush between timed steps"},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_burst,
                     "unit": "TFLOP/s", "frac": achieved / peak_burst, "traffic": traffic,
                     "peak_kind": f"{peak_kind} bf16 burst (dense fp16 = bf16 rate)",
                     "frac_of_sustained": achieved / peak_sust if peak_sust else None,
                     "frac_of_datasheet_2250": achieved / 2250.0,
                     "kernel": "pasa_fwd_kernel<128,true>"},
        "cpu_baseline": cpu_base,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": bytes_in,
                "d2h_bytes_per_step": bytes_out,
                "api": "pasa_b200_attention_host (C-ABI, pinned host buffers)", "pcie": pcie},
        "gpu_launches": 3 * args.steps,  # key pre-pass, V scale, fused forward
        "clocks": clocks,
        "rmse_vs_fp32": rmse_fp32, "rmse_golden": "FP64 golden_attention on device, 4 heads x 256 rows",
        "nonfinite_outputs": nonfinite, "parity_sample": parity, "qwen_bias": qwen_bias,
        "fa16_baseline": fa16,
        "sweep": sweep,
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
