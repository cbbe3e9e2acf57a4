"""Device parts of the benchmark surface: the input
generators against the oracle (bit-exact uniform), the FP64 device golden,
rmse/nan_stats and range_report against the reference's CPU versions, and the
device sweep/CLI against the reference's overflow outcomes."""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle.oracle import Problem
from paper_2503_01873_b200 import bench_api as ba
from paper_2503_01873_b200.api import BETA_STAR, PasaParams, PolicyId

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def _np(t):
    return t.double().cpu().numpy()


@pytest.mark.parametrize("kind,x0,am", [("uniform", 30.0, 0.5), ("uniform", -3.0, 1e3),
                                        ("hybrid", 0.0, 10.0), ("hybrid", 20.0, 100.0)])
def test_generator_matches_reference(dev, orc, kind, x0, am):
    B, H, S, D = 2, 3, 1000, 64  # 384000 elements per tensor
    spec = ba.DistributionSpec(ba.DistKind.UNIFORM if kind == "uniform" else ba.DistKind.HYBRID,
                               x0, am, 0.001, 7, B, H, S, D)
    gi = ba.generate(spec, dev)
    want = orc.generate(kind, x0, am, 7, B, H, S, D)
    for got, w in zip((gi.q, gi.k, gi.v), want):
        g = _np(got)
        mism = int((g != w).sum())
        if kind == "uniform":
            assert mism == 0  # integer hash + exact double ops: bit-exact
        else:
            assert mism <= 2, mism  # device log/cos within 1 ulp; FP16 rounding hides it


def test_generator_offsets_gqa_and_errors(dev, orc):
    t = ba.generate_tensor(ba.DistKind.HYBRID, 1.0, 5.0, 0.01, 3, 1, (4096,), dev, start=12345)
    a = np.empty(4096)
    orc.lib.orc_generate(1, 1.0, 5.0, 0.01, 3, 1, 12345, a.size, a)
    assert int((_np(t) != a).sum()) <= 1
    gi = ba.generate(ba.DistributionSpec(ba.DistKind.UNIFORM, 0, 1, 0.001, 1, 1, 4, 256, 128, 2),
                     dev)
    assert gi.q.shape == (1, 4, 256, 128) and gi.k.shape == (1, 2, 256, 128)
    assert np.array_equal(_np(gi.k), orc.generate("uniform", 0, 1, 1, 1, 4, 256, 128, Hkv=2)[1])
    with pytest.raises(ValueError, match="p must lie"):
        ba.generate(ba.DistributionSpec(ba.DistKind.HYBRID, p=0.0), dev)


def test_resonance_generator_matches_oracle(dev, orc):
    gi = ba.generate_resonance(0, 1, 2, 512, 64, device=dev)
    want = orc.generate_resonance(0, 1, 2, 512, 64)
    for got, w in zip((gi.q, gi.k, gi.v), want):
        assert int((_np(got) != w).sum()) <= 2


def test_device_golden_rmse_nan_stats_match_reference(dev, orc, ref):
    q, k, v = orc.generate("hybrid", 5.0, 10.0, 4, 1, 2, 384, 64)
    pb = Problem(q, k, v)
    gold_cpu = ref.golden(pb)
    qt, kt, vt = (torch.from_numpy(x).half().to(dev) for x in (q, k, v))
    gold = _np(ba.golden_attention(qt, kt, vt))
    assert np.abs(gold - gold_cpu).max() <= 1e-12
    g32 = _np(ba.golden_attention(qt, kt, vt, dtype=torch.float32))
    assert np.abs(g32 - gold_cpu).max() <= 2e-4  # FP32 softmax over 384 keys, |O| ~ 5
    gs = _np(ba.golden_attention(qt, kt, vt, rows=slice(128, 256)))
    assert np.abs(gs - gold_cpu[:, :, 128:256]).max() <= 1e-12
    o = ref.pasa(pb)
    ot = torch.from_numpy(o).to(dev)
    assert abs(ba.rmse(ot, torch.from_numpy(gold_cpu).to(dev)) - ref.rmse(o, gold_cpu)) <= 1e-15
    bad = o.copy()
    bad[0, 0, 0, 0] = np.inf
    assert math.isnan(ba.rmse(torch.from_numpy(bad).to(dev), torch.from_numpy(gold_cpu).to(dev)))
    assert ba.nan_stats(torch.from_numpy(bad).to(dev)) == ref.nan_stats(bad)
    with pytest.raises(ba.ZeroNormError):
        ba.rmse(ot, torch.zeros_like(ot))


def test_causal_golden_matches_oracle(dev, orc):
    q, k, v = orc.generate("hybrid", 0.0, 10.0, 9, 1, 2, 256, 64)
    gold_cpu = orc.golden(Problem(q, k, v, causal=True))
    qt, kt, vt = (torch.from_numpy(x).half().to(dev) for x in (q, k, v))
    assert np.abs(_np(ba.golden_attention(qt, kt, vt, causal=True)) - gold_cpu).max() <= 1e-12


def test_range_report_reduces_biased_range(dev):
    """SPEC.md acceptance 7: biased inputs (x0 >= 10 Am): max|S'| < 0.2 max|S/alpha|."""
    gi = ba.generate(ba.DistributionSpec(ba.DistKind.UNIFORM, 30.0, 0.5, 0.001, 0, 1, 2, 512, 128),
                     dev)
    params = PasaParams.make(128, BETA_STAR, math.sqrt(128.0))
    rep = ba.range_report(gi.q, gi.k, params, 128)
    t = rep.total
    assert len(rep.per_head) == 2
    assert max(abs(t.s_after_min), abs(t.s_after_max)) < 0.2 * max(abs(t.s_before_min),
                                                                  abs(t.s_before_max))
    assert rep.overflow_predicted(params.alpha)  # x0 = 30: |QK^T| > 65504 (Appendix E)
    csv = ba.range_csv(rep).splitlines()
    assert csv[0].startswith("batch,head,k_min_before") and len(csv) == 3


def test_sweep_appendix_e_outcomes(dev, orc, ref):
    """The six Appendix-E cells at (1, 2, 256, 128): FA_PARTIAL_FP16 overflows exactly where
    the reference's does, PASA_FP16 never does, and the PASA rmse meets Tier 1 against the
    reference's own PASA rmse on identical (device-generated) inputs."""
    from paper_2503_01873_b200.__main__ import PRESETS
    specs = [ba.DistributionSpec(ba.DistKind.UNIFORM if k == "uniform" else ba.DistKind.HYBRID,
                                 x0, am, 0.001, 0, 1, 2, 256, 128)
             for k, x0, am in PRESETS["appendix-e"]]
    opts = ba.SweepOptions(policies=[PolicyId.PASA_FP16, PolicyId.FA_PARTIAL_FP16,
                                     PolicyId.FA_FP32], diagnose=True)
    rows = ba.sweep(specs, opts, dev)
    assert len(rows) == 18
    for i, (k, x0, am) in enumerate(PRESETS["appendix-e"]):
        pasa, fa, fp32 = rows[3 * i:3 * i + 3]
        q, kk, v = orc.generate(k, x0, am, 0, 1, 2, 256, 128)
        pb = Problem(q, kk, v)
        gold = ref.golden(pb)
        r_ref = ref.rmse(ref.pasa(pb), gold)
        assert pasa.nan_pct == 0.0 and not pasa.error
        assert pasa.rmse <= 1.25 * r_ref + 1e-3, (k, x0, am, pasa.rmse, r_ref)
        assert fa.nan_pct == ref.nan_stats(ref.flash(pb)), (k, x0, am)
        assert "FA_PARTIAL_FP16 only" in fp32.error and math.isnan(fp32.rmse)  # never aborts
        assert pasa.has_ranges
        assert max(abs(pasa.s_min_after), abs(pasa.s_max_after)) < max(
            abs(pasa.s_min_before), abs(pasa.s_max_before))
    csv = ba.report_csv(rows)
    assert csv.count("\n") == 19


def test_cli_sweep_gate_and_run(dev, tmp_path):
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "paper_2503_01873_b200"]
    r = subprocess.run(cmd + ["sweep", "--preset", "appendix-e", "--small", "--must-be-finite",
                              "PASA_FP16", "--json", str(tmp_path / "s.json")],
                       capture_output=True, text=True, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr
    doc = json.load(open(tmp_path / "s.json"))
    assert doc["config"]["shape"] == [1, 2, 256, 64] and len(doc["rows"]) == 12
    r = subprocess.run(cmd + ["sweep", "--preset", "appendix-e", "--shape", "1,2,256,128",
                              "--must-be-finite", "FA_PARTIAL_FP16"], capture_output=True,
                       text=True, cwd=ROOT, env=env)
    assert r.returncode == 2  # naive FP16 FA overflows on the x0 = 30 cells at d = 128
    d = str(tmp_path / "in")
    r = subprocess.run(cmd + ["gen", "--kind", "hybrid", "--x0", "30", "--am", "10", "--shape",
                              "1,2,256,128", "--out-dir", d], capture_output=True, text=True,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr
    r = subprocess.run(cmd + ["run", "--q", f"{d}/q.npy", "--k", f"{d}/k.npy", "--v", f"{d}/v.npy",
                              "--policy", "PASA_FP16", "--diagnose", "--out", f"{d}/o.npy"],
                       capture_output=True, text=True, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr
    row = r.stdout.splitlines()[1].split(",")
    assert row[0] == "PASA_FP16" and row[1] == "file" and float(row[12]) == 0.0
    assert float(row[11]) < 0.05 and row[13] != ""  # rmse vs the device golden; ranges filled
    assert np.load(f"{d}/o.npy").shape == (1, 2, 256, 128)


def test_device_api_rejects_misread_tensors(dev):
    """The C-ABI takes raw fp16 pointers: the Python entry points reject wrong dtypes,
    host/device mixes and mis-shaped outputs before launching, and take the workspace
    size in bytes whatever its dtype."""
    from paper_2503_01873_b200 import flash_fp16_fwd, pasa_attention_fwd
    q = torch.randn(1, 2, 256, 64, device=dev).half()
    with pytest.raises(ValueError, match="must be float16"):
        pasa_attention_fwd(q.float(), q, q)
    with pytest.raises(ValueError, match="must be float16"):
        flash_fp16_fwd(q, q.float(), q)
    with pytest.raises(ValueError, match="CUDA tensors"):
        flash_fp16_fwd(q, q.cpu(), q)
    with pytest.raises(ValueError, match="out must be"):
        pasa_attention_fwd(q, q, q, out=torch.empty(1, 2, 128, 64, device=dev, dtype=torch.float16))
    ref = pasa_attention_fwd(q, q, q)
    ws = torch.empty(1 << 20, dtype=torch.float32, device=dev)  # 4 MiB as floats
    assert torch.equal(pasa_attention_fwd(q, q, q, workspace=ws), ref)
