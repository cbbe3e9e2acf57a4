"""CPU tests of the host surface around the path: the beta
solver (beta_solver.cpp), NPY ingestion, the report schema
(bench.cpp:249-331) and the CLI's non-GPU subcommands.  The device parts of
the same modules are in tests/test_gpu_surface.py."""
import json
import math
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from paper_2503_01873_b200 import bench_api as ba
from paper_2503_01873_b200.beta import (SolverDivergenceError, invariance_parameter,
                                        optimal_beta)
from paper_2503_01873_b200.npy import NpyFormatError, load_tensor_file, save_tensor_file

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ----------------------------------------------------------------------------- beta solver
def test_optimal_beta_matches_paper():
    # SPEC.md acceptance 1: {1-2^-4, 1-2^-5, 1-2^-6} -> {0.937500, 0.968994, 0.984497}
    for b0, want in [(1 - 2**-4, 0.937500), (1 - 2**-5, 0.968994), (1 - 2**-6, 0.984497)]:
        assert round(optimal_beta(b0, 128).beta_star, 6) == want


def test_invariance_matches_appendix_a_and_oracle(orc):
    # Appendix A: ideal {9, 15, 31, 63, 99, 999}; actual {8.971, 15.00, 31.25, 63.50, 102.2, 1031}
    rows = [(0.9, 8.971), (0.9375, 15.00), (0.96875, 31.25), (0.984375, 63.50), (0.99, 102.2),
            (0.999, 1031)]
    for beta, actual in rows:
        r = invariance_parameter(beta, 128)
        assert float(f"{r.inva_actual:.4g}") == actual, (beta, r.inva_actual)
        o = orc.invariance(beta, 128)
        assert (r.a, r.b, r.inva_actual, r.rel_err) == (o["a"], o["b"], o["inva_actual"],
                                                        o["rel_err"])
    for b0 in (1 - 2**-4, 1 - 2**-5, 1 - 2**-6, 0.9):
        s = optimal_beta(b0, 128)
        assert (s.beta_star, s.iterations) == orc.optimal_beta(b0, 128)


def test_beta_solver_errors():
    with pytest.raises(ValueError, match="beta must lie in"):
        invariance_parameter(1.0, 128)
    with pytest.raises(ValueError, match="n must be"):
        invariance_parameter(0.5, 0)
    with pytest.raises(ValueError, match="tol must be"):
        optimal_beta(0.9, 128, 0.0)
    assert issubclass(SolverDivergenceError, RuntimeError)


# ----------------------------------------------------------------------------- NPY
def test_npy_round_trip_and_numpy_interop(tmp_path):
    a = np.random.default_rng(0).standard_normal((1, 2, 3, 8)).astype(np.float16)
    p = str(tmp_path / "a.npy")
    save_tensor_file(p, a)
    assert np.array_equal(load_tensor_file(p).view(np.uint16), a.view(np.uint16))
    assert np.array_equal(np.load(p), a)  # our writer is a valid NPY v1.0 file
    np.save(p, a.astype(np.float32))
    assert np.array_equal(load_tensor_file(p), a)  # float32 -> float16 is exact here
    one = np.ones((1, 1, 1, 1), np.float32)
    np.save(p, one)
    assert load_tensor_file(p)[0, 0, 0, 0] == 1.0  # SPEC.md:457 minimal example


def test_npy_bf16_and_errors(tmp_path):
    p = str(tmp_path / "b.npy")
    x = np.array([1.0, -2.5, 3.140625, 65280.0], np.float32).reshape(1, 1, 1, 4)
    np.save(p, (x.view(np.uint32) >> 16).astype(np.uint16))  # bfloat16 bit patterns
    with pytest.raises(NpyFormatError, match="bf16"):
        load_tensor_file(p)
    assert np.array_equal(load_tensor_file(p, bf16=True), x.astype(np.float16))
    np.save(p, np.zeros((2, 3), np.float16))
    with pytest.raises(NpyFormatError, match="4-D"):
        load_tensor_file(p)
    np.save(p, np.zeros((1, 1, 1, 2), np.float64))
    with pytest.raises(NpyFormatError, match="unsupported dtype"):
        load_tensor_file(p)
    with open(p, "wb") as f:
        f.write(b"NOTNUMPY" + b"\0" * 16)
    with pytest.raises(NpyFormatError, match="bad magic at byte 0"):
        load_tensor_file(p)
    hdr = b"{'descr': '<f2', 'fortran_order': False, 'shape': (1, 1, 1, 4), }"
    with open(p, "wb") as f:
        f.write(b"\x93NUMPY\x01\x00" + struct.pack("<H", len(hdr)) + hdr + b"\0\0")
    with pytest.raises(NpyFormatError, match="payload truncated"):
        load_tensor_file(p)


# ----------------------------------------------------------------------------- reports
def _row(**kw):
    base = dict(policy="PASA_FP16", kind="hybrid", x0=30.0, am=10.0, p=0.001, seed=0, batch=1,
                heads=16, seq=1280, dim=128, beta=0.984497, rmse=0.0123456789012, nan_pct=0.0,
                wall_s=0.123456)
    base.update(kw)
    return ba.RunReport(**base)


def test_report_csv_schema():
    rows = [_row(), _row(policy="FA_PARTIAL_FP16", kind="uniform", rmse=math.nan, nan_pct=100.0),
            _row(has_ranges=True, s_min_before=-412.0, s_max_before=234.0, s_min_after=-12.54,
                 s_max_after=9.976)]
    lines = ba.report_csv(rows).splitlines()
    assert lines[0] == ("policy,kind,x0,Am,p,seed,B,N,S,d,beta,rmse,nan_pct,s_min_before,"
                        "s_max_before,s_min_after,s_max_after,wall_s")
    assert lines[1] == "PASA_FP16,hybrid,30,10,0.001,0,1,16,1280,128,0.984497,0.0123456789,0,,,,,0.1235"
    assert lines[2].startswith("FA_PARTIAL_FP16,uniform,30,10,,0,")  # p only for hybrid
    assert ",nan,100," in lines[2]
    assert lines[3].endswith(",-412,234,-12.54,9.976,0.1235")


def test_report_json_round_trip():
    rows = [_row(), _row(rmse=math.nan, error="boom"),
            _row(has_ranges=True, s_min_before=-1.0, s_max_before=2.0, s_min_after=-0.5,
                 s_max_after=0.25)]
    text = ba.report_json_rows(rows)
    arr = json.loads(text)
    assert arr[0]["N"] == 16 and arr[0]["Am"] == 10.0 and arr[0]["s_min_before"] is None
    assert arr[1]["rmse"] is None and arr[1]["error"] == "boom"
    assert list(arr[0]) == sorted(arr[0])  # nlohmann::json orders keys
    back = ba.runs_from_json(text)
    assert ba.report_csv(back) == ba.report_csv(rows)


def test_range_overflow_prediction():
    rep = ba.RangeReport()
    rep.total.s_before_min, rep.total.s_before_max = -6000.0, 10.0
    assert rep.overflow_predicted(11.3137)       # 6000 * 11.3 > 65504
    assert not rep.overflow_predicted(8.0)


# ----------------------------------------------------------------------------- CLI
def _cli(*args, cwd=ROOT):
    return subprocess.run([sys.executable, "-m", "paper_2503_01873_b200", *args],
                          capture_output=True, text=True, cwd=cwd)


def test_cli_solve_beta():
    r = _cli("solve-beta", "--beta0", "0.984375", "--n", "128")
    assert r.returncode == 0 and r.stdout.startswith("beta=0.984497 ")


def test_cli_report_and_config_errors(tmp_path):
    j = tmp_path / "r.json"
    j.write_text(json.dumps({"config": {}, "rows": json.loads(ba.report_json_rows([_row()]))}))
    r = _cli("report", "--json", str(j))
    assert r.returncode == 0 and r.stdout == ba.report_csv([_row()])
    r = _cli("sweep")  # no grid -> configuration error, exit 1
    assert r.returncode == 1 and "grid" in r.stderr
    r = _cli("sweep", "--preset", "nope")
    assert r.returncode == 1 and "unknown preset" in r.stderr


def test_reports_match_reference_text(ref):
    """Our report_csv is byte-identical to the reference's (bench.cpp:249-277); the JSON
    rows parse to the same objects in the same key order (bench.cpp:279-316)."""
    rows = [_row(), _row(policy="FA_PARTIAL_FP16", kind="uniform", rmse=math.nan, nan_pct=100.0,
                         error="cell failed"),
            _row(has_ranges=True, s_min_before=-412.0, s_max_before=234.0, s_min_after=-12.54,
                 s_max_after=9.976, x0=0.1, am=1e-7, rmse=3.0e-12, wall_s=1234.5678),
            _row(kind="uniform", x0=-20.0, am=15.0, seed=2**40 + 3, nan_pct=8.14, beta=0.9375)]
    assert ba.report_csv(rows) == ref.report(rows)
    assert ba.report_csv([]) == ref.report([])
    ours, theirs = json.loads(ba.report_json_rows(rows)), json.loads(ref.report(rows, json=True))
    assert ours == theirs
    assert [list(o) for o in ours] == [list(o) for o in theirs]


def test_shifting_matrix_inverse_theorem_2_1():
    """SPEC KAT (Theorem 2.1, pasa.cpp:37-51): (I - lambda J)^-1 = I + lambda/(1 - lambda s) J,
    singular exactly at lambda s = 1; the Python mirror and the C++ drop-in (shim_kat, linked
    against pasa_shim.o like the reference's harness) agree."""
    import os
    import subprocess
    from paper_2503_01873_b200 import SingularMatrixError, shifting_matrix_inverse
    s = 128
    for beta in (0.5, 0.9375, 0.984497):
        lam = beta / s
        m = np.eye(s) - lam * np.ones((s, s))
        assert np.abs(m @ shifting_matrix_inverse(s, lam) - np.eye(s)).max() < 1e-12
    with pytest.raises(SingularMatrixError):
        shifting_matrix_inverse(s, 1.0 / s)
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                       "shim_kat")
    if os.path.exists(exe):  # built where the reference's headers exist (build())
        r = subprocess.run([exe], capture_output=True, text=True, timeout=60)
        assert r.returncode == 0 and "KAT OK" in r.stdout, r.stdout + r.stderr


def test_recovery_relation():
    """SPEC KAT: with the FP64 shifting matrix M = I/alpha - beta J/(alpha s2),
    rowmean(S M) / (1 - beta) = rowmean(S) / alpha -- the shift removes exactly a beta fraction
    of each row's mean, which the global-recovering step puts back."""
    from paper_2503_01873_b200 import Prec, build_shifting_matrix
    rng = np.random.default_rng(7)
    for s2, beta, alpha in ((128, 0.984497, math.sqrt(128.0)), (64, 0.9375, 8.0), (128, 0.5, 1.0)):
        m = build_shifting_matrix(s2, beta, alpha, Prec.FP64)
        s = rng.normal(30.0, 5.0, (16, s2))
        lhs = (s @ m).mean(axis=1) / (1.0 - beta)
        rhs = s.mean(axis=1) / alpha
        assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max() * s2


def test_bench_reference_arm_passes_thread_count(monkeypatch):
    """The reference arm hands its thread count to pasa_attention explicitly
    (AttnOptions::threads, parallel.hpp:20-32): under torchrun OMP_NUM_THREADS=1 would
    otherwise pin the reference to one thread while the line reports every core."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench

    seen = {}

    class FakeRef:
        def pasa(self, pb, beta, policy, threads=0):
            seen["threads"] = threads
            return np.zeros(pb.q.shape)

    q = np.zeros((1, 1, 128, 128))
    monkeypatch.setenv("OMP_NUM_THREADS", "1")
    dt, _ = bench.time_reference_step(FakeRef(), q, q, q, 7)
    assert seen["threads"] == 7 and dt >= 0.0
