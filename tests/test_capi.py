"""CPU tests of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/pasa_b200.h declares, and validates arguments
with the reference's rules and messages (tensor.cpp:19-55, pasa.cpp:200-211).
No compute entry point is called here."""
import ctypes as C
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2503_01873_b200 import _lib
from paper_2503_01873_b200.api import BETA_STAR, PasaParams, build_shifting_matrix

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol(lib):
    declared = _lib.exported_symbols_from_header()
    assert len(declared) >= 10
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.SO], capture_output=True, text=True,
                        check=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(lib, s)
    # nothing else leaks out of the library
    assert {s for s in exported if s.startswith("pasa_b200")} == set(declared)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.SO], capture_output=True, text=True).stdout
    archs = {ln.split(".")[-2] for ln in out.splitlines() if ".cubin" in ln}
    assert archs == {"sm_100a"}, archs


def _desc(**kw):
    base = dict(batch=1, heads_q=2, heads_kv=2, seq_q=1024, seq_kv=1024, head_dim=128, s1=128,
                s2=128, causal=0, layout=0, beta=BETA_STAR, alpha=math.sqrt(128.0))
    base.update(kw)
    return _lib.Desc(**base)


def _check(lib, **kw):
    d = _desc(**kw)
    rc = lib.pasa_b200_check(C.byref(d))
    return rc, lib.pasa_b200_last_error().decode()


def test_check_accepts_config1_and_qwen(lib):
    assert _check(lib)[0] == 0
    assert _check(lib, beta=0.0)[0] == 0  # beta == 0: the FP16 FA mode (pasa.cpp:212-221)
    # ragged: short KV block (SVD temporal N = 25) and S1 not a multiple of 128
    assert _check(lib, seq_q=25, seq_kv=25, s1=25, s2=25, head_dim=64, alpha=8.0)[0] == 0
    assert _check(lib, seq_q=200, seq_kv=256, s1=200, s2=64)[0] == 0
    assert _check(lib, heads_q=28, heads_kv=4, seq_q=16384, seq_kv=16384, causal=1)[0] == 0
    assert _check(lib, seq_q=512, seq_kv=1024, causal=1)[0] == 0  # bottom-right aligned
    assert _check(lib, seq_q=256, seq_kv=320, s2=64, causal=1)[0] == 0  # causal, short KV blocks
    assert _check(lib, head_dim=64, alpha=8.0)[0] == 0


@pytest.mark.parametrize("kw,code,msg", [
    (dict(seq_q=1000), _lib.EINVAL, "multiples of the block sizes"),
    (dict(heads_kv=3), _lib.EINVAL, "K heads must divide Q heads"),
    (dict(alpha=11.0), _lib.EINVAL, "alpha does not match sqrt(d)"),
    (dict(beta=1.0), _lib.EINVAL, "beta must lie in [0, 1)"),
    (dict(beta=-0.1), _lib.EINVAL, "beta must lie in [0, 1)"),
    (dict(batch=0), _lib.EINVAL, "empty query tensor"),
    (dict(head_dim=96, alpha=math.sqrt(96.0)), _lib.EUNSUPPORTED, "head_dim"),
    (dict(s2=256, s1=256), _lib.EUNSUPPORTED, "s2 must be <= 128"),
    (dict(causal=1, seq_q=1024, seq_kv=512), _lib.EUNSUPPORTED, "causal requires S1 <= S2"),
    (dict(layout=2), _lib.EINVAL, "layout must be 0 (BHSD) or 1 (BSHD)"),
])
def test_check_rejects(lib, kw, code, msg):
    rc, err = _check(lib, **kw)
    assert rc == code and msg in err, (rc, err)


def test_check_accepts_bshd(lib):
    assert _check(lib, layout=1)[0] == 0
    assert _check(lib, layout=1, heads_q=28, heads_kv=4, seq_q=16384, seq_kv=16384, causal=1)[0] == 0


def test_host_multi_argument_errors(lib):
    """pasa_b200_attention_host_multi validates before touching a device (CPU test)."""
    buf = (C.c_uint16 * 8)()
    devs = (C.c_int32 * 2)(0, 1)
    d = _desc(layout=1)
    assert lib.pasa_b200_attention_host_multi(C.byref(d), buf, buf, buf, buf, devs, 2) == \
        _lib.EUNSUPPORTED
    assert "BHSD only" in lib.pasa_b200_last_error().decode()
    d = _desc()
    assert lib.pasa_b200_attention_host_multi(C.byref(d), buf, buf, buf, buf, devs, 0) == _lib.EINVAL


def test_errors_map_to_reference_exception_types(lib):
    with pytest.raises(ValueError, match="alpha does not match"):
        _lib.check(lib.pasa_b200_check(C.byref(_desc(alpha=2.0))))
    with pytest.raises(_lib.PasaError):
        _lib.check(lib.pasa_b200_check(C.byref(_desc(s2=256, s1=256))))


def test_workspace_size(lib):
    d = _desc(heads_q=28, heads_kv=4, seq_q=16384, seq_kv=16384)
    n = lib.pasa_b200_workspace_size(C.byref(d))
    assert n >= 4 * 16384 * 128 * 2 + 4 * 4


def test_shift_entries_match_oracle(orc):
    for s2, beta, d in [(128, BETA_STAR, 128), (128, 0.9375, 64), (64, 0.5, 32), (128, 0.0, 128)]:
        m = build_shifting_matrix(s2, beta, math.sqrt(d))
        diag, off = orc.shift_entries(s2, beta, math.sqrt(d))
        assert m[0, 0] == diag and (s2 == 1 or m[0, 1] == off)
        assert np.all(np.diag(m) == diag)


def test_params_validation():
    with pytest.raises(ValueError, match="beta must lie"):
        PasaParams.make(128, 1.0, 11.3)
    p = PasaParams.make(128, BETA_STAR, math.sqrt(128.0))
    assert p.m.shape == (128, 128)


def test_integration_shim_links_reference_harness():
    """integration/ref_sweep_b200 = reference objects + our pasa_shim.o (no pasa.o)."""
    exe = os.path.join(ROOT, "integration", "_build", "ref_sweep_b200")
    if not os.path.exists(exe):
        pytest.skip("integration binary not built (needs /root/reference)")
    nm = subprocess.run(["nm", "-C", exe], capture_output=True, text=True).stdout
    assert "pasa::sweep" in nm and "pasa::pasa_attention" in nm
    assert "pasa::OnlineState::absorb" not in nm  # the reference PASA core is not linked in


def test_no_cpu_fallback_without_a_gpu(lib):
    """On a machine without an sm_100 device every compute entry point fails loudly
    (there is no CPU fallback); this container has no GPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2503_01873_b200.api import PasaParams, make_problem, pasa_attention
    d = _desc(seq_q=128, seq_kv=128)
    buf = (C.c_uint16 * (2 * 128 * 128))()
    rc = lib.pasa_b200_attention_host(C.byref(d), buf, buf, buf, buf)
    assert rc in (_lib.ENODEV, _lib.ECUDA) and lib.pasa_b200_last_error()
    q = torch.zeros(1, 2, 128, 128, dtype=torch.float16)
    pb = make_problem(q, q, q, 128, 128)
    with pytest.raises(_lib.PasaError):
        pasa_attention(pb, PasaParams.make(128, BETA_STAR, pb.alpha))
    from paper_2503_01873_b200 import pasa_attention_fwd
    with pytest.raises(ValueError, match="CUDA tensors"):
        pasa_attention_fwd(q, q, q)


def test_attention_fwd_tiles_range_errors(lib):
    """pasa_b200_attention_fwd_tiles validates its query-tile range before any device work."""
    d = _lib.Desc(1, 2, 2, 1000, 1000, 128, 100, 100, 1, 0, 0.984497, math.sqrt(128.0))
    ws_bytes = lib.pasa_b200_workspace_size(C.byref(d))
    buf = C.c_void_p(16)  # never dereferenced: the range check comes first
    for t0, n in [(-1, 2), (0, 9), (8, 1), (3, -1)]:
        rc = lib.pasa_b200_attention_fwd_tiles(C.byref(d), buf, buf, buf, buf, buf, ws_bytes, t0, n, None)
        assert rc == _lib.EINVAL, (t0, n)
        assert b"tile range" in lib.pasa_b200_last_error()
