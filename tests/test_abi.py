"""C-ABI library: loads, exports every symbol include/eclip.h declares, parses the SPEC
profile format exactly, validates, and refuses to plan without a GPU (no CPU fallback).
CPU only (no compute calls)."""
import os
import re

import numpy as np
import pytest

import oracle
import synth
import paper_2506_12598_b200 as ec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "eclip.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(eclip_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = ec.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(ec.EXPORTS)
    assert b"sm_100a" in L.eclip_version()


def test_profiles_roundtrip_exact():
    ms = synth.library_models()
    txt = synth.write_profile_text(ms)
    pr = ec.Profiles.from_text(txt)
    info = pr.info()
    assert info["n_models"] == 7 and info["sizes"] == ms[0].sizes
    assert np.array_equal(info["exec_ns"], np.concatenate([m.exec_ns for m in ms]))
    assert info["names"] == [m.name for m in ms]
    # file path variant
    p = os.path.join(os.environ.get("TMPDIR", "/tmp"), "eclip_prof_test.txt")
    open(p, "w").write(txt)
    assert np.array_equal(ec.Profiles.from_file(p).info()["exec_ns"], info["exec_ns"])
    # from arrays
    pa = ec.Profiles.from_models(ms)
    assert np.array_equal(pa.info()["exec_ns"], info["exec_ns"])


def test_decimal_rounding_matches_oracle_parser():
    """no precision lost beyond 1 ns; ties to even."""
    rng = np.random.default_rng(5)
    cells = ["0.0005", "0.0015", "0.0025", "12.3456", "7.0004999", "7.00050001", "19.8", "3", "3.", ".5"]
    cells += [f"{rng.integers(1, 10**6)}.{rng.integers(0, 10**7):07d}" for _ in range(200)]
    for c in cells:
        v = oracle.us_to_ns(c)
        if v <= 0:
            continue
        txt = '{"model": "m", "kernels": 1, "configs": [1]}\n0, ' + c + "\n"
        got = int(ec.Profiles.from_text(txt).info()["exec_ns"][0, 0])
        assert got == v, c


@pytest.mark.parametrize("bad,code,msg", [
    ("not json\n", ec.eclip.E_PARSE, "parse failure"),
    ('{"model": "m", "kernels": 2, "configs": [15, 30]}\n0, 2, 1\n1, 2\n', ec.eclip.E_MISSING_CONFIG, "kernel 1"),
    ('{"model": "m", "kernels": 2, "configs": [15, 30]}\n0, 2, 1\n1, 2, 3\n', ec.eclip.E_NONMONOTONE, "kernel 1"),
    ('{"model": "m", "kernels": 1, "configs": [15, 30]}\n0, 2, 0\n', ec.eclip.E_NONMONOTONE, "non-positive"),
    ('{"model": "m", "kernels": 1, "configs": [15, 30]}\n0, 2, x\n', ec.eclip.E_PARSE, "not a decimal"),
    ('{"model": "m", "kernels": 3, "configs": [15, 30]}\n0, 2, 1\n', ec.eclip.E_PARSE, "expected 3"),
])
def test_profile_errors(bad, code, msg):
    with pytest.raises(ec.EclipError, match=msg) as ei:
        ec.Profiles.from_text(bad)
    assert ei.value.code == code


def test_missing_file_is_io_error():
    with pytest.raises(ec.EclipError) as ei:
        ec.Profiles.from_file("/nonexistent/profile.txt")
    assert ei.value.code == ec.eclip.E_IO


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    p = synth.make_c1()
    pr = ec.Profiles.from_models(p.models)
    with pytest.raises(ec.EclipError) as ei:
        ec.plan_problem(pr, p)
    assert ei.value.code == ec.eclip.E_CUDA
    with pytest.raises(ec.EclipError) as ei:
        ec.plan_batch(pr, np.zeros((2, 2), np.int32), total_sms=60)
    assert ei.value.code == ec.eclip.E_CUDA


def test_argument_validation_precedes_device():
    """invalid problems are rejected before any device work (error, not a fallback)"""
    p = synth.make_c1()
    pr = ec.Profiles.from_models(p.models)
    with pytest.raises(ec.EclipError) as ei:
        ec.plan(pr, [0, 5], total_sms=60)
    assert ei.value.code == ec.eclip.E_INVALID_ARG
    with pytest.raises(ec.EclipError) as ei:
        ec.plan(pr, [0, 1], total_sms=50)          # size 60 > N
    assert ei.value.code == ec.eclip.E_INVALID_ARG
    with pytest.raises(ec.EclipError) as ei:
        ec.plan(pr, [0, 1], total_sms=60, switch_max=-1)
    assert ei.value.code == ec.eclip.E_INVALID_ARG
    with pytest.raises(ec.EclipError) as ei:
        ec.plan(pr, [0, 1], total_sms=60, slowdown="matrix")
    assert ei.value.code == ec.eclip.E_INVALID_ARG
    with pytest.raises(ec.EclipError) as ei:
        ec.plan(pr, [0, 1], total_sms=60, allowed_mask=[0, 1])
    assert ei.value.code == ec.eclip.E_INVALID_ARG
