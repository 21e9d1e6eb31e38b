"""CPU-side checks of the C-ABI library and the host mirror (no GPU needed):
the library loads, exports every entry point include/cqg.h declares, fails
loudly without a device, and the pure-host parts of the quant mirror keep the
reference's frozen formats and messages."""
import math
import os
import re

import numpy as np
import pytest

from paper_1101_0395_b200 import cabi, quant

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    with open(os.path.join(ROOT, "include", "cqg.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(cqg_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1101_0395_b200 import _build
    _build.build()
    L = cabi.load()
    declared = header_functions()
    assert set(declared) == set(cabi.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.cqg_version().startswith(b"cqg")


def test_create_fails_loudly_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(cabi.CqgError):
        cabi.Context(0)


def test_sass_contains_packed_fp32_sweep():
    """The sweep is FFMA2 (packed FP32 FMA chains) + 3-input FMNMX3 on sm_100a."""
    import subprocess
    so = os.path.join(ROOT, "paper_1101_0395_b200", "libcqg.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper() or "arch = sm_100a" in out
    assert "FFMA2" in out and "FMNMX3" in out


# ---- host mirror: frozen formats (tests/test_metrics.cpp:94-162) -------------

def test_report_csv_frozen():
    assert quant.QuantReport.csv_header() == (
        "image,method,k,run,seed,sampling,mse,psnr,iterations,ndc_per_point_iter,time_ms,"
        "actual_k,flags")
    r = quant.QuantReport(image="img.ppm", method="wsm-wu", k_requested=32, k_actual=32, run=2,
                          seed=3, sampling="unique", mse=71.25, psnr=29.603, iterations=14,
                          ndc_per_point_iter=3.9812, time_ms=12.5,
                          flags=["repairs:1", "padded_init"])
    assert r.csv_row() == ("img.ppm,wsm-wu,32,2,3,unique,71.250000,29.6030,14,3.9812,12.500,32,"
                           "repairs:1;padded_init")
    r.mse = float("nan")
    r.psnr = float("nan")
    r.flags = ["error:boom"]
    assert r.csv_row() == "img.ppm,wsm-wu,32,2,3,unique,nan,nan,14,3.9812,12.500,32,error:boom"


def test_psnr_and_mse():
    assert quant.psnr_from_mse(65025.0) == pytest.approx(0.0, abs=1e-12)
    assert quant.psnr_from_mse(100.0) == pytest.approx(28.1308, rel=1e-3)
    assert math.isinf(quant.psnr_from_mse(0.0))
    with pytest.raises(ValueError):
        quant.psnr_from_mse(-1.0)
    a = np.array([[[0, 0, 0]]], np.uint8)
    b = np.array([[[3, 4, 0]]], np.uint8)
    assert quant.mse(a, b) == 25.0


def test_channel_to_u8_rounds_half_up():
    assert quant.channel_to_u8(0.5) == 1
    assert quant.channel_to_u8(-3.0) == 0
    assert quant.channel_to_u8(300.0) == 255
    assert quant.channel_to_u8(254.49) == 254


def test_method_tokens():
    # tests/test_pipeline.cpp:37-71
    s = quant.parse_method("wu")
    assert not s.refine and s.token() == "wu"
    s = quant.parse_method("wsm-kpp")
    assert s.refine and s.base == "kpp"
    assert quant.parse_method("wsm").base == "fgy"
    assert quant.parse_method("wsm", "lbg").base == "lbg"
    for bad in [("wsm-xyz", ""), ("xyz", ""), ("mc", "fgy")]:
        with pytest.raises(ValueError):
            quant.parse_method(*bad)
    assert quant.all_method_tokens() == [
        "mc", "ott", "oct", "wan", "wu", "bs", "wsm-fgy", "wsm-lbg", "wsm-mmx", "wsm-den",
        "wsm-var", "wsm-sff", "wsm-kpp", "wsm-mc", "wsm-ott", "wsm-oct", "wsm-wan", "wsm-wu",
        "wsm-bs"]


def test_sampling_tokens():
    for t in ("none", "2to1", "unique", "both"):
        assert quant.parse_sampling_mode(t) == t
    with pytest.raises(ValueError):
        quant.parse_sampling_mode("fancy")


def test_convergence_rule():
    # tests/test_kmeans.cpp:239-244
    assert not quant.check_convergence(100.0, 99.9, 0.001)
    assert quant.check_convergence(100.0, 99.95, 0.001)
    assert quant.check_convergence(5.0, 0.0, 0.001)
    assert quant.check_convergence(7.0, 7.0, 0.0)


def test_wsm_validation_messages_before_device():
    pts = np.array([[0, 0, 0], [1, 1, 1]], float)
    w = np.array([0.5, 0.5])
    one = np.array([[0, 0, 0]], float)
    three = np.array([[0, 0, 0], [1, 1, 1], [2, 2, 2]], float)
    with pytest.raises(ValueError, match="no initial centers"):
        quant.wsm(pts, w, np.zeros((0, 3)))
    with pytest.raises(ValueError, match=r"k \(3\) exceeds number of points \(2\)"):
        quant.wsm(pts, w, three)
    with pytest.raises(ValueError, match="size mismatch"):
        quant.wsm(pts, np.array([0.5]), one)
    with pytest.raises(ValueError, match="weights must be positive"):
        quant.wsm(pts, np.array([0.5, -0.5]), one)
    bad = quant.ClusterOptions(quant.Termination(fixed_iterations=0))
    with pytest.raises(ValueError, match="fixed_iterations"):
        quant.wsm_counts(np.array([1, 2], np.uint32), np.array([1, 1], np.uint32), 2, one, bad)


# ---- PPM I/O on the host (image.hpp:26-44) -----------------------------------

def test_ppm_roundtrip_and_errors(tmp_path):
    from paper_1101_0395_b200 import quant
    rng = np.random.default_rng(3)
    img = quant.RawImage(5, 3, rng.integers(0, 256, (3, 5, 3), dtype=np.uint8))
    p = str(tmp_path / "a.ppm")
    quant.save_image(img, p)
    raw = open(p, "rb").read()
    assert raw[:11] == b"P6\n5 3\n255\n" and len(raw) == 11 + 45
    back = quant.load_image(p)
    assert back.width == 5 and back.height == 3 and np.array_equal(back.pixels, img.pixels)
    # comments between tokens; error messages of the reference (image.cpp)
    q = str(tmp_path / "b.ppm")
    open(q, "wb").write(b"P6 # note\n2 1\n255\n" + bytes(range(6)))
    assert np.array_equal(quant.load_image(q).pixels.reshape(-1), np.arange(6, dtype=np.uint8))
    cases = {b"P6\n2 1\n255\nab": "truncated PPM pixel data (expected 6 bytes, got 2)",
             b"P6\n2 x\n255\n": "malformed PPM height 'x'",
             b"P6\n2 1\n65535\n": "unsupported PPM maxval 65535 (only 255)",
             b"P6\n0 1\n255\n": "non-positive PPM dimensions",
             b"P6\n2": "truncated PPM header (missing height)",
             b"P3\n": "unsupported format (expected binary PPM 'P6' or PNG)",
             b"P": "file too short to identify"}
    for data, msg in cases.items():
        open(q, "wb").write(data)
        with pytest.raises(RuntimeError) as ei:
            quant.load_image(q)
        assert str(ei.value) == f"{q}: {msg}"
    with pytest.raises(RuntimeError, match="unknown output extension"):
        quant.save_image(img, str(tmp_path / "a.bmp"))
