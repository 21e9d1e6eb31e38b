"""The reference-style C++ checks (tests/cpp/test_dropin.cpp) against the
C++ quant:: drop-in library (libquant_b200.so over libcqg.so)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_binary_builds():
    from paper_1101_0395_b200 import _build
    _build.build()
    assert os.path.exists(_build.HOST_LIB) and os.path.exists(_build.CPP_TEST_BIN)


@pytest.mark.gpu
def test_cpp_dropin_suite(tmp_path, reflib):
    from paper_1101_0395_b200 import _build
    _build.build()
    csv = tmp_path / "sweep.csv"
    r = subprocess.run([_build.CPP_TEST_BIN, os.path.join(ROOT, "tests", "golden"), str(csv)],
                       capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
    # the sweep's device rows equal the reference run_quantize's rows byte for
    # byte (zero_time; reference bench.cpp:55-90 builds them the same way)
    rows = csv.read_text().strip().split("\n")[1:]
    import numpy as np
    want = []
    for img_seed in (61, 62):
        img = np.fromfile(os.path.join(ROOT, "tests", "golden", f"acc_{img_seed}.rgb"), np.uint8).reshape(40, 40, 3)
        for method in ("wsm-kpp", "wsm-mmx"):
            for k in (4, 8):
                for run in (0, 1):
                    want.append(reflib.run_quantize(img, 40, 40, method, k, 3 + run, name=f"acc_{img_seed}.ppm",
                                                    run=run)["csv_row"])
    got = [row for row in rows if ",wu," not in row]
    assert got == sorted(want)
    assert sum(",wu," in row and "error:" in row for row in rows) == 8
