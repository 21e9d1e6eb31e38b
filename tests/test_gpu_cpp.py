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
def test_cpp_dropin_suite():
    from paper_1101_0395_b200 import _build
    _build.build()
    r = subprocess.run([_build.CPP_TEST_BIN, os.path.join(ROOT, "tests", "golden")],
                       capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
