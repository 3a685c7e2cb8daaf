"""The C++ host API (include/latch_b200.hpp: namespace latch over the C ABI) against the
oracle and the golden fixtures — tests/cpp/test_latch_host.cpp, built by build()."""
import subprocess

import pytest

from conftest import ROOT

BIN = ROOT / "tests" / "cpp" / "test_latch_host"


def _build():
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "liblatch_oracle.so"], check=True,
                   stdout=subprocess.DEVNULL)
    subprocess.run(["make", "-C", str(BIN.parent)], check=True, stdout=subprocess.DEVNULL)
    from paper_1609_03986_b200.pattern import ensure_default_pattern_file
    ensure_default_pattern_file()


@pytest.mark.gpu
def test_cpp_host_api_parity():
    _build()
    r = subprocess.run([str(BIN), str(ROOT)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "PASSED" in r.stdout


def test_cpp_host_api_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    _build()
    r = subprocess.run([str(BIN), str(ROOT)], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0
    assert "DeviceUnavailable" in r.stderr and "no CPU fallback" in r.stderr
