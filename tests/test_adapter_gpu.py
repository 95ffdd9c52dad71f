"""The C++ drop-in adapter (include/dosegpu/ddm_adapter.hpp) driven by the reference's own
types, generator and CPU engines: oracle/_ref/adapter_test (tests/cpp/adapter_test.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


@pytest.mark.gpu
def test_cpp_adapter_matches_reference_engines():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_test not built (make -C oracle adapter)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_cpp_adapter_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_test not built")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "NoDevice" in (r.stdout + r.stderr)
