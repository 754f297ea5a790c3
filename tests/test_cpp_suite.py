"""Runs the C++ ports of the reference test suites (tests/cpp) against libtlsph.so.1 on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)


def test_cpp_suites_compile():
    _build()  # host-only: the C++ operator API headers and libtlsph.so.1 link


@pytest.mark.gpu
@pytest.mark.parametrize("binary", ["test_operator_api", "test_capi"])
def test_cpp_suite(binary):
    _build()
    out = subprocess.run([os.path.join(ROOT, "build", "tests", binary)], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


def test_config_and_output_writers_host_only():
    """tests/cpp/test_config.cpp: parse_config messages and kinds, probe CSV / report.json bytes (no device)."""
    _build()
    out = subprocess.run([os.path.join(ROOT, "build", "tests", "test_config")], capture_output=True, text=True,
                         timeout=120)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
