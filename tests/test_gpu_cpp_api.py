"""GPU: the C++ mirror of the reference API (include/double_b200.hpp) — reference datastore and
pipeline unit cases restated in C++ (tests/cpp/test_cpp_api.cpp) against libdouble_b200.so."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_api_program():
    from paper_2601_05524_b200.build import CPP_TEST, build_cpp_test
    build_cpp_test()  # always: a stale binary would pass old struct layouts across the C-ABI
    r = subprocess.run([CPP_TEST], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
