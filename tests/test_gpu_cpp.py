"""C++ programs against the drop-in mpic:: API (tests/cpp/*.cpp), run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin")


@pytest.mark.parametrize("prog", ["test_weight_edit"])
def test_cpp_program(prog):
    path = os.path.join(BIN, prog)
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", os.path.dirname(BIN)], check=True)
    r = subprocess.run([path], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
