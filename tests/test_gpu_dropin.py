"""The C++ drop-in headers (include/embdispatch/) compiled against libedx.so:
code written to the reference's API runs unchanged and matches the oracle."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def test_cpp_dropin_matches_oracle():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    r = subprocess.run([os.path.join(HERE, "dropin_test")], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "OK" in r.stdout
