"""CPU check: the drop-in headers compile against include/edx.h (no GPU)."""
import os
import subprocess

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def test_cpp_dropin_compiles():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    assert os.path.exists(os.path.join(HERE, "dropin_test"))
