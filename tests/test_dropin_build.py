"""CPU check: the drop-in headers compile against include/edx.h (no GPU)."""
import os
import subprocess

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp")


def test_cpp_dropin_compiles():
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    assert os.path.exists(os.path.join(HERE, "dropin_test"))


def test_report_formats_match_reference():
    """report_io.hpp drop-in (JSON lines, comparison CSV) byte-identical to the
    compiled reference's on randomized RunResults (host formatting only)."""
    ref = os.path.join(os.path.dirname(HERE), "..", "oracle", "_ref", "libedx_ref.so")
    ref = os.path.abspath(ref)
    if not os.path.exists(ref):
        import pytest
        pytest.skip("oracle/_ref not built (reference sources absent)")
    subprocess.run(["make", "-s", "-C", HERE, "report_test"], check=True)
    r = subprocess.run([os.path.join(HERE, "report_test"), ref], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "OK" in r.stdout


def test_trace_stream_dropin():
    """TraceStream / load_schema / write_trace through the drop-in C++ headers:
    the reference's trace tests (test_workload.cpp:179-281), host only."""
    subprocess.run(["make", "-s", "-C", HERE, "trace_test"], check=True)
    r = subprocess.run([os.path.join(HERE, "trace_test")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "OK" in r.stdout
