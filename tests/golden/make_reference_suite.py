"""Golden results of the reference's OWN unit tests built against the
reference headers (tests/cpp/Makefile `reftests_ref`, same Catch2 stand-in):
the failing checks and the counts, so tests/test_reference_suite.py can check
the drop-in fails exactly where the reference itself fails even on a host
without the reference binaries.  Run here: python tests/golden/make_reference_suite.py"""
import json
import os
import re
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(os.path.dirname(HERE), "cpp")
SUITES = ["core", "cache", "cost", "assign", "sim", "workload", "config", "experiment"]


def summarize(out):
    m = re.search(r"(\d+) test cases, (\d+) failed; (\d+) checks, (\d+) failed", out)
    failed = re.findall(r"^FAILED (.+?) \[(.*)\]\n  (.*)$", out, re.M)
    # a failure's location is the reference test file:line; drop the path prefix
    norm = [(os.path.basename(f), name, what) for f, name, what in failed]
    return {"cases": int(m.group(1)), "failed_cases": int(m.group(2)),
            "checks": int(m.group(3)), "failed_checks": int(m.group(4)),
            "failures": [list(x) for x in norm]}


if __name__ == "__main__":
    subprocess.run(["make", "-s", "-C", CPP, "reftests_ref"], check=True)
    res = {}
    for s in SUITES:
        r = subprocess.run([os.path.join(CPP, "reftests_ref", f"test_{s}")], capture_output=True,
                           text=True, timeout=1800)
        res[f"test_{s}"] = summarize(r.stdout + r.stderr)
    with open(os.path.join(HERE, "reference_suite.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))
