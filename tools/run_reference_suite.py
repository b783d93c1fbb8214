"""The reference's own callers of the hot path, run on the B200 drop-in:

  1. its test suite for the path, pkg/tests/test_routing.py (37 tests), with moelab.routing
     served by paper_2603_07685_b200.routing (tools/moelab_b200_shim.py);
  2. its only product caller, the `moe-check` CLI entry (cli._moe_check, cli.py:269-308).

Needs the reference installed in baseline/_ref (pip --target) and its test
file copied next to it (baseline/_ref/reference_tests/, git-ignored). Exact tests (routing
maps, counts, permutation maps, capacity, padding, error messages) are expected to pass;
tests that assert fp64 identities at 1e-6 / 1e-8 measure the bf16 device path and are
reported with their measured error.

    python tools/run_reference_suite.py [--numpy]   (--numpy: the unmodified reference)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "reference_tests", "test_routing.py")


def main():
    numpy_only = "--numpy" in sys.argv
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tools")]),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", TESTS, "-q", "-rA", "--tb=line", "-p",
           "no:cacheprovider"]
    if not numpy_only:
        cmd += ["-p", "moelab_b200_shim"]
    print("$", " ".join(cmd), flush=True)
    r = subprocess.run(cmd, env=env, cwd="/tmp", capture_output=True, text=True)
    print(r.stdout[-20000:])
    print(r.stderr[-3000:])
    # the moe-check CLI entry on the same backend
    code = ("import json, sys; sys.path[:0] = %r; " % [REF, ROOT, os.path.join(ROOT, "tools")]
            + ("" if numpy_only else "import moelab_b200_shim; moelab_b200_shim.install(); ")
            + "from moelab import cli; print(json.dumps(cli._moe_check(0, 50)))")
    r2 = subprocess.run([sys.executable, "-c", code], env=env, cwd="/tmp", capture_output=True,
                        text=True)
    print("moe-check (seed 0, 50 instances):", r2.stdout.strip(), r2.stderr[-2000:])


if __name__ == "__main__":
    main()
