"""The reference's own test files (test_core, test_assembly, test_transport,
test_repart, test_update, test_solver, test_acceptance), unmodified, run
against the drop-in through an ``import ldurepart`` alias (tools/ref_suite.py).
Needs the staged copy of the reference tests (``tools/ref_suite.py --stage``
in the build container; it travels with the repo snapshot)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGE = os.path.join(ROOT, "baseline", "_ref_tests")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.isdir(STAGE) or
                    not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "ldurepart")),
                    reason="reference tests / package not staged (tools/ref_suite.py --stage)")
def test_reference_suite_passes_against_drop_in():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_suite.py"), "-q",
                          "-p", "no:randomly"], cwd=ROOT, capture_output=True, text=True,
                         timeout=1200)
    tail = "\n".join(res.stdout.splitlines()[-15:])
    assert res.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
