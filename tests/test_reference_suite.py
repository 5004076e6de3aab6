"""The reference's OWN unit tests (pkg/tests: test_modpoly.py, test_upoly.py,
test_bisolve.py -- copied next to the installed reference by build()) run with
the B200 engine installed: every curvekit name they import is the GPU
version (a conftest installs it before they bind the names), and at least one
of the engine's kernels must have run.  The strongest drop-in check there is:
the reference's own expectations, unmodified."""

import json
import os
import subprocess
import sys
import tempfile

import pytest

from conftest import reference_consumer

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# test_bisolve.py::test_known_x_oracle_suite solves 30 systems with ALL filters; the
# reference's pure-Python numeric filter (certified numerics, outside the path)
# takes more than 10 minutes for it on its own, engine or not.  The same 30
# systems are compared box for box under the combinatorial filter set in
# tests/test_bisolve_e2e.py.
DESELECT = {"test_bisolve.py": "not test_known_x_oracle_suite"}


@pytest.mark.parametrize("suite", ["test_modpoly.py", "test_upoly.py", "test_bisolve.py"])
def test_reference_unit_tests_pass_on_the_engine(suite, curvekit_mod):
    ref = reference_consumer()
    tests = os.path.join(ref, "ref_tests")
    if not os.path.exists(os.path.join(tests, suite)):
        pytest.fail("the reference's tests are not installed: run __graft_entry__.build() where /root/reference "
                    "exists (oracle.install_reference copies them next to the package)")
    with tempfile.TemporaryDirectory() as td:
        report = os.path.join(td, "report.json")
        env = dict(os.environ, CKB_REF_SUITE_REPORT=report, PYTHONPATH=ref)
        sel = ["-k", DESELECT[suite]] if suite in DESELECT else []
        r = subprocess.run([sys.executable, "-m", "pytest", suite, "-q", "-p", "no:cacheprovider", "-x", *sel],
                           cwd=tests, env=env, capture_output=True, text=True, timeout=1200)
        assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-2000:])
        with open(report) as fh:
            launches = json.load(fh)["launches"]
    assert launches > 0, "the reference's tests did not reach the GPU engine"
