"""The reference's own hot-path tests (pkg/tests: prng, reduction, model, buckets, sampling, engine,
checkpoint, scenarios, runlog) run UNMODIFIED against the drop-in on the GPU.

tools/vendor_reference_tests.py (run by __graft_entry__.build()) copies them into the git-ignored
tests/_reference/ with a conftest that aliases `bittrain` to paper_2208_14228_b200; this test runs
that directory in a child pytest and requires every test to pass except the two that import the
out-of-scope planner (test_checkpoint.py:223-262, `bittrain.planner`).
"""

import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
SUITE = ROOT / "tests" / "_reference"
OUT_OF_SCOPE = {  # import bittrain.planner (out of scope)
    "test_checkpoint.py::test_reconfigure_follows_planner_output",
    "test_checkpoint.py::test_reconfigure_rejects_infeasible_plan",
}


def test_reference_suite_passes_on_the_drop_in():
    if not (SUITE / "conftest.py").exists():
        pytest.skip("reference tests not vendored here (tools/vendor_reference_tests.py needs /root/reference)")
    out = subprocess.run([sys.executable, "-m", "pytest", str(SUITE), "-q", "-rf", "-p", "no:cacheprovider",
                          "--confcutdir", str(SUITE), "-o", "addopts="], cwd=ROOT, capture_output=True, text=True,
                         timeout=1800)
    log = out.stdout + out.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite.log").write_text(log)
    failed = {m.group(1).split("/")[-1] for m in re.finditer(r"^FAILED (\S+)", log, re.M)}
    failed = {f.split(" ")[0] for f in failed}
    m = re.search(r"(\d+) passed", log)
    assert m and int(m.group(1)) > 100, log[-3000:]
    assert failed <= OUT_OF_SCOPE, sorted(failed - OUT_OF_SCOPE)
