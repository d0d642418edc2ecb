"""Copy the reference's own hot-path tests next to the drop-in, behind a `bittrain` alias.

    python tools/vendor_reference_tests.py      (also run by __graft_entry__.build())

The reference (`/root/reference/pkg/tests`) is read-only here and absent on the GPU boxes, so its
test modules for the path (★ rows) are copied UNMODIFIED into `tests/_reference/`
-- a git-ignored directory (test infrastructure, never part of the package or the history) that
travels to the GPU box with the working tree -- together with a conftest that maps `bittrain` and
its submodules onto `paper_2208_14228_b200`.  `tests/test_gpu_reference_suite.py` runs them on
the GPU.  Out-of-scope suites (planner, scheduler, simulator, CLI, configio, and the acceptance
suite, which imports all of them at module level) are not copied.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = Path("/root/reference/pkg/tests")
DST = ROOT / "tests" / "_reference"
SUITES = ["test_prng.py", "test_reduction.py", "test_model.py", "test_buckets.py", "test_sampling.py",
          "test_engine.py", "test_checkpoint.py", "test_scenarios.py", "test_runlog.py"]
MODULES = ["engine", "checkpoint", "scenarios", "model", "buckets", "reduction", "prng", "sampling", "runlog",
           "errors", "configio"]

CONFTEST = '''"""`bittrain` -> paper_2208_14228_b200 (the drop-in), for the reference's own tests."""
import importlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2208_14228_b200 as _pkg  # noqa: E402

sys.modules["bittrain"] = _pkg
for _name in {modules!r}:
    sys.modules["bittrain." + _name] = importlib.import_module("paper_2208_14228_b200." + _name)
'''


def vendor() -> bool:
    if not SRC.is_dir():
        return False
    DST.mkdir(parents=True, exist_ok=True)
    for name in SUITES:
        shutil.copyfile(SRC / name, DST / name)
    (DST / "conftest.py").write_text(CONFTEST.format(modules=MODULES))
    (DST / "__init__.py").write_text("")
    return True


if __name__ == "__main__":
    ok = vendor()
    print(f"vendored into {DST}" if ok else f"{SRC} not present: nothing to do")
    sys.exit(0)
