"""The reference's own code, run unmodified against the drop-in (VERDICT r1
#7, SURVEY §8(b) "Callers"): the vendored roboserve package's test suite and
its scratch_fig4.py script (configs[0]), with the hot-path names routed to the
CUDA path by tests/ref_swap.py.  Skipped when baseline/_ref has not been
vendored (tools/vendor_reference.sh)."""

from __future__ import annotations

import contextlib
import io
import json
import os
import runpy
import subprocess
import sys
from pathlib import Path

import pytest

import ref_swap

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_swap.available(),
                                 reason="baseline/_ref not vendored (tools/vendor_reference.sh)")]

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden" / "fig4.json"


def test_scratch_fig4_script_with_dropin_plan():
    """scratch_fig4.py (scratch_fig4.py:97-159) unmodified, its `plan` and
    state types served by the drop-in: the printed orders and total waits
    equal the reference run's stdout (tests/golden/fig4.json)."""
    swapped = ref_swap.install()
    assert "scheduler.plan" in swapped and "core.TaskState" in swapped
    import roboserve.scheduler
    import paper_2605_11381_b200 as kb
    assert roboserve.scheduler.plan is kb.plan
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        runpy.run_path(str(ref_swap.REF / "pkg" / "scratch_fig4.py"), run_name="__main__")
    assert buf.getvalue() == json.loads(GOLD.read_text())["stdout"]


def test_reference_test_suite_against_dropin():
    """The reference's pytest suite (pkg/tests, 132 tests) with every hot-path
    name it imports served by the drop-in."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(ROOT / "tests"), str(ref_swap.REF), str(ROOT),
                                         env.get("PYTHONPATH", "")])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "ref_swap", "-p",
                        "no:cacheprovider", "--rootdir", str(ref_swap.REF / "pkg"), "-c",
                        os.devnull, str(ref_swap.REF / "pkg" / "tests")],
                       capture_output=True, text=True, env=env, timeout=1200)
    tail = r.stdout[-3000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
