"""The reference package's own test suite run against this package (SURVEY.md
§4's reuse plan): ``oracle/ref_suite/fetch.sh`` copies /root/reference/pkg/tests
into the git-ignored ``oracle/_ref/pkg_tests`` (test infrastructure, shipped to
the GPU box with the snapshot), and ``oracle.ref_suite.kinefold_alias`` aliases
``kinefold`` to this package.  Only the out-of-scope subsystems are deselected
(the list and reasons live in the plugin).  The run's summary is written to
gpurun_out/reference_suite.json when that directory exists."""

from __future__ import annotations

import json
import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
SUITE = os.path.join(ROOT, "oracle", "_ref", "pkg_tests")


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="run oracle/ref_suite/fetch.sh in the build container")
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_reference_suite_passes_against_this_package(precision):
    """fp64 pair math: every in-scope reference test passes.  fp32 (the default):
    the same, except four tests whose tolerances are below fp32 rounding
    (XFAIL_FP32 in the plugin, with reasons)."""
    env = dict(os.environ, KFB200_PAIR_PRECISION=precision)
    out = subprocess.run([sys.executable, "-m", "pytest", "-p", "oracle.ref_suite.kinefold_alias", SUITE,
                          "-q", "-rfx", "-p", "no:cacheprovider", "--rootdir", SUITE],
                         cwd=ROOT, capture_output=True, text=True, timeout=3000, env=env)
    tail = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else ""
    counts = {k: int(v) for v, k in
              re.findall(r"(\d+) (passed|failed|deselected|error|errors|skipped|xfailed|xpassed)", tail)}
    from oracle.ref_suite.kinefold_alias import DESELECT, XFAIL_FP32
    summary = {"precision": precision, "summary_line": tail, "counts": counts,
               "deselected_modules_and_tests": DESELECT,
               "xfail_in_fp32": XFAIL_FP32 if precision == "fp32" else {},
               "failures": [ln for ln in out.stdout.splitlines() if ln.startswith(("FAILED", "XFAIL"))]}
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        with open(os.path.join(ROOT, "gpurun_out", f"reference_suite_{precision}.json"), "w") as fh:
            json.dump(summary, fh, indent=1)
    assert out.returncode == 0, out.stdout[-4000:]
    assert counts.get("passed", 0) >= (144 if precision == "fp64" else 140), tail
