"""The reference's own in-scope test files, run against the GPU package
through the NumPy façade (paper_2503_05046_b200/compat.py) installed as
``mpmrb`` -- the drop-in claim checked with the reference's tests rather than
restatements of them.

The reference tests are not part of this repository: tools/refsuite_run.sh
copies /root/reference/pkg/tests/{conftest,oracles,test_transfer,test_mpm,
test_collision,test_contact_model,test_solver,test_coupling,
test_materials,test_geometry,test_rigid}.py into
tests/refsuite/_staged/ (git-ignored) for one GPU run and removes them
afterwards; the run's per-test outcome is committed under profiles/.  Without
the staged files this test skips.

Expected differences would be the reference's bitwise-equality tests whose
summation order the GPU does not reproduce (SURVEY.md §4 lists eight); all
eight pass bitwise here.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
STAGED = ROOT / "tests" / "refsuite" / "_staged"

# reference tests that assert bitwise equality of float sums in an order the
# GPU path does not follow, with the reason.  None remain: the
# façade's advance_step in the reference's default mode="deterministic" runs
# the operator pipeline with the particle-id-order P2G fold
# (compat._advance_step_by_mode), so test_substep_equivalence_bitwise holds
# bitwise; the fused substep (mode="fast") agrees with it to roundoff
# (tests/test_gpu_parity.py::test_fused_substep_equivalence).
EXPECTED_DIFF: dict = {}


def test_reference_suite_against_gpu_package(tmp_path):
    if not STAGED.exists() or not any(STAGED.glob("test_*.py")):
        pytest.skip("reference tests not staged (tools/refsuite_run.sh)")
    report = tmp_path / "report.jsonl"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [str(ROOT / "tests" / "refsuite"), str(STAGED), str(ROOT), os.environ.get("PYTHONPATH", "")]))
    cmd = [sys.executable, "-m", "pytest", str(STAGED), "-p", "refsuite_plugin", "-q",
           "-p", "no:cacheprovider", "-o", "addopts=", "--rootdir", str(STAGED),
           f"--junitxml={tmp_path / 'junit.xml'}"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=3000)
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / "reference_suite.log").write_text(r.stdout + r.stderr)
    import xml.etree.ElementTree as ET
    cases = ET.parse(tmp_path / "junit.xml").getroot().iter("testcase")
    results = {}
    for c in cases:
        name = f"{Path(c.get('file') or c.get('classname').replace('.', '/') + '.py').name}::{c.get('name')}"
        kind = "passed"
        for child in c:
            if child.tag in ("failure", "error"):
                kind = "failed"
            elif child.tag == "skipped":
                kind = "skipped"
        results[name] = kind
    with open(out / "reference_suite.json", "w") as fh:
        json.dump(results, fh, indent=1)
    failed = sorted(k for k, v in results.items() if v == "failed")
    unexpected = sorted(k for k in failed if k.split("[")[0] not in EXPECTED_DIFF)
    assert len(results) >= 80, r.stdout[-2000:]
    assert not unexpected, f"unexpected failures: {unexpected}\n{r.stdout[-4000:]}"
