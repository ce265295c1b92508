"""pytest plugin: run the reference's own test files against the GPU package.

Loaded with ``-p refsuite_plugin`` (tests/refsuite on PYTHONPATH); installs
paper_2503_05046_b200.compat as ``mpmrb`` before the staged test modules are
imported (tests/test_reference_suite.py, tools/refsuite_run.sh)."""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2503_05046_b200 import compat  # noqa: E402

compat.install("mpmrb")
