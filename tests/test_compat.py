"""The NumPy façade (paper_2503_05046_b200/compat.py), host logic on CPU:
module layout under the ``mpmrb`` alias and the mode mapping of
``advance_step`` (no device calls)."""

import sys
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2503_05046_b200 import compat, coupling  # noqa: E402


def test_advance_step_maps_by_mode(monkeypatch):
    """mode="deterministic" (the reference's default) -> advance_step_ops
    (particle-id-order P2G, bitwise reproducible); "fast" -> the fused
    advance_step; extra arguments (profiling) always go to the fused path."""
    calls = []
    monkeypatch.setattr(coupling, "advance_step_ops", lambda st: calls.append(("ops", st)) or 1)
    monkeypatch.setattr(coupling, "advance_step",
                        lambda st, *a, **k: calls.append(("fused", st, a, k)) or 2)
    det, fast = SimpleNamespace(mode="deterministic"), SimpleNamespace(mode="fast")
    assert compat._advance_step_by_mode(det) == 1
    assert compat._advance_step_by_mode(fast) == 2
    assert compat._advance_step_by_mode(det, profile={}) == 2
    assert [c[0] for c in calls] == ["ops", "fused", "fused"]


def test_install_registers_reference_module_layout():
    saved = {k: v for k, v in sys.modules.items() if k == "mpmrb" or k.startswith("mpmrb.")}
    try:
        root = compat.install("mpmrb")
        for name in ("transfer", "grid", "mpm", "particles", "materials", "collision",
                     "contact_model", "solver", "coupling", "geometry", "bodies", "rotations"):
            assert sys.modules[f"mpmrb.{name}"] is getattr(root, name)
        assert callable(sys.modules["mpmrb.coupling"].advance_step)
        assert callable(root.advance_step)
    finally:
        for k in [k for k in sys.modules if k == "mpmrb" or k.startswith("mpmrb.")]:
            del sys.modules[k]
        sys.modules.update(saved)
