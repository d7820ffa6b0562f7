"""BASELINE.json configs[2] (Sec. VI-A): 1e6 frames at 1e8 mu/s with
mu->eee injected in 1% of frames — the CUDA path's signal-track and
signal-event efficiency and reduction factor equal the oracle's on the same
frames (tools/configs2_efficiency.py), and every frame's decision agrees."""
import importlib.util
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_configs2_efficiency_vs_oracle(monkeypatch):
    spec = importlib.util.spec_from_file_location("configs2_efficiency",
                                                  os.path.join(ROOT, "tools", "configs2_efficiency.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    monkeypatch.setattr("sys.argv", ["configs2_efficiency.py", "--frames", "1000000"])
    out = mod.main()
    g, o = out["cuda"], out["oracle"]
    assert out["frames_with_equal_decision"] == 1_000_000
    assert g["kept"] == o["kept"] and g["reduction_factor"] > 100
    for k in ("signal_track_eff", "signal_event_eff", "signal_event_vertex_eff"):
        assert g[k] == o[k], (k, g[k], o[k])
    assert g["signal_track_eff"] >= 0.97
