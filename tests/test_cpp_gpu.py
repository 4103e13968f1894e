"""C++ orchestrator on a B200: LP plan -> AveragingRound -> bit-exact vs oracle."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_round_orchestrator():
    exe = os.path.join(ROOT, "tests", "cpp_gpu", "_build", "round_check")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "round_check ok" in r.stdout
    assert "fractions=0.045455 0.045455 0.045455 0.863636" in r.stdout  # het4b, Appendix A
