"""Runs the C++ unit tests of the host API (tests/cpp/*.cpp, built by
paper_2106_10207_b200/_build.py) — warm-start LP, strategy/partition/groups
through the C++ declarations the reference's callers compile against."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_unit_tests():
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "unit_tests")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed checks" in r.stdout
