"""The C++ drop-in (include/bmpc_b200.hpp, `bmpc::b200::solve`) against the
unmodified reference `bmpc::solve` on the same BmpcProblem objects, built by
the reference's own builders: oracle/adapter_check.cpp, compiled by
`make -C oracle` into oracle/_ref/ (needs /root/reference at build time; the
binary travels to the GPU box). Each case must show identical status /
iteration counts / alpha sequences and trajectories within 1e-8 relative."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference_solve():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    bad = [l for l in lines if l.get("ok") is False]
    assert not bad, bad
    assert lines and lines[-1] == {"failures": 0}, out.stdout + out.stderr
    assert out.returncode == 0
    assert sum(1 for l in lines if l.get("ok")) >= 14
