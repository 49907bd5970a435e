"""CPU: the C-ABI library loads, exports every entry point declared in
include/bmpc_b200.h, and fails loudly (no CPU fallback) without a GPU."""
import os
import re
import subprocess

import pytest

import _oracle as O
import paper_2506_13624_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bmpc_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bmpc_\w+)\s*\(", src)))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def test_library_exports_every_declared_symbol():
    decl = declared_functions()
    assert len(decl) >= 25
    syms = exported(B.LIB_PATH)
    missing = [d for d in decl if d not in syms]
    assert not missing, missing


def test_library_is_sm100a_fatbin():
    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_defaults():
    assert "sm_100a" in B.version()
    o = B.SolverOptions()
    assert (o.max_inner_iterations, o.max_outer_iterations, o.alpha_levels) == (100, 10, 11)  # solver.hpp:35-37


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    with pytest.raises(B.BmpcError):
        B.Context(0)
    p = B.build_intersection_case(B.intersection_spec(20, 4.0, 0.4), 2, 2)
    with pytest.raises(B.BmpcError):
        B.solve(p)


def test_oracle_library_exports():
    syms = exported(O.SO)
    for s in ("bo_solve", "bo_lqr_tree", "bo_build_tree", "bo_random_lq", "bo_rollout", "bo_evaluate"):
        assert s in syms
