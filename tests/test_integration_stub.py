"""The INTEGRATION.md binding (integration/_b200.py + the dispatch inserted
into the reference's kernels.py by integration/run_reference_tests.py): the
anchors apply to the installed reference and the result is valid Python.
The GPU run of the reference's own suite through it is recorded in
profiles/r2_reference_suite_b200.log."""

import ast
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KP = os.path.join(ROOT, "baseline", "_ref", "ternpack", "kernels.py")
sys.path.insert(0, os.path.join(ROOT, "integration"))


def test_backend_module_parses():
    with open(os.path.join(ROOT, "integration", "_b200.py")) as f:
        ast.parse(f.read())


@pytest.mark.skipif(not os.path.isfile(KP), reason="baseline/_ref not installed")
def test_dispatch_patch_applies():
    import run_reference_tests as R
    with open(KP) as f:
        out = R.patch(f.read())
    ast.parse(out)
    assert out.count("_b200.enabled()") == 4
    assert "from . import _b200" in out
