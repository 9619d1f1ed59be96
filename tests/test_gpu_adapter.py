"""The reference-side binding of INTEGRATION.md, compiled against the
reference's own headers (oracle/adapter/gpu_eval.cpp, oracle/Makefile) and run
next to the reference's CPU evaluation through the reference's C++ API:
evaluate_with_setup_b200 / evaluate_potential_b200 must agree with
hfmm::evaluate_with_setup / evaluate_potential within 1e-10 and raise the same
exception type on an invalid RunConfig."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


def test_reference_side_binding_matches_reference(native):
    if not os.path.exists(EXE):
        pytest.fail("oracle/_ref/adapter_check missing: run __graft_entry__.build() where /root/reference exists")
    res = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "ADAPTER CHECK OK" in res.stdout
    assert res.stdout.count("rel_l2=") == 6
