"""The reference-side binding of INTEGRATION.md, compiled against the
reference's own headers (oracle/adapter/gpu_eval.cpp, oracle/Makefile) and run
next to the reference's CPU evaluation through the reference's C++ API
(oracle/adapter/adapter_check.cpp, following proj/tests/test_traversal.cpp):
the caller's GlobalSetup is imported (no build_setup on the B200 side),
evaluate_with_setup_b200 / evaluate_potential_b200 agree with
hfmm::evaluate_with_setup / evaluate_potential within 1e-10 at 1 and 4 ranks
with the reference's ledger flop charges, the traversal tests' accuracy and
ledger checks pass on the B200 path, the RankEngine seam reproduces the
serial root multipole at 2, 3 and 5 ranks, and an invalid RunConfig raises
the same exception type."""
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
    assert res.stdout.count(" ok (") == 17, res.stdout
