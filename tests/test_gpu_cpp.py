"""GPU: the reference's own pagerank driver, fuzz generators and ToleranceBound
(compiled from /root/reference/proj into oracle/_ref/b200_ref_driver) running
over merbit::B200Backend -- the drop-in boundary exercised from C++."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
DRIVER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "oracle", "_ref", "b200_ref_driver")


@pytest.mark.skipif(not os.path.exists(DRIVER), reason="built only where /root/reference exists")
def test_reference_drivers_over_b200_backend():
    r = subprocess.run([DRIVER], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout and r.stdout.count("[PASS]") >= 7
