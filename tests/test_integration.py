"""The reference-side binding (integration/): the C++ shim in namespace
rlcuts::b200 compiles against the reference headers and, on a B200,
renders the same frame as the reference's own render_frame."""
import os
import subprocess

import pytest

from rlc_testutil import has_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "integration", "shim_demo")


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"),
                    reason="reference headers not mounted")
def test_shim_builds_against_reference_headers():
    subprocess.run(["make", "-s", "-B", "-C", os.path.join(ROOT, "integration")], check=True)
    assert os.path.exists(DEMO)


@pytest.mark.skipif(has_gpu(), reason="checks the no-device error mapping")
def test_shim_reports_missing_device():
    if not os.path.exists(DEMO):
        pytest.skip("integration/shim_demo not built")
    r = subprocess.run([DEMO], capture_output=True, text=True)
    assert r.returncode == 2 and "no CPU fallback" in r.stdout


@pytest.mark.gpu
def test_shim_matches_reference_render_frame():
    if not os.path.exists(DEMO):
        pytest.skip("integration/shim_demo not built")
    for k in ("1", "2", "session"):
        r = subprocess.run([DEMO, k], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.startswith("MATCH"), r.stdout + r.stderr
