"""The bounce sampler's sin/cos (paper_1911_10217_b200/csrc/rlc_libm.h).

sample_cosine_hemisphere (proj/include/rlcuts/math.hpp:101-107) calls the
host libm's std::cos / std::sin, which glibc does not round correctly, so the
device restates glibc's own algorithm.  CPU tests: the restatement (run on
the host through the same header) equals the host libm on sampler angles and
on the angles nearest every multiple of pi/4, for both x86-64 glibc builds
(the SSE2 build forced in a subprocess); the committed table regenerates
identically.  GPU test: the device path equals the host libm."""
import ctypes
import ctypes.util
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1911_10217_b200", "csrc")


def host_libm(x):
    m = ctypes.CDLL(ctypes.util.find_library("m"))
    for f in (m.sin, m.cos):
        f.restype = ctypes.c_double
        f.argtypes = [ctypes.c_double]
    return (np.array([m.sin(float(v)) for v in x]), np.array([m.cos(float(v)) for v in x]))


def sampler_angles(n, seed):
    """phi = 2 pi u2 with u2 on the RandomSequence grid k / 2^53 (rng.hpp)."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, 1 << 53, n, dtype=np.uint64).astype(np.float64) * 2.0 ** -53
    near = []
    for c in np.arange(9) / 8.0:  # u2 near k/8: phi near multiples of pi/4
        k = np.arange(-300, 301, dtype=np.float64)
        v = c + k * 2.0 ** -53
        near.append(v[(v >= 0) & (v < 1)])
    u = np.concatenate([u] + near)
    return 2.0 * np.pi * u


def test_host_restatement_matches_libm():
    variant = rlcuts.libm_variant()
    assert variant in (0, 1), "host libm build not recognised"
    x = sampler_angles(60000, 1)
    s, c = rlcuts.libm_sincos_host(x, variant)
    hs, hc = host_libm(x)
    assert np.array_equal(s, hs) and np.array_equal(c, hc)
    # the two builds really differ, so the variant choice is load-bearing
    other_s, other_c = rlcuts.libm_sincos_host(x, 1 - variant)
    assert not (np.array_equal(other_s, hs) and np.array_equal(other_c, hc))


def test_probe_follows_glibc_dispatch():
    """With FMA masked out glibc runs its SSE2 build; the probe must follow."""
    code = ("from paper_1911_10217_b200 import rlcuts; import numpy as np;"
            "import test_libm as t;"
            "v = rlcuts.libm_variant(); x = t.sampler_angles(20000, 2);"
            "s, c = rlcuts.libm_sincos_host(x, v); hs, hc = t.host_libm(x);"
            "print(v, bool(np.array_equal(s, hs) and np.array_equal(c, hc)))")
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA", PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    variant, ok = out.stdout.split()
    assert ok == "True"
    assert variant == "0"  # the SSE2 build


def test_table_regenerates():
    sys.path.insert(0, CSRC)
    try:
        import gen_sincostab
    finally:
        sys.path.pop(0)
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        gen_sincostab.main()
    with open(os.path.join(CSRC, "rlc_sincostab.h")) as f:
        assert buf.getvalue() == f.read()


@pytest.mark.gpu
def test_device_sincos_matches_libm():
    scene = scenes.cornell_grid(1, 1, dome_triangles=8, width=8, height=8)
    ctx = rlcuts.build_context(scene, rlcuts.RenderConfig())
    x = sampler_angles(200000, 3)
    s, c = ctx.libm_sincos(x)
    hs, hc = host_libm(x)
    assert np.array_equal(s, hs) and np.array_equal(c, hc)
