"""CPU-side checks of the C-ABI boundary: the library loads, exports every
function include/rlcuts_b200.h declares, and refuses to run without a B200
(there is no CPU fallback)."""
import ctypes as C

import pytest

from paper_1911_10217_b200 import _lib, rlcuts, scenes
from rlc_testutil import has_gpu


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _lib.declared_functions()
    assert len(declared) >= 25
    missing = [n for n in declared if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers exactly the header
    assert sorted(_lib.SIGNATURES) == declared


def test_struct_layouts_match_header():
    # sizes of the plain-data structs as the C compiler lays them out
    assert C.sizeof(_lib.CutConfigC) == 40
    assert C.sizeof(_lib.HashConfigC) == 32
    assert C.sizeof(_lib.RenderConfigC) == 16 + 40 + 32 + 16
    assert C.sizeof(_lib.CellKeyC) == 20


def test_defaults_match_reference():
    lib = _lib.load()
    c = _lib.RenderConfigC()
    assert lib.rlc_render_config_default(C.byref(c)) == 0
    py = rlcuts.RenderConfig()
    assert (c.spp, c.passes, c.max_depth, c.sampler, c.seed) == (py.spp, py.passes, 1, 0, 1)
    assert (c.cut.cut_size, c.cut.alpha, c.cut.split_threshold, c.cut.eps_q,
            c.cut.iterations) == (128, 0.2, 4.0, -1.0, 1)
    assert (c.hash.capacity, c.hash.probe_limit, c.hash.normal_bits, c.hash.base_tile,
            c.hash.jitter_scale) == (65536, 32, 4, 0.0, 0.0)
    assert lib.rlc_abi_version() == 1


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_no_cpu_fallback():
    s = scenes.cornell_grid(1, 1, dome_triangles=8, width=8, height=8)
    with pytest.raises(rlcuts.NoDeviceError):
        rlcuts.build_context(s, rlcuts.RenderConfig())


def test_null_arguments_are_invalid_argument():
    lib = _lib.load()
    assert lib.rlc_render_config_default(None) == _lib.RLC_ERR_INVALID_ARGUMENT
    assert b"null" in lib.rlc_last_error()
    assert lib.rlc_context_create(None, None, 0, None) == _lib.RLC_ERR_INVALID_ARGUMENT
