"""TEST INFRASTRUCTURE -- the parity oracle of the RL-lightcuts path.

Two CPU checkers live here, neither of which the product may call:

* ``RefRun`` / ``ref_*``: the unmodified reference library
  (/root/reference/proj/src, compiled in place by oracle/Makefile into
  oracle/_ref/librlcuts_ref.so) driven through its own public API via the
  thin wrapper oracle/ref_capi.cpp.
* ``Oracle*``: the CPU restatement of the path (oracle/rlc_oracle.cpp, built
  into oracle/librlc_oracle.so), pinned against the reference run here and
  against the golden vectors in tests/golden/.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this package.
"""
from .ref import (RefRun, ref_available, ref_lib, ref_mse, ref_read_pfm,  # noqa: F401
                  ref_render_frame, ref_write_pfm, ref_write_ppm)
