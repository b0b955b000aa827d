"""B200-native RL-lightcuts direct-lighting path (arXiv 1911.10217).

Host runtime and sm_100a kernels live in ``librlcuts_b200.so`` (built from
``csrc/`` by ``__graft_entry__.build()``) behind the C-ABI in
``include/rlcuts_b200.h``; ``rlcuts`` mirrors the reference's render API over
it and ``scenes`` builds the synthetic BASELINE configurations.
"""
from . import scenes  # noqa: F401
from .rlcuts import (  # noqa: F401
    AlphaSchedule, CutConfig, Framebuffer, HashConfig, HashGrid, RenderConfig, RenderContext,
    RenderResult, SamplerKind, build_context, end_of_pass_update, kernel_launches, render_frame,
    render_pass)
