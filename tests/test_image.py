"""The image module behind the C-ABI (proj/include/rlcuts/image.hpp:65-78,
proj/src/image.cpp:43-136) against the compiled reference: PFM and PPM files
byte-identical to the reference's writers, PFM reads identical, mse and
relative_mse bit-identical; the error classes of ImageIoError; the stats CSV
row of the reference CLI (tools/main.cpp:224-258).  Host code: CPU tests.
Per-pass scoring inside render_frame runs on the GPU (test at the end)."""
import struct

import numpy as np
import pytest

from paper_1911_10217_b200 import rlcuts, scenes


def rand_image(h, w, seed, lo=-0.2, hi=1.4):
    return np.random.default_rng(seed).uniform(lo, hi, (h, w, 3))


def test_pfm_bytes_and_roundtrip(ref, tmp_path):
    img = rand_image(7, 11, 1, -3, 5e3)
    img[0, 0] = [1e-40, -0.0, 3.4e38]  # float32 denormal, signed zero, near max
    ours, theirs = tmp_path / "a.pfm", tmp_path / "b.pfm"
    rlcuts.write_pfm(img, ours)
    ref.ref_write_pfm(img, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(rlcuts.read_pfm(ours), ref.ref_read_pfm(theirs))


def test_pfm_read_big_endian_and_scale(ref, tmp_path):
    h, w = 3, 4
    vals = np.arange(h * w * 3, dtype=np.float32) * 0.37 - 2
    for scale, fmt in ((2.5, ">f"), (-0.5, "<f")):
        p = tmp_path / f"s{scale}.pfm"
        body = b"".join(struct.pack(fmt, float(v)) for v in vals)
        p.write_bytes(f"PF\n{w} {h}\n{scale}\n".encode() + body)
        assert np.array_equal(rlcuts.read_pfm(p), ref.ref_read_pfm(p))


def test_ppm_bytes(ref, tmp_path):
    img = rand_image(9, 13, 2, -0.5, 1.5)
    img[1, 1] = [0.0, 1.0, 0.5]
    ours, theirs = tmp_path / "a.ppm", tmp_path / "b.ppm"
    rlcuts.write_ppm(img, ours)
    ref.ref_write_ppm(img, theirs)
    assert ours.read_bytes() == theirs.read_bytes()


def test_mse_bit_exact(ref):
    a, b = rand_image(31, 17, 3), rand_image(31, 17, 4)
    assert rlcuts.mse(a, b) == ref.ref_mse(a, b)
    assert rlcuts.relative_mse(a, b) == ref.ref_mse(a, b, relative=True)
    z = np.zeros_like(a)
    assert rlcuts.relative_mse(a, z) == np.inf == ref.ref_mse(a, z, relative=True)
    assert rlcuts.relative_mse(z, z) == 0.0 == ref.ref_mse(z, z, relative=True)
    with pytest.raises(ValueError, match="dimensions disagree"):
        rlcuts.mse(a, rand_image(17, 31, 5))


def test_image_errors(tmp_path):
    with pytest.raises(rlcuts.ImageIoError) as e:
        rlcuts.read_pfm(tmp_path / "missing.pfm")
    assert e.value.code == "io_error"
    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"P6\n2 2\n255\n")
    with pytest.raises(rlcuts.ImageIoError) as e:
        rlcuts.read_pfm(bad)
    assert e.value.code == "parse_error"
    short = tmp_path / "short.pfm"
    short.write_bytes(b"PF\n2 2\n-1.0\n" + b"\0" * 20)
    with pytest.raises(rlcuts.ImageIoError, match="truncated"):
        rlcuts.read_pfm(short)
    with pytest.raises(rlcuts.ImageIoError) as e:
        rlcuts.write_pfm(np.zeros((2, 2, 3)), tmp_path / "no" / "dir.pfm")
    assert e.value.code == "io_error"


def test_stats_row_format():
    """write_stats_row (tools/main.cpp:230-258): flags at the stream's default
    precision, results at precision 17, series joined with ';'."""
    cfg = rlcuts.RenderConfig(spp=64, passes=16, sampler=rlcuts.SamplerKind.rl_lightcuts,
                              cut=rlcuts.CutConfig(alpha=0.25, eps_q=1e-5))
    res = rlcuts.RenderResult(np.zeros((1, 1, 3)), 12.5, 7, 1000, 3, [1, 0, 2],
                              [0.1, 1.0 / 3.0])
    row = rlcuts.stats_row("maze,1", cfg, 256, 128, 1.0 / 16, res, 1.0 / 3.0, 2.0 / 3.0)
    assert row.endswith("\n") and row.count("\n") == 1
    assert row == ('"maze,1",rl,64,16,256,128,1,1,1,128,0.25,4,1e-05,1,0.0625,65536,32,4,0,'
                   "fixed,12.5,0.33333333333333331,0.66666666666666663,"
                   "0.10000000000000001;0.33333333333333331,1;0;2,7,1000,3,0.0030000000000000001,\n")
    empty = rlcuts.stats_row("s", rlcuts.RenderConfig(), 8, 8, 0.5, error_message='bad "x"')
    assert empty.endswith(',,,,,,,,,,"bad ""x"""\n')
    assert rlcuts.STATS_HEADER.count(",") == empty.count(",")  # 30 fields


@pytest.mark.gpu
def test_render_frame_pass_mse_matches_reference(ref):
    """render_frame with a reference image (render.cpp:226-228): the per-pass
    mse of the device path equals the reference's sequential sums."""
    scene = scenes.cornell_grid(2, 1, dome_triangles=32, width=40, height=30)
    cfg = rlcuts.RenderConfig(spp=6, passes=3, sampler=rlcuts.SamplerKind.rl_lightcuts, max_depth=2)
    target = ref.ref_render_frame(scene, rlcuts.RenderConfig(spp=8, passes=2, seed=7,
                                                             sampler=cfg.sampler))["image"]
    ctx = rlcuts.build_context(scene, cfg)
    got = rlcuts.render_frame(ctx, cfg, reference=target)
    want = ref.ref_render_frame(scene, cfg, reference=target)
    assert np.array_equal(got.image, want["image"])
    assert got.pass_mse == want["pass_mse"] and len(got.pass_mse) == 3
    assert got.pass_mse[-1] == rlcuts.mse(got.image, target)
    with pytest.raises(ValueError, match="dimensions disagree"):
        rlcuts.render_frame(ctx, cfg, reference=target[:, :-1])
