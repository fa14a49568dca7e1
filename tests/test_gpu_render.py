"""The device renderer (renderer.py, csrc/st_render.cu)
against the numpy restatement of the reference renderer (oracle/synth.py,
itself pinned to the reference by test_synth_port.py) and against the frame
digests the reference recorded for the bench configs C1-C4.  Bar: every
image, prior, ground-truth mask, background and disparity bit-identical."""

import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def st():
    import paper_2003_11076_b200 as pkg
    pkg.device.require_cuda()
    return pkg


def _same(a, b, what):
    if not np.array_equal(a, b):
        bad = np.argwhere(a != b) if a.shape == b.shape else None
        raise AssertionError(f"{what}: {0 if bad is None else len(bad)} values differ, "
                             f"first {None if bad is None else bad[:4].tolist()}")


def _compare(spec):
    from oracle import synth as ref
    from paper_2003_11076_b200 import synth
    rf, rgt = ref.render(spec)
    df, dgt = synth.render(spec)
    for k, (a, b) in enumerate(zip(rf.images, df.images)):
        _same(a, b, f"image {k}")
    for k, (a, b) in enumerate(zip(rf.priors, df.priors)):
        assert b.dtype == np.float32
        _same(a, b, f"prior {k}")
    for k, (a, b) in enumerate(zip(rgt.masks, dgt.masks)):
        _same(np.asarray(a, bool), np.asarray(b, bool), f"mask {k}")
    _same(rgt.background, dgt.background, "background")
    _same(rgt.disparity, dgt.disparity, "disparity")


@pytest.mark.parametrize("maker,kw", [
    ("occluder_scene", dict(width=160, height=120, p_flip=0.1, blur_radius=2)),
    ("occluder_scene", dict(width=96, height=80, cameras=9, coverage=0.4, seed=5)),
    ("occluder_scene", dict(width=120, height=90, seed=23, p_flip=0.3, blur_radius=0)),
    ("occluder_scene", dict(width=64, height=48, seed=2 ** 33 + 7, p_flip=0.2, blur_radius=5)),
    ("two_plane_scene", dict(width=144, height=96)),
    ("low_texture_scene", dict(width=128, height=80)),
])
def test_device_render_equals_reference_renderer(st, maker, kw):
    from paper_2003_11076_b200 import synth
    _compare(getattr(synth, maker)(**kw))


def test_device_render_ref_index_and_multiple_occluders(st):
    from paper_2003_11076_b200 import synth
    spec = synth.occluder_scene(width=120, height=96, cameras=6, seed=9, p_flip=0.05,
                                blur_radius=1)
    spec.ref_index = 3
    spec.occluders.append(synth.OccluderSpec(depth=0.8, width=0.05, height=0.08,
                                             center_x=-0.04, center_y=0.02, seed=31))
    spec.occluders.append(synth.OccluderSpec(depth=0.5, width=0.03, height=0.03,
                                             center_x=0.05, center_y=-0.03, seed=32))
    _compare(spec)


def test_device_render_rejects_a_scene_without_backdrop(st):
    from paper_2003_11076_b200 import synth
    spec = synth.two_plane_scene(width=48, height=32)
    spec.planes = [synth.PlaneSpec(depth=6.0, seed=1, x_max=0.3)]
    with pytest.raises(ValueError, match="scene constraint violated"):
        synth.render(spec)


def _digest(arrs):
    h = hashlib.sha256()
    for x in arrs:
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_device_render_bench_frames_match_reference_digests(st, cfg):
    """The bench inputs (BASELINE configs C1-C4, up to 3840x2160 x 9 views)
    rendered on the device hash to the digests the reference recorded."""
    import bench
    path = os.path.join(GOLDEN, f"bench_{cfg}.npz")
    if not os.path.exists(path):
        pytest.skip("bench inputs not recorded")
    z = np.load(path)
    w, h, k, dmax, iters = bench.CONFIGS[cfg]
    from paper_2003_11076_b200 import synth
    frame, _ = synth.render(synth.occluder_scene(width=w, height=h, cameras=k, **bench.SCENE))
    assert _digest(frame.images) == str(z["image_digest"])
    assert _digest(frame.priors) == str(z["prior_digest"])
