"""The numpy restatement of the reference renderer (oracle/synth.py) is
bit-identical to the reference (synth.py) here, and to the digests the
reference recorded in tests/golden/bench_*.npz (CPU).  It is the checker of
the device renderer (tests/test_gpu_render.py).
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import synth as port
from paper_2003_11076_b200 import synth as specs

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("maker,kw", [
    ("occluder_scene", dict(width=96, height=64, p_flip=0.1, blur_radius=2)),
    ("occluder_scene", dict(width=80, height=60, cameras=9, coverage=0.4, seed=5)),
    ("two_plane_scene", dict(width=72, height=48)),
    ("low_texture_scene", dict(width=64, height=40)),
])
def test_render_matches_reference(reference, maker, kw):
    ref_spec = getattr(reference, maker)(**kw)
    my_spec = getattr(specs, maker)(**kw)
    rf, rgt = reference.render(ref_spec)
    mf, mgt = port.render(my_spec)
    for a, b in zip(rf.images, mf.images):
        assert np.array_equal(a, b)
    for a, b in zip(rf.priors, mf.priors):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    assert np.array_equal(rgt.disparity, mgt.disparity)
    assert np.array_equal(rgt.background, mgt.background)
    for a, b in zip(rgt.masks, mgt.masks):
        assert np.array_equal(a, b)


def test_box_blur_and_corruption_match_reference(reference):
    rng = np.random.default_rng(4)
    a = (rng.random((23, 31)) < 0.5).astype(np.float64)
    for r in (0, 1, 3):
        assert np.array_equal(port.box_blur(a, r), reference.box_blur(a, r))
        assert np.array_equal(port.corrupt_prior(a, 0.2, r, seed=[1, 2, 17]),
                              reference.corrupt_prior(a, 0.2, r, seed=[1, 2, 17]))


def _digest(arrs):
    h = hashlib.sha256()
    for x in arrs:
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


@pytest.mark.slow
def test_c1_bench_frame_matches_recorded_digest():
    path = os.path.join(GOLDEN, "bench_C1.npz")
    if not os.path.exists(path):
        pytest.skip("bench inputs not recorded")
    z = np.load(path)
    w, h, k = (int(x) for x in z["config"][:3])
    frame, _ = port.render(specs.occluder_scene(width=w, height=h, cameras=k, coverage=0.25,
                                               seed=11, p_flip=0.1, blur_radius=2))
    assert _digest(frame.images) == str(z["image_digest"])
    assert _digest(frame.priors) == str(z["prior_digest"])
