"""Memory-safety checks without compute-sanitizer (closed on this GPU pool).

* Guard zones: every device buffer of a FramePipeline / BandPipeline sits
  between two 4 KiB zones of a known byte pattern; after the whole product
  path runs (descriptors, surface raster, support groups, harvest, the
  dense, dynamic_only and forced-iteration solves, the synchronous solve
  with per-kernel timing, refocus + median, the native one-call frame, a row
  band) no zone may have changed: no kernel writes outside its buffers.
* Repetition: worklists are appended by warp-aggregated atomics and the
  statistics fold in the last block; results must not depend on the
  scheduling, so 8 back-to-back runs (and runs on concurrent streams) must
  give byte-identical artefacts and EMStats.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _inputs(name):
    import bench
    if name.startswith("C"):
        frame, rig, tri, exact = bench.load_inputs(name)
        sp, pp = bench.params_for(name)
        return frame, rig, tri, sp, pp
    import paper_2003_11076_b200 as st
    from golden_io import load
    from test_gpu_parity import _Rig, _Tri, _frame, _params
    g = load(name)
    sp, pp = _params(st, g)
    return _frame(st, g), _Rig(g), _Tri(g), sp, pp


@pytest.mark.parametrize("name", ["occ160_tilt", "occ128_k9", "C2"])
def test_no_kernel_writes_outside_its_buffers(name):
    import torch

    from paper_2003_11076_b200.prior import TriDevice
    from paper_2003_11076_b200.reconstruct import FramePipeline
    from paper_2003_11076_b200.sharding import BandPipeline
    frame, rig, tri, sp, pp = _inputs(name)
    h, w = frame.shape
    pipe = FramePipeline(rig, w, h, sp, pp, guard_bytes=4096)
    pipe.load(frame.images, frame.priors)
    td = TriDevice(tri)
    if name.startswith("C"):  # the harvest needs the full CameraRig (cameras, baselines)
        pipe.harvest()
    for kw in (dict(), dict(dynamic_only=True), dict(forced_iters=5), dict(timing=True),
               dict(median_radius=2)):
        pipe.run(td, **kw)
        pipe.fetch()
    block, _ = pipe.run_native(td, out_stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert pipe.check_guards() == 0
    bp = BandPipeline(rig, w, h, sp, pp, guard_bytes=4096)
    bp.load(frame.images, frame.priors)
    bp.run(td)
    bp.run(td, dynamic_only=True)
    torch.cuda.synchronize()
    assert bp.pipe.check_guards() == 0


@pytest.mark.parametrize("name", ["C2", "occ128_k9"])
def test_results_do_not_depend_on_scheduling(name):
    import torch

    import paper_2003_11076_b200 as st
    frame, rig, tri, sp, pp = _inputs(name)
    ref = st.reconstruct(frame, rig, tri, sp, pp)
    outs = list(st.reconstruct_stream([(frame, tri)] * 8, rig, sp, pp))
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):  # another stream, racing the default one's work
        outs.append(st.reconstruct(frame, rig, tri, sp, pp))
    for r in outs:
        for a, b in ((r.disparity.values, ref.disparity.values),
                     (r.disparity.status, ref.disparity.status),
                     (r.segmentation.static_bits, ref.segmentation.static_bits),
                     (r.segmentation.valid_bits, ref.segmentation.valid_bits),
                     (r.image, ref.image), (r.provenance, ref.provenance),
                     (r.n_rays, ref.n_rays)):
            assert np.array_equal(a, b)
        assert list(r.stats.mean_energy) == list(ref.stats.mean_energy)
        assert list(r.stats.prev_energy) == list(ref.stats.prev_energy)
        assert r.stats.energy_evals == ref.stats.energy_evals


@pytest.mark.parametrize("mode", ["slot", "main", "2"])
@pytest.mark.parametrize("dyn", [False, True])
def test_stream_modes_keep_frames_apart(monkeypatch, mode, dyn):
    """reconstruct_stream's compute-stream modes (ST_STREAM_COMPUTE: one
    stream per slot, the caller's stream, two slot streams) with several
    frames in flight: every output equals reconstruct() of its own frame,
    for two alternating frames (distinct active sets and results)."""
    import paper_2003_11076_b200 as st
    frame, rig, tri, sp, pp = _inputs("C1")
    other = st.LightFieldFrame(images=[np.ascontiguousarray(np.roll(x, 7, axis=1))
                                       for x in frame.images],
                               priors=[np.ascontiguousarray(np.roll(x, 7, axis=1))
                                       for x in frame.priors])
    frames = [frame, other]
    refs = [st.reconstruct(f, rig, tri, sp, pp, dynamic_only=dyn) for f in frames]
    assert not np.array_equal(refs[0].image, refs[1].image)
    monkeypatch.setenv("ST_STREAM_COMPUTE", mode)
    outs = list(st.reconstruct_stream([(frames[i % 2], tri) for i in range(9)], rig, sp, pp,
                                      dynamic_only=dyn))
    assert len(outs) == 9
    for i, r in enumerate(outs):
        ref = refs[i % 2]
        for a, b in ((r.disparity.values, ref.disparity.values),
                     (r.segmentation.static_bits, ref.segmentation.static_bits),
                     (r.image, ref.image), (r.provenance, ref.provenance)):
            assert np.array_equal(a, b), (mode, dyn, i)
        assert list(r.stats.mean_energy) == list(ref.stats.mean_energy)
