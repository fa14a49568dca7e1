"""Reference C4 whole frame (em_solve + synthesize) -> sha256 digests of every output
array and the EMStats (build container; ~40 min on 8 cores):

    OPENBLAS_NUM_THREADS=8 python tests/golden/make_ref_c4_digests.py [dynamic]

`dynamic`: the person-only mode (em_solve(dynamic_only=True) + synthesize
with the copy mask, pipeline.py:250-260) -> ref_C4_dynamic_digests.json.
"""
import hashlib, json, os, sys, time
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)
sys.path.insert(0, os.environ.get("SEETHROUGH_REF", "/root/reference/pkg/src"))
import make_ref_configs as M
import seethrough as st
t0 = time.time()
frame, rig, tri, sp, pp = M.bench_inputs("C4")
t1 = time.time()
dyn = "dynamic" in sys.argv[1:]
dmap, seg, stats = st.em_solve(frame, rig, tri, params=sp, prior_params=pp, dynamic_only=dyn)
t2 = time.time()
copy_mask = frame.priors[rig.ref_index] >= sp.threshold if dyn else None
img, prov, nr = st.synthesize(frame, rig, dmap, seg, min_static_rays=sp.min_static_rays,
                              median_radius=1, copy_mask=copy_mask)
t3 = time.time()
def dg(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
out = dict(values=dg(dmap.values), status=dg(dmap.status), static_bits=dg(seg.static_bits),
           valid_bits=dg(seg.valid_bits), image=dg(img), provenance=dg(prov), n_rays=dg(nr),
           stats=dict(iterations_run=stats.iterations_run, converged_after=stats.converged_after,
                      mean_energy=stats.mean_energy, prev_energy=stats.prev_energy,
                      changed_fraction=stats.changed_fraction),
           seconds=dict(inputs=t1 - t0, solve=t2 - t1, refocus=t3 - t2))
name = "ref_C4_dynamic_digests.json" if dyn else "ref_C4_digests.json"
json.dump(out, open(os.path.join(HERE, name), "w"), indent=1)
print(json.dumps(out["seconds"]), flush=True)
