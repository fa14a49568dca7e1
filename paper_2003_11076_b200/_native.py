"""ctypes binding of include/seethrough_b200.h (the C ABI of the CUDA library).

The product path has no CPU fallback: importing a compute entry point
without the built library, or calling it without a CUDA device, raises.
"""

import ctypes as C
import os

import numpy as np

from .build import LIB

MAX_VIEWS = 12


class StRig(C.Structure):
    _fields_ = [("num_views", C.c_int32), ("ref_index", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32),
                ("warp_a", (C.c_double * 9) * MAX_VIEWS),
                ("warp_b", (C.c_double * 3) * MAX_VIEWS),
                ("view_w", C.c_int32 * MAX_VIEWS), ("view_h", C.c_int32 * MAX_VIEWS)]


MAX_SURFACES = 8


class StSurface(C.Structure):
    _fields_ = [("is_occluder", C.c_int32), ("seed", C.c_int32),
                ("has_x_min", C.c_int32), ("has_x_max", C.c_int32),
                ("depth", C.c_double), ("base", C.c_double), ("amplitude", C.c_double),
                ("frequency", C.c_double), ("x_min", C.c_double), ("x_max", C.c_double),
                ("half_w", C.c_double), ("half_h", C.c_double),
                ("center_x", C.c_double), ("center_y", C.c_double),
                ("c0", C.c_double * 3), ("ca", C.c_double * 3), ("sa", C.c_double * 3),
                ("ph", (C.c_double * 3) * 3), ("nw", C.c_double * 3)]


class StScene(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("n_surfaces", C.c_int32),
                ("pad_", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
                ("cx", C.c_double), ("cy", C.c_double),
                ("surf", StSurface * MAX_SURFACES)]


class StParams(C.Structure):
    _fields_ = [("beta", C.c_double), ("threshold", C.c_double),
                ("max_iters", C.c_int32), ("min_static_rays", C.c_int32),
                ("epsilon_prior", C.c_double), ("sigma", C.c_double),
                ("gamma", C.c_double), ("d_max", C.c_double),
                ("neighborhood_radius", C.c_double),
                ("forced_iters", C.c_int32), ("timing", C.c_int32)]


MAX_ITERS = 1024  # ST_MAX_ITERS (include/seethrough_b200.h)


class StStats(C.Structure):
    _fields_ = [("iterations_run", C.c_int32), ("converged_after", C.c_int32),
                ("mean_energy", C.c_double * MAX_ITERS), ("prev_energy", C.c_double * MAX_ITERS),
                ("changed_fraction", C.c_double * MAX_ITERS), ("active_pixels", C.c_int64),
                ("support_records", C.c_int64), ("candidates_total", C.c_int64),
                ("energy_evals", C.c_int64), ("prev_evals", C.c_int64),
                ("msteps", C.c_int64), ("esteps", C.c_int64),
                ("kernel_ms", C.c_double * 4), ("kernel_launches", C.c_int32 * 4),
                ("hopeless_msteps", C.c_int64), ("energy_samples", C.c_int64)]


class StFrame(C.Structure):
    _fields_ = [("images", C.c_void_p), ("priors", C.c_void_p), ("desc", C.c_void_p),
                ("mu", C.c_void_p), ("sup_tile_start", C.c_void_p),
                ("sup_value", C.c_void_p), ("sup_mask", C.c_void_p),
                ("mu_unsafe", C.c_void_p)]


class StTri(C.Structure):
    _fields_ = [("points", C.c_void_p), ("disparities", C.c_void_p), ("simplices", C.c_void_p),
                ("planes", C.c_void_p), ("neighbors", C.c_void_p), ("transform", C.c_void_p),
                ("equations", C.c_void_p), ("n_pts", C.c_int32), ("n_tri", C.c_int32),
                ("paraboloid_scale", C.c_double), ("paraboloid_shift", C.c_double),
                ("min_bound", C.c_double * 2), ("max_bound", C.c_double * 2),
                ("centroid", C.c_double * 2)]


class StCams(C.Structure):
    _fields_ = [("num_views", C.c_int32), ("ref_index", C.c_int32),
                ("width", C.c_int32), ("height", C.c_int32),
                ("nn", C.c_int32 * MAX_VIEWS),
                ("fx", C.c_double * MAX_VIEWS), ("fy", C.c_double * MAX_VIEWS),
                ("cx", C.c_double * MAX_VIEWS), ("cy", C.c_double * MAX_VIEWS),
                ("rot", (C.c_double * 9) * MAX_VIEWS), ("trans", (C.c_double * 3) * MAX_VIEWS),
                ("unit_baseline", C.c_double),
                ("fw_a", (C.c_double * 9) * MAX_VIEWS), ("fw_b", (C.c_double * 3) * MAX_VIEWS),
                ("bw_a", (C.c_double * 9) * MAX_VIEWS), ("bw_b", (C.c_double * 3) * MAX_VIEWS),
                ("lr_scale", C.c_double * MAX_VIEWS)]


class StFramePlan(C.Structure):
    _fields_ = [("frame", StFrame), ("rig", StRig), ("params", StParams),
                ("median_radius", C.c_int32), ("descriptors_ready", C.c_int32),
                ("values", C.c_void_p), ("status", C.c_void_p), ("static_bits", C.c_void_p),
                ("valid_bits", C.c_void_p), ("image", C.c_void_p), ("prov", C.c_void_p),
                ("n_rays", C.c_void_p), ("scratch", C.c_void_p), ("stats_dev", C.c_void_p),
                ("mu_ws", C.c_void_p), ("mu_ws_bytes", C.c_int64),
                ("sup_ws", C.c_void_p), ("sup_ws_bytes", C.c_int64),
                ("solve_ws", C.c_void_p), ("solve_ws_bytes", C.c_int64),
                ("main_stream", C.c_void_p), ("side_stream", C.c_void_p),
                ("side2_stream", C.c_void_p), ("out_stream", C.c_void_p),
                ("events", C.c_void_p * 4)]


REDUCE_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_int32, C.c_void_p)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)  # st_exchange_fn(stream, user)

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_D = C.c_double
_SIGS = {
    "st_last_error": (C.c_char_p, []),
    "st_version": (C.c_int, []),
    "st_device_count": (C.c_int, []),
    "st_launch_count": (C.c_int64, []),
    "st_tail_graph_count": (C.c_int64, [C.c_int32]),
    "st_struct_size": (C.c_int64, [_I32]),
    "st_fp64_peak": (C.c_int, [C.POINTER(C.c_double), _P]),
    "st_selftest": (C.c_int, [_I32, _I64, C.c_uint64, C.POINTER(C.c_int64), _P]),
    "st_descriptors": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P, _P, _P]),
    "st_bilinear": (C.c_int, [_P, _I32, _I32, _I32, _P, _P, _I64, _P, _P]),
    "st_warp": (C.c_int, [C.POINTER(StRig), _I32, _P, _P, _P, _I64, _P, _P, _P, _P]),
    "st_mu_raster": (C.c_int, [C.POINTER(StTri), _I32, _I32, _D, _P, _P, _I64, _P]),
    "st_mu_raster_workspace": (C.c_int64, [_I32, _I32, _I32]),
    "st_mu_raster_rows": (C.c_int, [C.POINTER(StTri), _I32, _I32, _D, _P, _P, _I64, _I32, _I32,
                                    _P, _P]),
    "st_support_build": (C.c_int, [_P, _P, _I32, _I32, _I32, C.POINTER(StParams),
                                   C.POINTER(StFrame), _P, _I64, C.POINTER(C.c_int64), _P]),
    "st_support_workspace": (C.c_int64, [_I32, _I32, _I32, _D]),
    "st_support_build_rows": (C.c_int, [_P, _P, _I32, _I32, _I32, C.POINTER(StParams),
                                        C.POINTER(StFrame), _P, _I64, C.POINTER(C.c_int64),
                                        _I32, _I32, _P]),
    "st_solve_async": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams),
                                 _P, _P, _P, _P, _P, _P, _I64, _P]),
    "st_frame_plan_init": (C.c_int, [C.POINTER(StFramePlan)]),
    "st_frame_plan_destroy": (C.c_int, [C.POINTER(StFramePlan)]),
    "st_frame_run": (C.c_int, [C.POINTER(StFramePlan), C.POINTER(StTri), _P, _P, _I32, _P, _P,
                               _P]),
    "st_frame_host_bytes": (C.c_int64, [_I32, _I32]),
    "st_l2_set_aside": (C.c_int, [_I64]),
    "st_clocks_start": (C.c_int, [_I32]),
    "st_clocks_stop": (C.c_int64, [_P, _P, _P, _I64]),
    "st_stream_l2_window": (C.c_int, [_P, _P, _I64, C.c_float]),
    "st_host_gather": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64), _I32]),
    "st_h2d_gather": (C.c_int, [_P, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64), _I32, _P]),
    "st_tri_tables": (C.c_int, [C.POINTER(StTri), _P, _P, _P, _P]),
    "st_harvest": (C.c_int, [_P, _P, C.POINTER(StCams), _D, _I32, C.c_float, _I32, _D,
                             _P, _P, _P, _P, _P, _P, _P, _I64, _P]),
    "st_harvest_capacity": (C.c_int64, [_I32, _I32, _I32, _I32]),
    "st_harvest_workspace": (C.c_int64, [_I32, _I32, _I32, _I32]),
    "st_support_dedup": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _I32, _P, _P]),
    "st_initial_masks": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams),
                                   _P, _I64, _P, _P, _P]),
    "st_gather_rays": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), _P, _P, _I64, _P, _P,
                                 _P, _P]),
    "st_energy": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams), _P, _P,
                            _P, _I64, _P, _P, _P]),
    "st_m_step": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams), _P,
                            _I64, _P, _P, _P, _P, _P]),
    "st_e_step_at": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams), _P,
                               _P, _I64, _P, _P, _P]),
    "st_e_step": (C.c_int, [_P, _P, _P, _I64, _I32, C.POINTER(StParams), _P, _P]),
    "st_masked_variance": (C.c_int, [_P, _P, _I64, _I32, _P, _P]),
    "st_solve_workspace": (C.c_int64, [_I32, _I32, _I32]),
    "st_solve": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams), _I32, _P,
                           _P, _P, _P, _P, C.POINTER(StStats), _P, _I64, REDUCE_FN, _P, _P]),
    "st_band_record_bytes": (C.c_int64, []),
    "st_numpy_mean": (C.c_int, [_P, _I64, _P, _P, _I64, _P]),
    "st_numpy_mean_workspace": (C.c_int64, [_I64]),
    "st_solve_rows": (C.c_int, [C.POINTER(StFrame), C.POINTER(StRig), C.POINTER(StParams), _I32,
                                _I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _I64,
                                EXCHANGE_FN, _P, _I32, _P, _P, _P]),
    "st_descriptors_rows": (C.c_int, [_P, _I32, _I32, _I32, _P, _I32, _I32, _P]),
    "st_synthesize_rows": (C.c_int, [_P, C.POINTER(StRig), _P, _P, _P, _I32, _I32, _P, _P, _P,
                                     _P, _P, _I32, _I32, _I32, _I32, _P]),
    "st_synthesize": (C.c_int, [_P, C.POINTER(StRig), _P, _P, _P, _I32, _I32, _P, _P, _P, _P,
                                _P, _P]),
    "st_refocus_pixels": (C.c_int, [_P, C.POINTER(StRig), _P, _P, _P, _I64, _I32, _P, _P, _P,
                                    _P, _P]),
    "st_copy_mask": (C.c_int, [_P, _I64, _D, _P, _P]),
    "st_render_view": (C.c_int, [C.POINTER(StScene), _P, _P, _P, _I32, _P, _P, _P, _P]),
    "st_render_background": (C.c_int, [C.POINTER(StScene), _P, _P, _D, _P, _P, _P, _P]),
    "st_corrupt_prior": (C.c_int, [_P, _I32, _I32, _P, _D, _I32, _P, _P, _I64, _P]),
    "st_corrupt_prior_workspace": (C.c_int64, [_I32, _I32]),
    "st_median": (C.c_int, [_P, _I32, _I32, _I32, _I32, _P, _P]),
}

_lib = None


class NativeError(RuntimeError):
    """CUDA / library failure inside the native path."""


ST_EAGAIN = -4


class BandRetry(RuntimeError):
    """st_solve_rows: a shard's row-window surface raster was not exact;
    every shard redoes the frame with the whole-frame raster."""


def lib():
    """Load the CUDA library (no fallback: raise if it is missing)."""
    global _lib
    if _lib is None:
        path = os.environ.get("ST_LIB_PATH") or LIB  # experiment variants (build.py)
        if not os.path.exists(path):
            raise ImportError(
                f"seethrough_b200 native library not built ({path}); run "
                "`python -m paper_2003_11076_b200.build` (needs nvcc, sm_100a)")
        h = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def check(rc):
    """Map a C ABI return code onto the reference's exception types."""
    if rc == 0:
        return
    msg = lib().st_last_error().decode(errors="replace")
    if rc == -1:
        raise ValueError(msg)
    if rc == ST_EAGAIN:
        raise BandRetry(msg)
    raise NativeError(msg)


def ptr(t):
    """Device (or host) pointer of a torch tensor / None.

    The caller must keep `t` referenced until the call that consumes the
    pointer has been issued; prefer `invoke`, which does that for you.
    """
    return None if t is None else C.c_void_p(t.data_ptr())


def invoke(name, *args):
    """Call a C ABI entry point, passing torch tensors as device pointers.

    The tensors stay referenced (in `args`) until the launch has been
    enqueued on the current stream, so the caching allocator cannot hand
    their blocks to another upload first; the trailing stream argument is
    appended automatically.
    """
    conv = []
    for a in args:
        if a is None:
            conv.append(None)
        elif hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
            conv.append(C.c_void_p(a.data_ptr()))
        else:
            conv.append(a)
    conv.append(stream_handle())
    check(getattr(lib(), name)(*conv))


def stream_handle():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_rig(rig, width, height):
    """st_rig from any object with the CameraRig interface (geometry.py:119-252)."""
    k = len(rig)
    if k > MAX_VIEWS:
        raise ValueError(f"mask enumeration is exponential; refusing {k} views "
                         f"(limit {MAX_VIEWS})")
    r = StRig()
    r.num_views = k
    r.ref_index = int(rig.ref_index)
    r.width = int(width)
    r.height = int(height)
    for i in range(k):
        a, b = rig.warp_coefficients(i)
        a = np.asarray(a, dtype=np.float64).reshape(9)
        b = np.asarray(b, dtype=np.float64).reshape(3)
        for j in range(9):
            r.warp_a[i][j] = float(a[j])
        for j in range(3):
            r.warp_b[i][j] = float(b[j])
        intr = rig.intrinsics(i)
        r.view_w[i] = int(intr.width)
        r.view_h[i] = int(intr.height)
    return r


def make_cams(rig, width, height):
    """st_cams from a CameraRig (geometry.py:128-252): intrinsics, extrinsics,
    nearest neighbours and both pair warps of every (view, neighbour) pair,
    computed by the rig's own numpy expressions."""
    k = len(rig)
    if k > MAX_VIEWS:
        raise ValueError(f"mask enumeration is exponential; refusing {k} views "
                         f"(limit {MAX_VIEWS})")
    c = StCams()
    c.num_views = k
    c.ref_index = int(rig.ref_index)
    c.width = int(width)
    c.height = int(height)
    c.unit_baseline = float(rig.unit_baseline)
    for i in range(k):
        intr, extr = rig.cameras[i]
        nn = int(rig.nearest_neighbor(i))
        c.nn[i] = nn
        c.fx[i], c.fy[i], c.cx[i], c.cy[i] = (float(intr.fx), float(intr.fy), float(intr.cx),
                                              float(intr.cy))
        rot = np.asarray(extr.rotation, dtype=np.float64).reshape(9)
        tr = np.asarray(extr.translation, dtype=np.float64).reshape(3)
        for j in range(9):
            c.rot[i][j] = float(rot[j])
        for j in range(3):
            c.trans[i][j] = float(tr[j])
        for (dst_a, dst_b), (src, dst) in (((c.fw_a, c.fw_b), (i, nn)),
                                           ((c.bw_a, c.bw_b), (nn, i))):
            a, b = rig.pair_warp_coefficients(src, dst)
            a = np.asarray(a, dtype=np.float64).reshape(9)
            b = np.asarray(b, dtype=np.float64).reshape(3)
            for j in range(9):
                dst_a[i][j] = float(a[j])
            for j in range(3):
                dst_b[i][j] = float(b[j])
        c.lr_scale[i] = float(intr.fx) / float(rig.intrinsics(nn).fx)  # prior.py:132
    return c


def make_params(sp, pp, forced_iters=0, timing=False):
    """st_params from SolverParams (solver.py:56-62) + PriorParams (prior.py:33-40)."""
    iters = int(forced_iters or 0) or int(sp.max_iters)
    if iters > MAX_ITERS:
        raise ValueError(f"max_iters {iters} exceeds the {MAX_ITERS} iterations the EM "
                         "statistics hold")
    p = StParams()
    p.beta = float(sp.beta)
    p.threshold = float(sp.threshold)
    p.max_iters = int(sp.max_iters)
    p.min_static_rays = int(sp.min_static_rays)
    p.epsilon_prior = float(sp.epsilon_prior)
    p.sigma = float(pp.sigma)
    p.gamma = float(pp.gamma)
    p.d_max = float(pp.d_max)
    p.neighborhood_radius = float(pp.neighborhood_radius)
    p.forced_iters = int(forced_iters or 0)
    p.timing = 1 if timing else 0
    return p


def gather_args(arrays, offsets):
    """ctypes (srcs, dst_off, sizes, n) for st_host_gather / st_h2d_gather."""
    n = len(arrays)
    srcs = (C.c_void_p * n)(*[a.ctypes.data for a in arrays])
    offs = (C.c_int64 * n)(*offsets)
    sizes = (C.c_int64 * n)(*[a.nbytes for a in arrays])
    return srcs, offs, sizes, n
