"""ctypes binding of libomnitrack.so (include/omnitrack.h).

The library is REQUIRED: importing a compute function without the built
.so, or without a CUDA device, raises -- there is no CPU fallback on the
product path.  Build it with `python -m paper_1910_06017_b200.build`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FT_LIB") or os.path.join(HERE, "libomnitrack.so")  # FT_LIB: A/B builds

FT_OK, FT_EINVAL, FT_ERANGE, FT_ECUDA, FT_ENOMEM, FT_ECAP = 0, -1, -2, -3, -4, -5
FT_STREAM_SKIP = -2  # n_dets of a stream that does not advance in a tracker step


class OmniTrackError(RuntimeError):
    """CUDA / capacity failure inside libomnitrack."""


class ft_flow_params(C.Structure):
    _fields_ = [("data_weight", C.c_double), ("huber_epsilon", C.c_double),
                ("time_step", C.c_double), ("warps_per_level", C.c_int32),
                ("iterations_per_warp", C.c_int32), ("pyramid_scales", C.c_int32),
                ("_pad", C.c_int32)]


class ft_det(C.Structure):
    _fields_ = [("class_id", C.c_int32), ("label_ref", C.c_int32), ("score", C.c_double),
                ("x", C.c_double), ("y", C.c_double), ("w", C.c_double), ("h", C.c_double)]


class ft_track(C.Structure):
    _fields_ = [("id", C.c_int64), ("class_id", C.c_int32), ("label_ref", C.c_int32),
                ("x", C.c_double), ("y", C.c_double), ("w", C.c_double), ("h", C.c_double),
                ("score", C.c_double), ("state", C.c_int32), ("born_at", C.c_int32),
                ("last_seen", C.c_int32), ("lost_at", C.c_int32)]


class ft_tracker_config(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("n_streams", C.c_int32),
                ("max_tracks", C.c_int32), ("max_dets", C.c_int32),
                ("rof_iterations", C.c_int32), ("gate", C.c_double),
                ("min_score", C.c_double), ("detection_blend", C.c_double),
                ("rof_weight", C.c_double), ("rof_blend", C.c_double),
                ("flow", ft_flow_params), ("motion", C.c_int32), ("klt_grid", C.c_int32),
                ("prefetch", C.c_int32), ("_pad", C.c_int32)]


MOTION_TVL1, MOTION_KLT = 0, 1


# numpy views of the record structs (same layout)
DET_DTYPE = np.dtype([("class_id", "<i4"), ("label_ref", "<i4"), ("score", "<f8"),
                      ("x", "<f8"), ("y", "<f8"), ("w", "<f8"), ("h", "<f8")])
TRACK_DTYPE = np.dtype([("id", "<i8"), ("class_id", "<i4"), ("label_ref", "<i4"),
                        ("x", "<f8"), ("y", "<f8"), ("w", "<f8"), ("h", "<f8"),
                        ("score", "<f8"), ("state", "<i4"), ("born_at", "<i4"),
                        ("last_seen", "<i4"), ("lost_at", "<i4")])
assert DET_DTYPE.itemsize == C.sizeof(ft_det)
assert TRACK_DTYPE.itemsize == C.sizeof(ft_track)

_P = C.c_void_p
_I = C.c_int
_D = C.c_double

# name -> (restype, argtypes); every symbol include/omnitrack.h declares
SIGNATURES = {
    "ft_last_error": (C.c_char_p, []),
    "ft_version": (_I, []),
    "ft_device_count": (_I, [C.POINTER(_I)]),
    "ft_ctx_create": (_I, [_I, C.POINTER(_P)]),
    "ft_ctx_destroy": (_I, [_P]),
    "ft_ctx_set_stream": (_I, [_P, _P]),
    "ft_ctx_synchronize": (_I, [_P]),
    "ft_select_level": (_I, [_I, _I, C.POINTER(_I)]),
    "ft_auto_scales": (_I, [_I, _I, C.POINTER(_I)]),
    "ft_gray8_to_unit": (_I, [_P, _P, _I, _I, _P]),
    "ft_check_plane": (_I, [_P, _P, C.c_int64, _D, _D, C.POINTER(C.c_int32)]),
    "ft_build_pyramid": (_I, [_P, _P, _I, _I, _I, _P]),
    "ft_structure_texture": (_I, [_P, _P, _I, _I, _D, _D, _I, _P]),
    "ft_rof_denoise": (_I, [_P, _P, _I, _I, _D, _I, _D, _P]),
    "ft_update": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _I, _D, _P, _P, _P, _P, C.POINTER(_I)]),
    "ft_flow_energy_terms": (_I, [_P, _P, _P, _P, _P, _I, _I, _D, _P, _P, _P]),
    "ft_compute_flow": (_I, [_P, _P, _P, _I, _I, C.POINTER(ft_flow_params), _P, _P]),
    "ft_compute_flow_traced": (_I, [_P, _P, _P, _I, _I, C.POINTER(ft_flow_params), _P, _P, _P]),
    "ft_predict": (_I, [_P, _P, _I, _P, _P, _I, _I, _I, _I, _I, _P, _P]),
    "ft_klt_predict": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _P, _P]),
    "ft_iou_matrix": (_I, [_P, _P, _I, _P, _I, _P]),
    "ft_hungarian": (_I, [_P, _P, _I, _I, _I, _D, _P, C.POINTER(_I)]),
    "ft_match": (_I, [_P, _P, _P, _I, _P, _P, _I, _D, _P, _P, C.POINTER(_I)]),
    "ft_tracker_create": (_I, [_P, C.POINTER(ft_tracker_config), C.POINTER(_P)]),
    "ft_tracker_destroy": (_I, [_P]),
    "ft_tracker_step": (_I, [_P, _P, _I, _P, _P, _P, _P]),
    "ft_tracker_input_buffers": (_I, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "ft_tracker_step_device": (_I, [_P, _P, _I, _P, _P]),
    "ft_tracker_slot_buffers": (_I, [_P, _I, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "ft_tracker_submit": (_I, [_P, _I, _I, _P, _P, _P]),
    "ft_tracker_wait": (_I, [_P, _I, _P, _P]),
    "ft_tracker_stage": (_I, [_P, _I, _I, _P, _I, _I, _P, _I]),
    "ft_tracker_submit_staged": (_I, [_P, _I]),
    "ft_tracker_flush": (_I, [_P, _I]),
    "ft_tracker_step_stream": (_I, [_P, _I, _P, _I, _I, _P, _I, _P, C.POINTER(C.c_int32)]),
    "ft_tracker_read": (_I, [_P, _P, _P]),
    "ft_tracker_field": (_I, [_P, _I, C.POINTER(_P), C.POINTER(_P), C.POINTER(_I),
                              C.POINTER(_I)]),
    "ft_tracker_read_field": (_I, [_P, _I, _P, _P]),
    "ft_tracker_profile_pd": (_I, [_P, _I, C.POINTER(_D), C.POINTER(_D), C.POINTER(_I)]),
    "ft_tracker_pd_span": (_I, [_P, C.POINTER(_D), C.POINTER(_I), C.POINTER(_D)]),
    "ft_tracker_launches": (_I, [_P, C.POINTER(C.c_int64)]),
    "ft_tracker_phase_times": (_I, [_P, _I, C.POINTER(_D), C.POINTER(C.c_char_p), _I,
                                    C.POINTER(_I)]),
    "ft_tracker_reset": (_I, [_P]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libomnitrack.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise OmniTrackError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_1910_06017_b200.build` (no CPU fallback exists)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int):
    if rc == FT_OK:
        return
    msg = load().ft_last_error().decode(errors="replace")
    if rc == FT_EINVAL:
        raise ValueError(msg)
    if rc == FT_ERANGE:
        raise IndexError(msg)
    raise OmniTrackError(f"libomnitrack error {rc}: {msg}")


_tls = threading.local()


def ctx(device: int | None = None):
    """Per-(thread, device) ft_ctx bound to torch's current stream."""
    import torch

    if not torch.cuda.is_available():
        raise OmniTrackError("libomnitrack needs a CUDA device (sm_100a); none is visible")
    dev = torch.cuda.current_device() if device is None else int(device)
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    h = cache.get(dev)
    lib = load()
    if h is None:
        hp = C.c_void_p()
        check(lib.ft_ctx_create(dev, C.byref(hp)))
        h = cache[dev] = hp.value
    stream = torch.cuda.current_stream(dev).cuda_stream
    check(lib.ft_ctx_set_stream(h, C.c_void_p(stream)))
    return h


def check_plane(t, lo: float, hi: float) -> int:
    """Device-side Frame / MotionField validation of a CUDA float64 tensor:
    0, or bit 0 = non-finite values, bit 1 = finite values outside [lo, hi]."""
    st = C.c_int32()
    check(load().ft_check_plane(ctx(t.device.index), ptr(t), t.numel(), float(lo), float(hi),
                                C.byref(st)))
    return st.value


def ptr(a) -> C.c_void_p:
    """Address of a torch tensor or numpy array."""
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def flow_params_struct(p) -> ft_flow_params:
    return ft_flow_params(float(p.data_weight), float(p.huber_epsilon), float(p.time_step),
                          int(p.warps_per_level), int(p.iterations_per_warp),
                          0 if p.pyramid_scales is None else int(p.pyramid_scales), 0)
