"""ctypes binding of the C ABI declared in include/ivfkm.h.

The library is built in-tree (``python -m paper_2002_09094_b200.build`` or
``__graft_entry__.build()``).  There is no fallback: if the shared object is
missing, importing anything that needs it raises ImportError.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# IVFKM_LIB: another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("IVFKM_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libivfkm.so")

IVFKM_OBJ_LIMBS = 34
IVFKM_MAXC = 32
IVFKM_E_WORKSPACE = -4  # include/ivfkm.h

_i64, _u64, _i32, _f64, _vp, _sz = C.c_int64, C.c_uint64, C.c_int32, C.c_double, C.c_void_p, C.c_size_t


class Stats(C.Structure):
    """Mirror of ``ivfkm_stats``."""

    _fields_ = [
        ("postings", C.c_ulonglong),
        ("changed", C.c_ulonglong),
        ("near_ties", C.c_ulonglong),
        ("overflow", C.c_ulonglong),
        ("queue_len", C.c_ulonglong),
        ("obj_flags", C.c_ulonglong),
        ("obj_limbs", C.c_longlong * IVFKM_OBJ_LIMBS),
    ]


class SynthSpec(C.Structure):
    _fields_ = [
        ("n", _i64), ("dim", _i64), ("nnz_kind", _i32), ("nnz_mean", _f64),
        ("nnz_sigma", _f64), ("nnz_lo", _i64), ("nnz_hi", _i64), ("zipf_s", _f64),
        ("seed", _i64),
    ]


# name -> (restype, argtypes); the exact set of symbols include/ivfkm.h declares
SIGNATURES = {
    "ivfkm_error_string": (C.c_char_p, [C.c_int]),
    "ivfkm_version": (C.c_int, []),
    "ivfkm_device_count": (C.c_int, []),
    "ivfkm_bivf_nblk": (_i64, [_i64]),
    "ivfkm_bivf_headers_size": (_i64, [_i64, _i64]),
    "ivfkm_bivf_values_capacity": (_i64, [_i64, _i64, _i64]),
    "ivfkm_set_bivf_options": (None, [C.c_float, C.c_int]),
    "ivfkm_bivf_workspace_size": (_sz, [_i64, _i64]),
    "ivfkm_bivf_plan": (C.c_int, [_i64, _i64, C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, _sz,
                                  _vp]),
    "ivfkm_bivf_fill_workspace_size": (_sz, [_i64, _i64, _i64]),
    "ivfkm_bivf_fill": (C.c_int, [_i64, _i64, C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, C.c_int,
                                  _vp, _i64, _vp, _sz, _vp]),
    "ivfkm_bivf_build": (C.c_int, [_i64, _i64, C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, C.c_int,
                                   _vp, _vp, _sz, _vp]),
    "ivfkm_assign_workspace_size": (_sz, [_i64, _i64]),
    "ivfkm_set_tuning": (None, [C.c_int, C.c_int, C.c_int]),
    "ivfkm_set_screen_warps": (None, [C.c_int]),
    "ivfkm_set_screen_option": (C.c_int, [C.c_int, C.c_int]),
    "ivfkm_set_update_option": (C.c_int, [C.c_int, C.c_int]),
    "ivfkm_screen_plan": (C.c_int, [_i64, C.c_int, C.c_int, _vp]),
    "ivfkm_row_order_workspace_size": (_sz, [_i64]),
    "ivfkm_row_order": (C.c_int, [_i64, _vp, _vp, _vp, _sz, _vp]),
    "ivfkm_assign": (C.c_int, [_i64, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, C.c_int, _vp,
                               _f64, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _sz, _vp]),
    "ivfkm_assign_screen": (C.c_int, [_i64, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, C.c_int,
                                      _f64, _vp,
                                      _vp, _vp, _sz, _vp]),
    "ivfkm_assign_screen_ex": (C.c_int, [_i64, _vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, C.c_int,
                                         _f64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ivfkm_doc_freq": (C.c_int, [_i64, _vp, _i64, _vp, _vp]),
    "ivfkm_bivf_slots": (C.c_int, [_i64, _i64, C.c_int, _i64, _vp, _vp, _vp, _vp, _vp]),
    "ivfkm_assign_finish": (C.c_int, [_i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                      _vp, _vp, C.c_int, _vp, _sz, _vp]),
    "ivfkm_score_labels": (C.c_int, [_i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp,
                                     _vp]),
    "ivfkm_update_workspace_size": (_sz, [_i64, _i64, _i64, _i64]),
    "ivfkm_update_count": (C.c_int, [_i64, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp,
                                     _vp, _sz, _vp]),
    "ivfkm_update_state_size": (_sz, [_i64, _i64, _i64, _i64]),
    "ivfkm_update_count_delta": (C.c_int, [_i64, _i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp,
                                           _vp, _vp, _sz, _vp, _sz, _vp]),
    "ivfkm_update_fill": (C.c_int, [_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _i64, _vp, _sz, _vp]),
    "ivfkm_assign_ivf_host": (C.c_int, [_i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                                        _vp]),
    "ivfkm_bivf_plan_fill": (C.c_int, [_i64, _i64, C.c_int, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                       _i64, C.c_int, _vp, _i64, _vp, _sz, _vp, _sz, _vp]),
    "ivfkm_assign_finish_dir": (C.c_int, [_i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp,
                                          _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp, _sz,
                                          _vp]),
    "ivfkm_rankdir_build": (C.c_int, [_i64, _i64, _vp, _vp, _vp, _vp]),
    "ivfkm_bivf_slots_size": (_sz, [_i64, _i64, _i64]),
    "ivfkm_rows_decode": (C.c_int, [_i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "ivfkm_rows_prepare": (C.c_int, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ivfkm_uci_parse": (C.c_int, [_vp, _sz, C.c_int, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                  _vp, _vp, _vp]),
    "ivfkm_bow_workspace_size": (_sz, [_i64]),
    "ivfkm_bow_sort": (C.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "ivfkm_bow_df": (C.c_int, [_i64, _i64, _vp, _vp, _vp]),
    "ivfkm_tfidf_workspace_size": (_sz, [_i64, _i64]),
    "ivfkm_tfidf": (C.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp, _sz, _vp]),
    "ivfkm_assign_ivfd_host": (C.c_int, [_i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp,
                                         _vp]),
    "ivfkm_objects_inverted_workspace_size": (_sz, [_i64, _i64]),
    "ivfkm_objects_inverted": (C.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                         _vp]),
    "ivfkm_ivfd_workspace_size": (_sz, [_i64, _i64]),
    "ivfkm_assign_ivfd": (C.c_int, [_i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp,
                                    _vp, _vp, _i64, _vp, _sz, _vp]),
    "ivfkm_fnv1a64": (_u64, [_vp, _sz]),
    "ivfkm_synth_rows": (C.c_int, [C.POINTER(SynthSpec), _vp]),
    "ivfkm_synth_fill": (C.c_int, [C.POINTER(SynthSpec), _vp, _vp, _vp, _vp,
                                   C.POINTER(_i64), C.POINTER(_i64)]),
}

_lib = None


def load() -> C.CDLL:
    """Load libivfkm.so (once).  Raises ImportError when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2002_09094_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            if not os.environ.get("IVFKM_LIB"):
                raise
            # an older A/B build: tuning setters it lacks become no-ops
            setattr(lib, name, lambda *a, **k: 0)
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class IvfkmError(RuntimeError):
    pass


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().ivfkm_error_string(rc).decode()
        raise IvfkmError(f"{what} failed: {msg} (code {rc})")
