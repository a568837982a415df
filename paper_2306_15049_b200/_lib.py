"""ctypes loader for librsk.so (the C ABI of include/rsk.h).

Fails loudly: there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librsk.so")

RSK_OK, RSK_EINVAL, RSK_ECUDA, RSK_EUNSUPPORTED, RSK_EPARTIAL, RSK_ENOMEM = range(6)
RSK_APPLY_SHIFTED, RSK_APPLY_SPLIT, RSK_APPLY_C_ONLY, RSK_APPLY_CT_ONLY = range(4)
RSK_PROJ_UTV, RSK_ADD_UC, RSK_SUB_UC = range(3)
(RSK_CG_CONVERGED, RSK_CG_MAXIT, RSK_CG_BREAKDOWN, RSK_CG_DEFL_DROPPED, RSK_CG_ZERO_RHS,
 RSK_NOT_SPD, RSK_SINGULAR) = range(7)
RSK_CG_NO_DEFLATION, RSK_CG_STORE_RES, RSK_CG_PROFILE = 1, 2, 4
RSK_MAX_GROUPS = 4
RSK_MAX_LOCAL = 17

_i64 = C.c_int64
_dp = C.c_void_p          # device pointers are passed as integers
_hp = C.POINTER(C.c_double)


class CgDesc(C.Structure):
    _fields_ = [
        ("nshift", C.c_int),
        ("gamma_h", _hp),
        ("b", _dp),
        ("X", _dp),
        ("ldx", _i64),
        ("has_xp_h", C.POINTER(C.c_int)),
        ("Gout", _dp),
        ("ldg", _i64),
        ("ngroups", C.c_int),
        ("group_of_shift_h", C.POINTER(C.c_int)),
        ("W", _dp * RSK_MAX_GROUPS),
        ("AW", _dp * RSK_MAX_GROUPS),
        ("EW", _dp * RSK_MAX_GROUPS),
        ("ldw", _i64),
        ("J", C.c_int * RSK_MAX_GROUPS),
        ("Ghat", _dp),
        ("ZGhat", _dp),
        ("ldgh", _i64),
        ("has_ghat_h", C.POINTER(C.c_int)),
        ("tol", C.c_double),
        ("maxit", C.c_int),
        ("check_every", C.c_int),
        ("flags", C.c_int),
        ("store", _dp),
        ("lds", _i64),
        ("store_cap", C.c_int),
        ("order_h", C.POINTER(C.c_int)),
        ("Ghat2", _dp),
        ("ZGhat2", _dp),
        ("has_ghat2_h", C.POINTER(C.c_int)),
    ]


class CgOut(C.Structure):
    _fields_ = [
        ("iters", C.POINTER(C.c_int)),
        ("applies", C.POINTER(C.c_int64)),
        ("relres_true", _hp),
        ("status", C.POINTER(C.c_int)),
        ("m_used", C.POINTER(C.c_int)),
        ("store_count", C.POINTER(C.c_int)),
        ("ms_loop", _hp),
    ]


_ip = C.POINTER(C.c_int)

_SIGS = {
    "rsk_version": (C.c_char_p, []),
    "rsk_launch_count": (C.c_int64, []),
    "rsk_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, _i64, _i64, _hp, C.c_int, C.c_int, C.c_int]),
    "rsk_destroy": (C.c_int, [C.c_void_p]),
    "rsk_create_slab": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, _i64, _i64, _i64, _i64, _hp, C.c_int, C.c_int,
                                  C.c_int, C.c_int]),
    "rsk_slab_info": (C.c_int, [C.c_void_p, C.POINTER(_i64)]),
    "rsk_create_ct": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, _i64, C.c_int, _hp, C.c_int, C.c_int]),
    "rsk_ct_info": (C.c_int, [C.c_void_p, C.POINTER(_i64), C.POINTER(_i64), _hp]),
    "rsk_last_error": (C.c_char_p, [C.c_void_p]),
    "rsk_set_weights": (C.c_int, [C.c_void_p, _dp, _dp, C.c_void_p]),
    "rsk_apply_shifted": (C.c_int, [C.c_void_p, C.c_int, _dp, _i64, _dp, _dp, _i64, _dp, _i64, _dp,
                                    C.c_int, C.c_void_p]),
    "rsk_apply_shifted_rows": (C.c_int, [C.c_void_p, C.c_int, _dp, _i64, _dp, _dp, _i64, _dp, _i64, _dp,
                                         C.c_int, _i64, _i64, C.c_void_p]),
    "rsk_recycle_project": (C.c_int, [C.c_void_p, C.c_int, _i64, C.c_int, _dp, _i64, C.c_int, _dp,
                                      _i64, _dp, _i64, C.c_void_p]),
    "rsk_irn_weights": (C.c_int, [C.c_void_p, _dp, C.c_double, _dp, _dp, _dp, C.c_void_p]),
    "rsk_irn_weights_iso": (C.c_int, [C.c_void_p, _dp, C.c_double, _dp, _dp, _dp, C.c_void_p]),
    "rsk_gazzola_weights": (C.c_int, [C.c_void_p, _dp, C.c_double, _dp, _dp, _dp, _dp, C.c_void_p]),
    "rsk_gazzola_max": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, C.c_void_p]),
    "rsk_gazzola_update": (C.c_int, [C.c_void_p, _dp, C.c_double, _dp, _dp, _dp, _dp, _dp, C.c_void_p]),
    "rsk_cg_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_int, C.c_int]),
    "rsk_cg_recycled_batch": (C.c_int, [C.c_void_p, C.POINTER(CgDesc), C.POINTER(CgOut), _dp,
                                        C.c_size_t, C.c_void_p]),
    "rsk_minres_workspace_bytes": (C.c_size_t, [C.c_void_p, C.c_int, C.c_int]),
    "rsk_minres_recycled_batch": (C.c_int, [C.c_void_p, C.POINTER(CgDesc), C.POINTER(CgOut), _dp,
                                            C.c_size_t, C.c_void_p]),
    "rsk_make_rhs": (C.c_int, [C.c_void_p, _dp, _dp, C.c_double, _dp, _dp, C.c_void_p]),
    "rsk_batch_dot": (C.c_int, [C.c_void_p, _i64, C.c_int, _dp, _i64, _dp, _i64, _dp, C.c_void_p]),
    "rsk_batch_axpby": (C.c_int, [C.c_void_p, _i64, C.c_int, _hp, _dp, _i64, _hp, _dp, _i64,
                                  C.c_void_p]),
    "rsk_qr_tall": (C.c_int, [C.c_void_p, _i64, C.c_int, _dp, _i64, _dp, _i64, _hp, C.c_void_p]),
    "rsk_lcurve_norms": (C.c_int, [C.c_void_p, C.c_int, _dp, _i64, _dp, _dp, _dp, _dp, C.c_void_p]),
    "rsk_seminorm_rows": (C.c_int, [C.c_void_p, C.c_int, _dp, _i64, _i64, _i64, _dp, C.c_void_p]),
    "rsk_get_counters": (C.c_int, [C.c_void_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
                                   C.c_int]),
    "rsk_oblique_guess": (C.c_int, [C.c_int, _hp, _hp, _hp, C.c_double, C.c_int, _hp, _hp, _ip]),
    "rsk_orth_guess": (C.c_int, [C.c_int, _hp, _hp, _hp, _hp, _hp, C.c_double, C.c_int, _hp, _hp,
                                 C.POINTER(C.c_int)]),
    "rsk_pencil_ritz": (C.c_int, [C.c_int, _hp, _hp, C.c_double, C.c_int, _hp, _hp]),
    "rsk_stabilize_small": (C.c_int, [C.c_int, _hp, _hp, C.c_double, C.c_int, _hp, C.POINTER(C.c_int)]),
    "rsk_carried_select": (C.c_int, [C.c_int, _hp, _hp, C.c_double, _hp, C.POINTER(C.c_int)]),
    "rsk_sym_eig": (C.c_int, [C.c_int, _hp, _hp, _hp]),
    "rsk_svd_small": (C.c_int, [C.c_int, _hp, _hp, _hp, _hp]),
    "rsk_chol_solve_small": (C.c_int, [C.c_int, _hp, C.c_int, _hp, _hp]),
    "rsk_lcurve_corner": (C.c_int, [C.c_int, _hp, _hp, C.POINTER(C.c_int), _hp]),
    "rsk_local_gram_factors": (C.c_int, [C.c_int, C.c_int, _ip, _ip, _hp, _hp, _hp, _hp, _hp, _hp, _hp, _hp,
                                         _ip, _ip, _ip]),
    "rsk_cholqr_pass": (C.c_int, [C.c_int, _i64, C.c_int, _hp, _hp, _hp]),
    "rsk_gram_solve": (C.c_int, [C.c_int, C.c_int, _hp, _ip, _ip, _hp, _hp, _hp, _hp, _hp]),
    "rsk_cg_alpha": (C.c_int, [C.c_int, _hp, _hp, _hp, _ip]),
    "rsk_cg_scalars": (C.c_int, [C.c_int, C.c_int, _ip, _hp, _hp, _hp, _hp, _hp, _ip, _ip, _hp, C.c_double,
                                 C.c_int, _hp, _hp, _hp, _ip, _hp, _ip, _ip]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str | None = None):
    """Load librsk.so (built in-tree). Raises if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("RSK_LIB_PATH") or LIB_PATH   # RSK_LIB_PATH: A/B builds (tools)
    if not os.path.exists(p):
        raise RuntimeError(f"librsk.so not found at {p}: build it with "
                           "`python -m paper_2306_15049_b200.build` (no CPU fallback exists)")
    try:
        import torch  # noqa: F401  (share torch's libcudart instance)
    except Exception:
        pass
    lib = C.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
