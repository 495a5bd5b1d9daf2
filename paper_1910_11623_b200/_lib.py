"""ctypes binding of include/bsde.h (argument marshalling only).

Loads the in-tree ``libbsde.so`` and fails loudly if it is missing: there is no
CPU fallback on the product path.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BSDE_LIB: an alternative build of the same library (kernel experiments)
LIB_PATH = os.environ.get("BSDE_LIB") or os.path.join(_HERE, "libbsde.so")

HEAT, HJB, ALLEN_CAHN, BLACK_SCHOLES = 0, 1, 2, 3
FP32, BF16 = 0, 1
KERNEL_AUTO, KERNEL_SIMT, KERNEL_TC = 0, 1, 2
PROLONG_COPY, PROLONG_INTERP, PROLONG_KEEP_ADAM = 0, 1, 16
OK, EINVAL, ECUDA, ENCCL, EDIVERGED, ESTATE, ENOMEM = 0, -1, -2, -3, -4, -5, -6
ERROR_NAMES = {EINVAL: "EINVAL", ECUDA: "ECUDA", ENCCL: "ENCCL", EDIVERGED: "EDIVERGED",
               ESTATE: "ESTATE", ENOMEM: "ENOMEM"}

# every symbol include/bsde.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "bsde_config_default", "bsde_create", "bsde_workspace_bytes", "bsde_train_step", "bsde_prolongate", "bsde_y0",
    "bsde_num_params", "bsde_get_params", "bsde_set_params", "bsde_get_grads",
    "bsde_get_adam_state", "bsde_set_adam_state", "bsde_get_iteration", "bsde_set_iteration",
    "bsde_current_steps", "bsde_compute_grad", "bsde_eval_loss", "bsde_debug_philox",
    "bsde_debug_dw", "bsde_debug_dw_fast", "bsde_debug_residuals", "bsde_debug_umma",
    "bsde_debug_phase_clocks", "bsde_profile_steps",
    "bsde_launches_per_step", "bsde_kernel_family", "bsde_nccl_unique_id", "bsde_last_error",
    "bsde_ipc_export", "bsde_fused_opt_enable", "bsde_destroy",
]


class Config(ctypes.Structure):
    _fields_ = [
        ("batch_global", ctypes.c_int64),
        ("x0", ctypes.c_double),
        ("lam", ctypes.c_double),
        ("lr", ctypes.c_double),
        ("beta1", ctypes.c_double),
        ("beta2", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("precision", ctypes.c_int),
        ("kernel", ctypes.c_int),
        ("prolong_mode", ctypes.c_int),
        ("max_levels", ctypes.c_int),
        ("device", ctypes.c_int),
        ("stream", ctypes.c_void_p),
        ("rank", ctypes.c_int),
        ("world", ctypes.c_int),
        ("nccl_id", ctypes.c_void_p),
        ("use_graph", ctypes.c_int),
        ("init_zero_head", ctypes.c_int),
        ("coupled_paths", ctypes.c_int),
        ("formulation", ctypes.c_int),
        ("sharded_adam", ctypes.c_int),
        ("deterministic", ctypes.c_int),
        ("shared_zN", ctypes.c_int),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
        ("arch", ctypes.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                "libbsde.so not built (%s); run `python -m paper_1910_11623_b200.build` "
                "— there is no CPU fallback" % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH)
        P, I64, I32, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        pI64, pD, pF = ctypes.POINTER(I64), ctypes.POINTER(D), ctypes.POINTER(ctypes.c_float)
        pU32 = ctypes.POINTER(ctypes.c_uint32)
        sig = {
            "bsde_config_default": (None, [ctypes.POINTER(Config)]),
            "bsde_create": (I32, [I32, I32, I32, D, ctypes.POINTER(I32), I32,
                                  ctypes.POINTER(Config), ctypes.POINTER(P)]),
            "bsde_train_step": (I32, [P, pD]),
            "bsde_workspace_bytes": (I32, [I32, I32, I32, ctypes.POINTER(I32), I32,
                                           ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_size_t)]),
            "bsde_compute_grad": (I32, [P, pD]),
            "bsde_prolongate": (I32, [P, I32]),
            "bsde_y0": (I32, [P, pD]),
            "bsde_num_params": (I32, [P, pI64]),
            "bsde_get_params": (I32, [P, pF, I64]),
            "bsde_set_params": (I32, [P, pF, I64]),
            "bsde_get_grads": (I32, [P, pF, I64]),
            "bsde_get_adam_state": (I32, [P, pF, pF, I64, pI64]),
            "bsde_set_adam_state": (I32, [P, pF, pF, I64, I64]),
            "bsde_get_iteration": (I32, [P, pI64]),
            "bsde_set_iteration": (I32, [P, I64]),
            "bsde_current_steps": (I32, [P, ctypes.POINTER(I32)]),
            "bsde_eval_loss": (I32, [P, ctypes.c_uint32, I64, pD]),
            "bsde_debug_philox": (I32, [P, pU32, pU32, I64, pU32]),
            "bsde_debug_dw": (I32, [P, I64, I32, I64, I64, pF]),
            "bsde_debug_dw_fast": (I32, [P, I64, I32, I64, I64, pF]),
            "bsde_debug_residuals": (I32, [P, I64, I64, pF]),
            "bsde_debug_umma": (I32, [I32, pF, pF, pF]),
            "bsde_profile_steps": (I32, [P, I32, pF, I32]),
            "bsde_debug_phase_clocks": (I32, [P, I32, ctypes.POINTER(ctypes.c_uint64), I32]),
            "bsde_launches_per_step": (I32, [P, ctypes.POINTER(I32)]),
            "bsde_kernel_family": (ctypes.c_char_p, [P]),
            "bsde_nccl_unique_id": (I32, [P]),
            "bsde_last_error": (ctypes.c_char_p, [P]),
            "bsde_ipc_export": (I32, [P, P, I64]),
            "bsde_fused_opt_enable": (I32, [P, P, I32]),
            "bsde_destroy": (None, [P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class BSDEError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (ERROR_NAMES.get(code, "?"), code, msg))
        self.code = code
