"""ctypes binding of libfluidrank_b200.so (include/fluidrank_b200.h).

The product has no CPU fallback: if the shared library is missing, importing
this module raises ImportError; if no CUDA device is visible, every device
entry point raises RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FR_LIB_PATH: development override to load a variant build (tools/build_variant.sh)
LIB_PATH = os.environ.get("FR_LIB_PATH") or os.path.join(_HERE, "libfluidrank_b200.so")

FR_OK = 0
FR_ERR_RANGE = 1
FR_ERR_SELF_LOOP = 2
FR_ERR_DUPLICATE = 3
FR_ERR_ARG = 4
FR_ERR_CUDA = 5
FR_ERR_NO_CONVERGENCE = 6
FR_ERR_NO_DEVICE = 7

SELECT = {"sweep": 0, "max": 1, "per": 2, "rand": 3, "op": 4, "op2": 5}
POLICY = {"exhaust": 0, "geometric": 1, "adaptive": 2}


class GenConfig(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("max_out", ctypes.c_int32),
                ("mean_degree", ctypes.c_double), ("alpha", ctypes.c_double),
                ("max_degree", ctypes.c_int32), ("window", ctypes.c_int32),
                ("dangling_frac", ctypes.c_double), ("local_frac", ctypes.c_double),
                ("zipf_s", ctypes.c_double)]


class SolverConfig(ctypes.Structure):
    _fields_ = [("damping", ctypes.c_double), ("target_error", ctypes.c_double),
                ("decay", ctypes.c_double), ("rand_frac", ctypes.c_double),
                ("edge_frac", ctypes.c_double), ("max_sweeps", ctypes.c_int64),
                ("max_diffusions", ctypes.c_int64),
                ("select", ctypes.c_int32), ("policy", ctypes.c_int32),
                ("fluid_fp32", ctypes.c_int32), ("thread_max_degree", ctypes.c_int32),
                ("block_min_degree", ctypes.c_int32), ("seed", ctypes.c_uint32),
                ("kernel_path", ctypes.c_int32), ("hot_slots", ctypes.c_int32),
                ("degree_exponent", ctypes.c_double), ("warm_slots", ctypes.c_int32)]


class TraceRow(ctypes.Structure):
    _fields_ = [("elementary_steps", ctypes.c_int64), ("diffusions", ctypes.c_int64),
                ("sweeps", ctypes.c_int64), ("residual", ctypes.c_double),
                ("theta", ctypes.c_double), ("t_ns", ctypes.c_int64)]


class SolveStats(ctypes.Structure):
    _fields_ = [("diffusions", ctypes.c_int64), ("elementary_steps", ctypes.c_int64),
                ("sweeps", ctypes.c_int64), ("residual", ctypes.c_double),
                ("theta", ctypes.c_double), ("trace_len", ctypes.c_int64),
                ("hub_edges", ctypes.c_int64)]


# every symbol the header declares, with its ctypes signature
_P, _I64, _I32, _F64, _U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_uint64
SIGNATURES = {
    "fr_last_error": (ctypes.c_char_p, []),
    "fr_abi_version": (ctypes.c_int, []),
    "fr_device_sms": (ctypes.c_int, []),
    "fr_gen_degrees": (ctypes.c_int, [_P, _I64, _U64, _P, _P, _P]),
    "fr_gen_edges": (ctypes.c_int, [_P, _I64, _U64, _P, _P, _P, _P]),
    "fr_gen_edges_round": (ctypes.c_int, [_P, _I64, _U64, ctypes.c_uint32, _P, _P, _P, _P, _P, _P]),
    "fr_csr_build": (ctypes.c_int, [_I64, _I64, _P, _P, _I32, _P, _P, _P, _P]),
    "fr_in_degree": (ctypes.c_int, [_I64, _I64, _P, _P, _P]),
    "fr_init_state": (ctypes.c_int, [_I64, _F64, _P, _P, _I32, _P, _P]),
    "fr_diffuse_node": (ctypes.c_int, [_I64, _P, _P, _P, _P, _I64, _F64, _P, _P]),
    "fr_abs_sum": (ctypes.c_int, [_I64, _P, _I32, _P, _P]),
    "fr_normalize": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "fr_solver_create": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P, _I64, _P, _P]),
    "fr_solver_run": (ctypes.c_int, [_P, _P, _P]),
    "fr_solver_run_profiled": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "fr_solver_trace": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "fr_solver_run_sampled": (ctypes.c_int, [_P, _P, _P, _I64, _P]),
    "fr_solver_trace_errors": (ctypes.c_int, [_P, _P, _I64, _P]),
    "fr_l1_error": (ctypes.c_int, [_I64, _P, _P, _P, _P]),
    "fr_solver_destroy": (ctypes.c_int, [_P]),
    "fr_power_create": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _F64, _P, _P, _P]),
    "fr_power_run": (ctypes.c_int, [_P, _F64, _I64, _P, _P, _P, _P]),
    "fr_power_run_profiled": (ctypes.c_int, [_P, _F64, _I64, _P, _P, _P, _P]),
    "fr_power_destroy": (ctypes.c_int, [_P]),
    "fr_pagerank_host": (ctypes.c_int, [_I64, _I64, _P, _P, _P, _P, _P, _P]),
    "fr_ppr_init": (ctypes.c_int, [_I64, _I32, _P, _I32, _F64, _P, _P, _P]),
    "fr_ppr_create": (ctypes.c_int, [_I64, _I64, _P, _P, _I32, _P, _P, _P, _P, _P]),
    "fr_ppr_run": (ctypes.c_int, [_P, _P, _P, _P]),
    "fr_ppr_set_pull": (ctypes.c_int, [_P, _P, _P]),
    "fr_ppr_destroy": (ctypes.c_int, [_P]),
    "fr_ppr_normalize": (ctypes.c_int, [_I64, _I32, _P, _P, _P]),
}


ABI_VERSION = 3  # FR_ABI_VERSION of include/fluidrank_b200.h


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "or `make -C paper_1202_6158_b200/csrc` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fr_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH} has ABI version {lib.fr_abi_version()}, this package binds "
                          f"{ABI_VERSION} (include/fluidrank_b200.h): rebuild the library")
    return lib


lib = _load()


class NoConvergenceError(RuntimeError):
    """The sweep or iteration budget ran out above the target error."""


def check(rc, exc=None):
    """Raise the exception matching an FR_* status (reference error types)."""
    if rc == FR_OK:
        return
    msg = lib.fr_last_error().decode("utf-8", "replace")
    if exc is not None:
        raise exc(msg)
    if rc in (FR_ERR_RANGE, FR_ERR_SELF_LOOP, FR_ERR_DUPLICATE, FR_ERR_ARG):
        raise ValueError(msg)
    if rc == FR_ERR_NO_CONVERGENCE:
        raise NoConvergenceError(msg)
    raise RuntimeError(msg)


def require_device():
    """The product runs on a CUDA device only; fail loudly otherwise."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1202_6158_b200 needs a CUDA device (B200); none is visible "
                           "and there is no CPU fallback")
    torch.cuda.current_device()  # make the primary context current
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())
