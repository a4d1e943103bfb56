"""ctypes mirror of include/lamfast_cuda.h and the loader of the CUDA library.

The product library is ``paper_1905_05417_b200/lib/liblamfast_b200.so`` (built
in-tree by ``__graft_entry__.build()``).  There is no CPU fallback: if the
library is missing, loading fails loudly; if no GPU is present, every compute
entry point returns ``LF_ERR_CUDA``.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_char_p, c_double, c_int, c_int32, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LAMFAST_LIB") or os.path.join(_HERE, "lib", "liblamfast_b200.so")

LF_OK = 0
LF_ERR_INVALID_ARGUMENT = 1
LF_ERR_DOMAIN = 2
LF_ERR_LOGIC = 3
LF_ERR_RUNTIME = 4
LF_ERR_CUDA = 5
LF_ERR_OUT_OF_MEMORY = 6
LF_ERR_UNSUPPORTED = 7

LF_BACKEND_STANDARD = 0
LF_BACKEND_FAST = 1
LF_BACKEND_VOIGT_FREE = 2

LF_GEOM_PLANAR = 0
LF_GEOM_BILINEAR = 1
LF_GEOM_FRAMES = 2

BACKENDS = {"standard": LF_BACKEND_STANDARD, "fast": LF_BACKEND_FAST,
            "voigt_free": LF_BACKEND_VOIGT_FREE}


class Orthotropic(ctypes.Structure):
    _fields_ = [(n, c_double) for n in
                ("E1", "E2", "E3", "G12", "G13", "G23", "nu12", "nu13", "nu23")]


class Layer(ctypes.Structure):
    _fields_ = [("constants", Orthotropic), ("angle", c_double)]


class Problem(ctypes.Structure):
    _fields_ = [
        ("degree_u", c_int32), ("degree_v", c_int32), ("degree_t", c_int32),
        ("n_knots_u", c_int32), ("n_knots_v", c_int32), ("n_knots_t", c_int32),
        ("knots_u", POINTER(c_double)), ("knots_v", POINTER(c_double)),
        ("knots_t", POINTER(c_double)),
        ("n_layers", c_int32),
        ("interfaces", POINTER(c_double)),
        ("layers", POINTER(Layer)),
        ("geometry_kind", c_int32),
        ("geometry", c_double * 12),
        ("direction", c_double * 3),
        ("frames", POINTER(c_double)),
        ("inplane_points", c_int32), ("thickness_points", c_int32),
        ("n_active_layers", c_int32),
        ("active_layers", POINTER(c_int32)),
        ("decompose_angles", c_int32),
        ("threads", c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [("qpoint_visits", c_int64), ("frame_evaluations", c_int64),
                ("operator_builds", c_int32), ("reserved", c_int32)]


class LamfastError(RuntimeError):
    """Raised for a non-zero lf_status; ``kind`` names the reference exception."""

    KINDS = {LF_ERR_INVALID_ARGUMENT: "invalid_argument", LF_ERR_DOMAIN: "domain_error",
             LF_ERR_LOGIC: "logic_error", LF_ERR_RUNTIME: "runtime_error",
             LF_ERR_CUDA: "runtime_error", LF_ERR_OUT_OF_MEMORY: "bad_alloc",
             LF_ERR_UNSUPPORTED: "unsupported"}

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = self.KINDS.get(status, "unknown")
        super().__init__(f"[{self.kind}] {message}")


_P = POINTER
# (name, restype, argtypes) for every symbol of include/lamfast_cuda.h
SIGNATURES = [
    ("lf_abi_version", c_int, []),
    ("lf_status_name", c_char_p, [c_int]),
    ("lf_last_error", c_char_p, []),
    ("lf_device_count", c_int, []),
    ("lf_voigt_from_constants", c_int, [_P(Orthotropic), _P(c_double)]),
    ("lf_rotate_inplane", c_int, [_P(c_double), c_double, _P(c_double)]),
    ("lf_angle_decomposition", c_int, [_P(Orthotropic), _P(c_double)]),
    ("lf_bracket_parameters", c_int, [_P(Orthotropic), _P(c_double)]),
    ("lf_gauss_legendre", c_int, [c_int32, c_double, c_double, _P(c_double), _P(c_double)]),
    ("lf_basis_eval", c_int, [c_int32, c_int32, _P(c_double), c_double, _P(c_int32), _P(c_double),
                              _P(c_double)]),
    ("lf_contraction_table", c_int, [_P(c_double), c_double, _P(c_double)]),
    ("lf_layup_configs", c_int, [_P(Problem), _P(c_int32), _P(c_int32), _P(c_double)]),
    ("lf_operator_terms", c_int, [_P(Problem), c_int, _P(c_int32), _P(c_double), _P(c_int32), _P(c_int32)]),
    ("lf_pattern_size", c_int, [_P(Problem), c_int, _P(c_int64), _P(c_int64)]),
    ("lf_pattern_columns", c_int, [_P(Problem), c_int, c_int64, c_int64, _P(c_int32), _P(c_int64)]),
    ("lf_slab_bounds", c_int, [_P(Problem), c_int, c_int, c_int, _P(c_int32), _P(c_int32),
                               _P(c_int64), _P(c_int64), _P(c_int64), _P(c_int64)]),
    ("lf_slab_bounds_functions", c_int, [_P(Problem), c_int, c_int, c_int, _P(c_int64), _P(c_int64),
                                         _P(c_int64), _P(c_int64), _P(c_int64), _P(c_int64)]),
    ("lf_plan_create", c_int, [_P(Problem), c_int, c_int, c_void_p, c_int32, c_int32,
                               _P(c_void_p)]),
    ("lf_plan_create_range", c_int, [_P(Problem), c_int, c_int, c_void_p, c_int64, c_int64,
                                     _P(c_void_p)]),
    ("lf_plan_destroy", c_int, [c_void_p]),
    ("lf_plan_info", c_int, [c_void_p, _P(c_int64), _P(c_int64), _P(c_int64), _P(c_int64)]),
    ("lf_plan_build_pattern", c_int, [c_void_p, c_void_p, c_void_p]),
    ("lf_plan_assemble", c_int, [c_void_p, c_void_p]),
    ("lf_plan_launch_count", c_int, [c_void_p]),
    ("lf_plan_combine_form", c_int, [c_void_p]),
    ("lf_plan_kernel_time", c_int, [c_void_p, c_int, _P(c_double), _P(c_int64)]),
    ("lf_plan_stats", c_int, [c_void_p, _P(Stats)]),
    ("lf_plan_synchronize", c_int, [c_void_p]),
    ("lf_assemble", c_int, [_P(Problem), c_int, c_int, c_void_p, c_void_p, c_void_p,
                            _P(Stats)]),
    ("lf_reference_bilinear", c_int, [_P(Problem), _P(c_double), _P(c_double), c_int, _P(c_double)]),
    ("lf_assemble_slab", c_int, [_P(Problem), c_int, c_int, c_int32, c_int32, c_void_p, c_void_p,
                                 c_void_p, _P(Stats)]),
    ("lf_assemble_range", c_int, [_P(Problem), c_int, c_int, c_int64, c_int64, c_void_p, c_void_p,
                                  c_void_p, _P(Stats)]),
    ("lf_assemble_stream", c_int, [_P(Problem), c_int, c_int, c_int64, c_void_p, c_void_p, _P(Stats)]),
    ("lf_inplane_operators", c_int, [_P(Problem), _P(c_double), c_int, _P(c_double),
                                     _P(c_char), _P(Stats)]),
    ("lf_inplane_operators_bracket", c_int, [_P(Problem), _P(c_double), c_int,
                                             _P(c_double), _P(c_char), _P(Stats)]),
    ("lf_thickness_operators", c_int, [c_int32, c_int32, _P(c_double), c_int32,
                                       _P(c_double), c_int32, c_int, _P(c_double),
                                       _P(c_char)]),
    ("lf_combine", c_int, [_P(Problem), c_int32, _P(c_double), _P(c_char), _P(c_double),
                           _P(c_char), c_int, _P(c_int64), c_void_p, c_void_p, c_void_p]),
    ("lf_csr_frobenius_sq", c_int, [c_int64, c_void_p, c_void_p, c_void_p, _P(c_double)]),
    ("lf_csr_spmv", c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                            c_void_p]),
    ("lf_csr_diff_sq", c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_void_p, c_void_p, _P(c_double)]),
    ("lf_csr_symmetry_sq", c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                   _P(c_double)]),
    ("lf_csr_symmetry_sq_slab", c_int, [c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                        _P(c_double), _P(c_int64)]),
    ("lf_plan_symmetry_sq", c_int, [c_void_p, c_void_p, _P(c_double)]),
    ("lf_release_memory", c_int, [c_int]),
]

# lf_chunk_sink
CHUNK_SINK = ctypes.CFUNCTYPE(c_int, c_void_p, c_int64, c_int64, c_int64, c_int64, POINTER(c_int64),
                              POINTER(c_int32), POINTER(c_double))

_lib = None


def library() -> ctypes.CDLL:
    """Loads the in-tree CUDA library (no fallback: raises if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                "There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != LF_OK:
        msg = library().lf_last_error().decode(errors="replace")
        raise LamfastError(status, msg)
