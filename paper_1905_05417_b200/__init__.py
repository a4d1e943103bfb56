"""B200-native laminate stiffness assembly (arXiv 1905.05417, reference `lamfast`).

The hot path -- fast (Kronecker-type) assembly of the 3D elastic stiffness
of a multi-ply laminate, plus the standard full-3D quadrature cross-check --
runs as hand-written sm_100a CUDA kernels behind a C ABI
(include/lamfast_cuda.h, lib/liblamfast_b200.so).  This package is the thin
Python host layer over that ABI; see DESIGN.md.
"""
from .abi import LamfastError, library
from .assembler import (CSR, Plan, assemble_fast, assemble_range, assemble_slab, assemble_stream, reference_bilinear, assemble_standard, assemble_voigt_free,
                        assemble_with, combine_operators, compute_inplane_operators,
                        compute_thickness_operators, device_csr_stats, operator_terms, pattern_columns, pattern_size, release_memory,
                        slab_bounds, slab_bounds_functions)
from .problem import (LaminateProblem, baseline_config, baseline_orthotropic, c0_knots,
                      cube_problem, equal_interfaces, isotropic, pagano, plate, sizes,
                      uniform_knots)

__all__ = [
    "reference_bilinear",
    "assemble_slab", "assemble_range", "assemble_stream", "slab_bounds_functions",
    "LamfastError", "library", "CSR", "Plan", "assemble_fast", "assemble_standard",
    "assemble_voigt_free", "assemble_with", "combine_operators", "compute_inplane_operators",
    "compute_thickness_operators", "device_csr_stats", "operator_terms", "pattern_columns", "pattern_size", "release_memory", "slab_bounds",
    "LaminateProblem", "baseline_config", "baseline_orthotropic", "c0_knots", "cube_problem",
    "equal_interfaces", "isotropic", "pagano", "plate", "sizes", "uniform_knots",
]
