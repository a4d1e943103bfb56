"""Python host API over the C ABI (include/lamfast_cuda.h).

Mirrors the reference's assembly entry points (reference proj/include):

  assemble_fast / assemble_standard / assemble_voigt_free / assemble_with
      -> assembleFast (fast.hpp:95), assembleStandard (assembly.hpp:52),
         assembleVoigtFree (voigt_free.hpp:69), assembleWith (bench.hpp:19)
  compute_inplane_operators / compute_inplane_operators_bracket
      -> computeInplaneOperators (fast.hpp:65), computeInplaneOperatorsBracket
  compute_thickness_operators -> computeThicknessOperators (fast.hpp:73)
  combine_operators           -> combineOperators (fast.hpp:86)

Errors raise ``LamfastError`` whose ``kind`` names the reference exception
(invalid_argument, domain_error, logic_error, runtime_error).  Results are CSR
triples ``(row_ptr int64, cols int32, values float64)`` like StiffnessMatrix.
``Plan`` keeps the problem resident on a device for the bench / slab path.
"""
from __future__ import annotations

import ctypes
from ctypes import POINTER, byref, c_char, c_double, c_int32, c_int64, c_void_p
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import abi
from .problem import LaminateProblem


@dataclass
class CSR:
    """StiffnessMatrix (sparse.hpp:56-81) as numpy arrays."""
    row_ptr: np.ndarray
    cols: np.ndarray
    values: np.ndarray
    stats: Optional[abi.Stats] = None

    @property
    def dim(self) -> int:
        return len(self.row_ptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1] - self.row_ptr[0])

    def astuple(self):
        return self.row_ptr, self.cols, self.values


def _dp(a: np.ndarray):
    return a.ctypes.data_as(POINTER(c_double))


def pattern_size(prob: LaminateProblem, backend: str = "fast") -> Tuple[int, int]:
    lib = abi.library()
    c = prob.to_c()
    dim, nnz = c_int64(), c_int64()
    abi.check(lib.lf_pattern_size(byref(c), abi.BACKENDS[backend], byref(dim), byref(nnz)))
    return dim.value, nnz.value


def operator_terms(prob: LaminateProblem, backend: str = "fast"):
    """Host-side view of the operator terms a plan combines (lf_operator_terms):
    (tables [n_terms, 81], slot_term [n_t, n_slots] or None when a thickness
    row sees more than three terms)."""
    lib = abi.library()
    c = prob.to_c()
    n, ns = c_int32(), c_int32()
    abi.check(lib.lf_operator_terms(byref(c), abi.BACKENDS[backend], byref(n), None, byref(ns), None))
    tables = np.empty((n.value, 81), dtype=np.float64)
    sched = np.full((prob.n_t, 3), -1, dtype=np.int32)
    abi.check(lib.lf_operator_terms(byref(c), abi.BACKENDS[backend], byref(n), _dp(tables), byref(ns),
                                    sched.ctypes.data_as(POINTER(c_int32))))
    if ns.value == 0:
        return tables, None
    return tables, sched.reshape(-1)[:prob.n_t * ns.value].reshape(prob.n_t, ns.value).copy()


def pattern_columns(prob: LaminateProblem, f_begin: int = 0, f_end: int = -1, backend: str = "fast") -> np.ndarray:
    """Host-written CSR columns of the functions [f_begin, f_end)
    (lf_pattern_columns: the closed form k_pattern_cols writes on the device)."""
    lib = abi.library()
    c = prob.to_c()
    n = c_int64()
    abi.check(lib.lf_pattern_columns(byref(c), abi.BACKENDS[backend], f_begin, f_end, None, byref(n)))
    cols = np.empty(max(1, n.value), dtype=np.int32)
    abi.check(lib.lf_pattern_columns(byref(c), abi.BACKENDS[backend], f_begin, f_end,
                                     cols.ctypes.data_as(POINTER(c_int32)), byref(n)))
    return cols[:n.value]


def slab_bounds(prob: LaminateProblem, n_parts: int, part: int, backend: str = "fast") -> dict:
    lib = abi.library()
    c = prob.to_c()
    t0, t1 = c_int32(), c_int32()
    r0, r1, z0, z1 = c_int64(), c_int64(), c_int64(), c_int64()
    abi.check(lib.lf_slab_bounds(byref(c), abi.BACKENDS[backend], n_parts, part, byref(t0), byref(t1),
                                 byref(r0), byref(r1), byref(z0), byref(z1)))
    return {"t_begin": t0.value, "t_end": t1.value, "row_begin": r0.value, "row_end": r1.value,
            "nnz_begin": z0.value, "nnz_end": z1.value}


def slab_bounds_functions(prob: LaminateProblem, n_parts: int, part: int, backend: str = "fast") -> dict:
    """Row slab cut at function boundaries (f = i_t * n_s + i_s), balanced by
    nnz to within one function (lf_slab_bounds_functions)."""
    lib = abi.library()
    c = prob.to_c()
    f0, f1, r0, r1, z0, z1 = (c_int64() for _ in range(6))
    abi.check(lib.lf_slab_bounds_functions(byref(c), abi.BACKENDS[backend], n_parts, part, byref(f0), byref(f1),
                                           byref(r0), byref(r1), byref(z0), byref(z1)))
    return {"f_begin": f0.value, "f_end": f1.value, "row_begin": r0.value, "row_end": r1.value,
            "nnz_begin": z0.value, "nnz_end": z1.value}


def assemble_stream(prob: LaminateProblem, sink, backend: str = "fast", device: int = 0,
                    max_chunk_nnz: int = 0) -> abi.Stats:
    """Streams the whole matrix through ``sink(row_begin, rows, nnz_begin,
    row_ptr, cols, values)`` chunk by chunk (lf_assemble_stream); the numpy
    arrays are views of pinned staging memory valid only during the call.
    A falsy return continues, a truthy one aborts."""
    lib = abi.library()
    c = prob.to_c()
    err = []

    def cb(_user, row_begin, rows, nnz_begin, nnz, rp, cols, vals):
        try:
            r = np.ctypeslib.as_array(rp, shape=(rows + 1,))
            cc = np.ctypeslib.as_array(cols, shape=(nnz,)) if nnz else np.zeros(0, np.int32)
            vv = np.ctypeslib.as_array(vals, shape=(nnz,)) if nnz else np.zeros(0)
            return 1 if sink(row_begin, rows, nnz_begin, r, cc, vv) else 0
        except Exception as exc:  # re-raised below
            err.append(exc)
            return 1

    fn = abi.CHUNK_SINK(cb)
    st = abi.Stats()
    status = lib.lf_assemble_stream(byref(c), abi.BACKENDS[backend], device, max_chunk_nnz,
                                    ctypes.cast(fn, c_void_p), None, byref(st))
    if err:
        raise err[0]
    abi.check(status)
    return st


def assemble_with(backend: str, prob: LaminateProblem, device: int = 0,
                  out: Optional[Tuple[np.ndarray, np.ndarray, np.ndarray]] = None) -> CSR:
    """One-shot assembly into host buffers (pinned buffers may be passed in
    ``out`` to reach full PCIe bandwidth)."""
    lib = abi.library()
    c = prob.to_c()
    dim, nnz = pattern_size(prob, backend)
    if out is None:
        rp = np.empty(dim + 1, dtype=np.int64)
        cols = np.empty(max(nnz, 1), dtype=np.int32)
        vals = np.empty(max(nnz, 1), dtype=np.float64)
    else:
        rp, cols, vals = out
    st = abi.Stats()
    abi.check(lib.lf_assemble(byref(c), abi.BACKENDS[backend], device, rp.ctypes.data,
                              cols.ctypes.data, vals.ctypes.data, byref(st)))
    return CSR(rp, cols[:nnz], vals[:nnz], st)


def assemble_slab(prob: LaminateProblem, t_begin: int, t_end: int, backend: str = "fast", device: int = 0,
                  out: Optional[Tuple] = None) -> CSR:
    """One-shot assembly of the row slab of thickness functions [t_begin,
    t_end) into host buffers (lf_assemble_slab): row offsets rebased to 0,
    global columns -- one rank's part of a multi-GPU assembly.  ``out`` may
    hold (row_ptr, cols, values) numpy arrays or pinned torch tensors."""
    lib = abi.library()
    c = prob.to_c()
    rows = 3 * prob.n_s * (t_end - t_begin)
    if out is None:
        plan = Plan(prob, backend, device, t_begin, t_end) # exact slab sizes for any backend
        nnz = plan.nnz
        plan.close()
        out = (np.empty(rows + 1, dtype=np.int64), np.empty(max(nnz, 1), dtype=np.int32),
               np.empty(max(nnz, 1), dtype=np.float64))
    ptrs = [a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data for a in out]
    st = abi.Stats()
    abi.check(lib.lf_assemble_slab(byref(c), abi.BACKENDS[backend], device, t_begin, t_end, *ptrs, byref(st)))
    rp, cols, vals = out
    nnz = int(rp[rows])
    return CSR(rp[:rows + 1], cols[:nnz], vals[:nnz], st)


def assemble_range(prob: LaminateProblem, f_begin: int, f_end: int, backend: str = "fast", device: int = 0,
                   out: Optional[Tuple] = None) -> CSR:
    """One-shot assembly of the functions [f_begin, f_end) (rows 3 f_begin ..
    3 f_end) into host buffers (lf_assemble_range): a slab cut inside
    thickness rows, row offsets rebased to 0, global columns."""
    lib = abi.library()
    c = prob.to_c()
    rows = 3 * (f_end - f_begin)
    if out is None:
        plan = Plan(prob, backend, device, f_begin=f_begin, f_end=f_end)
        nnz = plan.nnz
        plan.close()
        out = (np.empty(rows + 1, dtype=np.int64), np.empty(max(nnz, 1), dtype=np.int32),
               np.empty(max(nnz, 1), dtype=np.float64))
    ptrs = [a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data for a in out]
    st = abi.Stats()
    abi.check(lib.lf_assemble_range(byref(c), abi.BACKENDS[backend], device, f_begin, f_end, *ptrs, byref(st)))
    rp, cols, vals = out
    nnz = int(rp[rows])
    return CSR(rp[:rows + 1], cols[:nnz], vals[:nnz], st)


def reference_bilinear(prob: LaminateProblem, v: np.ndarray, u: np.ndarray, device: int = 0) -> float:
    """v^T K u by full 3D quadrature on the device without forming K
    (referenceBilinear, assembly.cpp:247-318; lf_reference_bilinear)."""
    lib = abi.library()
    c = prob.to_c()
    v = np.ascontiguousarray(v, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    if v.size != prob.dim or u.size != prob.dim:
        raise ValueError("referenceBilinear: coefficient length mismatch")
    out = c_double()
    abi.check(lib.lf_reference_bilinear(byref(c), v.ctypes.data_as(POINTER(c_double)),
                                        u.ctypes.data_as(POINTER(c_double)), device, byref(out)))
    return out.value


def assemble_fast(prob: LaminateProblem, device: int = 0) -> CSR:
    return assemble_with("fast", prob, device)


def assemble_standard(prob: LaminateProblem, device: int = 0) -> CSR:
    return assemble_with("standard", prob, device)


def assemble_voigt_free(prob: LaminateProblem, device: int = 0) -> CSR:
    return assemble_with("voigt_free", prob, device)


def compute_inplane_operators(prob: LaminateProblem, material: np.ndarray, device: int = 0,
                              bracket_table: Optional[np.ndarray] = None):
    """Banded InPlaneOperatorSet: blocks[4, n_s, 2p_v+1, 2p_u+1, 3, 3], flags."""
    lib = abi.library()
    c = prob.to_c()
    bu, bv = 2 * prob.degree_u + 1, 2 * prob.degree_v + 1
    blocks = np.zeros((4, prob.n_s, bv, bu, 3, 3))
    flags = np.zeros((prob.n_s, bv, bu), dtype=np.int8)
    st = abi.Stats()
    fp = flags.ctypes.data_as(POINTER(c_char))
    if bracket_table is not None:
        t = np.ascontiguousarray(bracket_table, dtype=np.float64).reshape(81)
        abi.check(lib.lf_inplane_operators_bracket(byref(c), _dp(t), device, _dp(blocks), fp, byref(st)))
    else:
        m = np.ascontiguousarray(material, dtype=np.float64).reshape(36)
        abi.check(lib.lf_inplane_operators(byref(c), _dp(m), device, _dp(blocks), fp, byref(st)))
    return blocks, flags, st


def compute_thickness_operators(degree: int, knots, interfaces, pts: int, device: int = 0):
    """ThicknessOperators: q[n_layers, 4, n_t, n_t], occupied[n_t, n_t]."""
    lib = abi.library()
    k = np.ascontiguousarray(knots, dtype=np.float64)
    f = np.ascontiguousarray(interfaces, dtype=np.float64)
    nt = len(k) - degree - 1
    q = np.zeros((len(f) - 1, 4, nt, nt))
    occ = np.zeros((nt, nt), dtype=np.int8)
    abi.check(lib.lf_thickness_operators(degree, len(k), _dp(k), len(f), _dp(f), pts, device, _dp(q),
                                         occ.ctypes.data_as(POINTER(c_char))))
    return q, occ


def combine_operators(prob: LaminateProblem, blocks: np.ndarray, flags: np.ndarray,
                      thickness: np.ndarray, occupied: np.ndarray, device: int = 0) -> CSR:
    """combineOperators over explicit terms: blocks[T,4,n_s,bv,bu,3,3] (or a list
    of per-term [4,...] arrays), thickness[T,4,n_t,n_t]."""
    lib = abi.library()
    c = prob.to_c()
    b = np.ascontiguousarray(blocks, dtype=np.float64)
    th = np.ascontiguousarray(thickness, dtype=np.float64)
    n_terms = th.shape[0]
    fl = np.ascontiguousarray(flags, dtype=np.int8)
    oc = np.ascontiguousarray(occupied, dtype=np.int8)
    nnz = c_int64()
    args = (byref(c), n_terms, _dp(b), fl.ctypes.data_as(POINTER(c_char)), _dp(th),
            oc.ctypes.data_as(POINTER(c_char)), device, byref(nnz))
    abi.check(lib.lf_combine(*args, None, None, None))
    rp = np.empty(prob.dim + 1, dtype=np.int64)
    cols = np.empty(max(1, nnz.value), dtype=np.int32)
    vals = np.empty(max(1, nnz.value), dtype=np.float64)
    abi.check(lib.lf_combine(*args, rp.ctypes.data, cols.ctypes.data, vals.ctypes.data))
    return CSR(rp, cols[:nnz.value], vals[:nnz.value])


class Plan:
    """A problem resident on one device (lf_plan): tables uploaded once,
    ``assemble(values)`` runs the whole hot path into a device buffer.

    Device buffers are torch tensors (torch is plumbing here: allocation and
    streams only)."""

    def __init__(self, prob: LaminateProblem, backend: str = "fast", device: int = 0,
                 t_begin: int = 0, t_end: int = -1, stream=None, f_begin: Optional[int] = None,
                 f_end: Optional[int] = None):
        """Rows of the thickness functions [t_begin, t_end), or -- with
        f_begin / f_end -- of the functions [f_begin, f_end) (a slab cut
        inside thickness rows, lf_plan_create_range)."""
        self.lib = abi.library()
        self.prob = prob
        self.backend = backend
        self.device = device
        self._c = prob.to_c()
        h = c_void_p()
        sp = c_void_p(stream) if stream else None
        if f_begin is not None:
            abi.check(self.lib.lf_plan_create_range(byref(self._c), abi.BACKENDS[backend], device, sp,
                                                    f_begin, -1 if f_end is None else f_end, byref(h)))
        else:
            abi.check(self.lib.lf_plan_create(byref(self._c), abi.BACKENDS[backend], device, sp,
                                              t_begin, t_end, byref(h)))
        self.handle = h
        rows, nnz, r0, z0 = c_int64(), c_int64(), c_int64(), c_int64()
        abi.check(self.lib.lf_plan_info(h, byref(rows), byref(nnz), byref(r0), byref(z0)))
        self.rows, self.nnz, self.row_begin, self.nnz_begin = rows.value, nnz.value, r0.value, z0.value

    def build_pattern(self, row_ptr_ptr: int, cols_ptr: int) -> None:
        abi.check(self.lib.lf_plan_build_pattern(self.handle, c_void_p(row_ptr_ptr), c_void_p(cols_ptr)))

    def assemble(self, values_ptr: int) -> None:
        abi.check(self.lib.lf_plan_assemble(self.handle, c_void_p(values_ptr)))

    def synchronize(self) -> None:
        abi.check(self.lib.lf_plan_synchronize(self.handle))

    @property
    def launch_count(self) -> int:
        return self.lib.lf_plan_launch_count(self.handle)

    @property
    def combine_form(self) -> str:
        """Combine kernel form the plan chose: per-term, slots or coefficient."""
        return {0: "per-term", 1: "slots", 2: "coefficient"}.get(self.lib.lf_plan_combine_form(self.handle), "none")

    def kernel_time(self, reset: bool = False) -> Tuple[float, int]:
        ms, n = c_double(), c_int64()
        abi.check(self.lib.lf_plan_kernel_time(self.handle, 1 if reset else 0, byref(ms), byref(n)))
        return ms.value, n.value

    def symmetry_sq(self, values_ptr: int) -> float:
        """||K - K^T||_F^2 numerator of symmetryRelError over this plan's slab
        (entries whose mirror row is in the slab), from the closed-form pattern
        (lf_plan_symmetry_sq)."""
        out = c_double()
        abi.check(self.lib.lf_plan_symmetry_sq(self.handle, c_void_p(values_ptr), byref(out)))
        return out.value

    def stats(self) -> abi.Stats:
        st = abi.Stats()
        abi.check(self.lib.lf_plan_stats(self.handle, byref(st)))
        return st

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.lf_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def device_csr_stats(rows: int, row_ptr_ptr: int, cols_ptr: int, values_ptr: int, stream: int = 0,
                     row_begin: int = 0) -> dict:
    """||K||_F^2 and ||K - K^T||_F^2 on the device (sparse.cpp:66-95) of a
    CSR holding the global rows [row_begin, row_begin + rows); for a slab the
    symmetry sum covers the entries whose mirror row is in the slab."""
    lib = abi.library()
    fro, sym, skipped = c_double(), c_double(), c_int64()
    abi.check(lib.lf_csr_frobenius_sq(rows, c_void_p(row_ptr_ptr), c_void_p(values_ptr),
                                      c_void_p(stream), byref(fro)))
    abi.check(lib.lf_csr_symmetry_sq_slab(rows, row_begin, c_void_p(row_ptr_ptr), c_void_p(cols_ptr),
                                          c_void_p(values_ptr), c_void_p(stream), byref(sym),
                                          byref(skipped)))
    return {"fro_sq": fro.value, "sym_sq": sym.value, "sym_skipped": skipped.value}


def release_memory(device: int = 0) -> None:
    """Returns the library's cached device memory to the driver (lf_release_memory)."""
    abi.check(abi.library().lf_release_memory(device))
