"""TEST INFRASTRUCTURE: Python access to the two CPU checkers.

  * ``Oracle`` -- the C restatement oracle/lamfast_oracle.c (always available:
    built by oracle/build_oracle.sh, travels to the GPU box as a .so).
  * ``Reference`` -- the unmodified reference sources compiled by
    oracle/build_ref.sh into oracle/_ref/libref_lamfast.so.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
--impl reference arm) may import this module.  Nothing in the product
package imports it.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_double, c_int, c_int32, c_int64

import numpy as np

from paper_1905_05417_b200 import abi
from paper_1905_05417_b200.problem import LaminateProblem

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblamfast_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_lamfast.so")

_dp = POINTER(c_double)
_P = abi.Problem


def _d(a):
    return a.ctypes.data_as(_dp)


class CheckerError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.kind = abi.LamfastError.KINDS.get(status, "unknown")
        super().__init__(f"[{self.kind}] {msg}")


class _Base:
    def _check(self, st):
        if st != 0:
            raise CheckerError(st, self.lib_error())


class Oracle(_Base):
    """C restatement of the reference algorithm (oracle/lamfast_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run oracle/build_oracle.sh")
        lib = ctypes.CDLL(path)
        sig = {
            "orc_last_error": (ctypes.c_char_p, []),
            "orc_basis_eval": (c_int, [c_int, c_int, _dp, c_double, POINTER(c_int), _dp, _dp]),
            "orc_gauss": (None, [c_int, c_double, c_double, _dp, _dp]),
            "orc_voigt_from_constants": (c_int, [POINTER(abi.Orthotropic), _dp]),
            "orc_rotate_inplane": (None, [_dp, c_double, _dp]),
            "orc_angle_decomposition": (c_int, [POINTER(abi.Orthotropic), _dp]),
            "orc_layup": (c_int, [POINTER(_P), POINTER(c_int), POINTER(c_int), _dp]),
            "orc_frame_at": (c_int, [POINTER(_P), c_double, c_double, _dp]),
            "orc_inplane_operators": (c_int, [POINTER(_P), _dp, _dp, POINTER(c_char)]),
            "orc_thickness_operators": (c_int, [c_int, c_int, _dp, c_int, _dp, c_int, _dp,
                                                POINTER(c_char)]),
            "orc_assemble_fast": (c_int, [POINTER(_P), c_int, c_int, POINTER(c_int64),
                                          POINTER(c_int32), _dp, POINTER(c_int64),
                                          POINTER(abi.Stats)]),
            "orc_fast_create": (c_int, [POINTER(_P), c_int, POINTER(ctypes.c_void_p)]),
            "orc_fast_destroy": (None, [ctypes.c_void_p]),
            "orc_fast_slab": (c_int, [ctypes.c_void_p, c_int, c_int, POINTER(c_int64), POINTER(c_int32), _dp,
                                      POINTER(c_int64)]),
            "orc_assemble_standard": (c_int, [POINTER(_P), c_int, c_int, POINTER(c_int64),
                                              POINTER(c_int32), _dp, POINTER(c_int64),
                                              POINTER(abi.Stats)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    def lib_error(self):
        return self.lib.orc_last_error().decode()

    def basis(self, degree, knots, x):
        k = np.ascontiguousarray(knots, dtype=np.float64)
        v = np.zeros(degree + 1)
        d = np.zeros(degree + 1)
        first = c_int()
        self._check(self.lib.orc_basis_eval(degree, len(k), _d(k), x, ctypes.byref(first),
                                            _d(v), _d(d)))
        return first.value, v, d

    def gauss(self, n, a=-1.0, b=1.0):
        p = np.zeros(n)
        w = np.zeros(n)
        self.lib.orc_gauss(n, a, b, _d(p), _d(w))
        return p, w

    def stiffness(self, constants, angle=0.0):
        d = np.zeros(36)
        self._check(self.lib.orc_voigt_from_constants(ctypes.byref(abi.Orthotropic(*constants)),
                                                      _d(d)))
        out = np.zeros(36)
        self.lib.orc_rotate_inplane(_d(d), angle, _d(out))
        return out.reshape(6, 6)

    def angle_decomposition(self, constants):
        out = np.zeros(180)
        self._check(self.lib.orc_angle_decomposition(
            ctypes.byref(abi.Orthotropic(*constants)), _d(out)))
        return out.reshape(5, 6, 6)

    def frame(self, prob: LaminateProblem, u, v):
        out = np.zeros(19)
        c = prob.to_c()
        self._check(self.lib.orc_frame_at(ctypes.byref(c), u, v, _d(out)))
        return out

    def inplane_operators(self, prob: LaminateProblem, material):
        c = prob.to_c()
        m = np.ascontiguousarray(material, dtype=np.float64).reshape(36)
        bu, bv = 2 * prob.degree_u + 1, 2 * prob.degree_v + 1
        blocks = np.zeros((4, prob.n_s, bv, bu, 3, 3))
        flags = np.zeros((prob.n_s, bv, bu), dtype=np.int8)
        self._check(self.lib.orc_inplane_operators(
            ctypes.byref(c), _d(m), _d(blocks), flags.ctypes.data_as(POINTER(c_char))))
        return blocks, flags

    def thickness_operators(self, degree, knots, interfaces, pts):
        k = np.ascontiguousarray(knots, dtype=np.float64)
        f = np.ascontiguousarray(interfaces, dtype=np.float64)
        nt = len(k) - degree - 1
        q = np.zeros((len(f) - 1, 4, nt, nt))
        occ = np.zeros((nt, nt), dtype=np.int8)
        self._check(self.lib.orc_thickness_operators(degree, len(k), _d(k), len(f), _d(f), pts,
                                                     _d(q), occ.ctypes.data_as(POINTER(c_char))))
        return q, occ

    def fast_terms(self, prob: LaminateProblem, want_values: bool = True) -> "FastTerms":
        return FastTerms(self, prob, want_values)

    def assemble(self, prob: LaminateProblem, backend="fast", t0=0, t1=-1, want_stats=False):
        """(row_ptr, cols, values[, stats]) of the rows of thickness functions [t0, t1)."""
        fn = {"fast": self.lib.orc_assemble_fast, "voigt_free": self.lib.orc_assemble_fast,
              "standard": self.lib.orc_assemble_standard}[backend]
        if backend == "voigt_free" and prob.decompose_angles:
            prob = prob.replace(decompose_angles=False)
        c = prob.to_c()
        if t1 < 0:
            t1 = prob.n_t
        rows = 3 * prob.n_s * (t1 - t0)
        rp = np.zeros(rows + 1, dtype=np.int64)
        nnz = c_int64()
        self._check(fn(ctypes.byref(c), t0, t1, rp.ctypes.data_as(POINTER(c_int64)), None, None,
                       ctypes.byref(nnz), None))
        cols = np.zeros(max(1, nnz.value), dtype=np.int32)
        vals = np.zeros(max(1, nnz.value), dtype=np.float64)
        st = abi.Stats()
        self._check(fn(ctypes.byref(c), t0, t1, rp.ctypes.data_as(POINTER(c_int64)),
                       cols.ctypes.data_as(POINTER(c_int32)), _d(vals), ctypes.byref(nnz),
                       ctypes.byref(st)))
        out = (rp, cols[:nnz.value], vals[:nnz.value])
        return out + (st,) if want_stats else out


class FastTerms:
    """Operator terms of one problem built once by the oracle (orc_fast_*):
    ``slab(t0, t1)`` combines any row slab, ``nnz_before(t)`` is the global
    offset of thickness function t (the oracle's row_ptr of rows [0, t))."""

    def __init__(self, oracle: "Oracle", prob: LaminateProblem, want_values: bool = True):
        self.o = oracle
        self.prob = prob
        self._c = prob.to_c()
        h = ctypes.c_void_p()
        oracle._check(oracle.lib.orc_fast_create(ctypes.byref(self._c), 1 if want_values else 0,
                                                 ctypes.byref(h)))
        self.h = h

    def slab(self, t0, t1):
        rows = 3 * self.prob.n_s * (t1 - t0)
        rp = np.zeros(rows + 1, dtype=np.int64)
        nnz = c_int64()
        lib = self.o.lib
        self.o._check(lib.orc_fast_slab(self.h, t0, t1, rp.ctypes.data_as(POINTER(c_int64)), None, None,
                                        ctypes.byref(nnz)))
        cols = np.zeros(max(1, nnz.value), dtype=np.int32)
        vals = np.zeros(max(1, nnz.value), dtype=np.float64)
        self.o._check(lib.orc_fast_slab(self.h, t0, t1, rp.ctypes.data_as(POINTER(c_int64)),
                                        cols.ctypes.data_as(POINTER(c_int32)), _d(vals), ctypes.byref(nnz)))
        return rp, cols[:nnz.value], vals[:nnz.value]

    def row_offsets(self, t0, t1):
        """Slab-local row offsets of thickness rows [t0, t1) (no values)."""
        rows = 3 * self.prob.n_s * (t1 - t0)
        rp = np.zeros(rows + 1, dtype=np.int64)
        nnz = c_int64()
        self.o._check(self.o.lib.orc_fast_slab(self.h, t0, t1, rp.ctypes.data_as(POINTER(c_int64)), None, None,
                                               ctypes.byref(nnz)))
        return rp

    def function_offset(self, f):
        """Global CSR offset of the first entry of function f = i_t n_s + i_s."""
        ns = self.prob.n_s
        t, i = divmod(f, ns)
        if t >= self.prob.n_t:
            return self.nnz_before(self.prob.n_t)
        return self.nnz_before(t) + int(self.row_offsets(t, t + 1)[3 * i])

    def nnz_before(self, t):
        nnz = c_int64()
        self.o._check(self.o.lib.orc_fast_slab(self.h, 0, t, None, None, None, ctypes.byref(nnz)))
        return nnz.value

    def close(self):
        if self.h:
            self.o.lib.orc_fast_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RefCsr(ctypes.Structure):
    _fields_ = [("dim", c_int64), ("nnz", c_int64), ("row_ptr", POINTER(c_int64)),
                ("cols", POINTER(c_int32)), ("values", _dp)]


class Reference(_Base):
    """The unmodified reference compiled from /root/reference (oracle/_ref)."""

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise ImportError(f"{path} missing: run oracle/build_ref.sh where /root/reference exists")
        lib = ctypes.CDLL(path)
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_csr_free": (None, [POINTER(RefCsr)]),
            "ref_assemble": (c_int, [POINTER(_P), c_int, c_int, POINTER(RefCsr),
                                     POINTER(abi.Stats)]),
            "ref_basis_eval": (c_int, [c_int, c_int, _dp, c_double, POINTER(c_int), _dp, _dp]),
            "ref_gauss": (c_int, [c_int, c_double, c_double, _dp, _dp]),
            "ref_stiffness": (c_int, [POINTER(abi.Orthotropic), c_double, _dp]),
            "ref_angle_decomposition": (c_int, [POINTER(abi.Orthotropic), _dp]),
            "ref_bracket_parameters": (c_int, [POINTER(abi.Orthotropic), _dp]),
            "ref_contraction_table": (c_int, [POINTER(abi.Orthotropic), c_double, _dp]),
            "ref_thickness_operators": (c_int, [c_int, c_int, _dp, c_int, _dp, c_int, _dp,
                                                POINTER(c_char)]),
            "ref_inplane_operators": (c_int, [POINTER(_P), _dp, _dp, POINTER(c_char),
                                              POINTER(abi.Stats)]),
            "ref_inplane_operators_bracket": (c_int, [POINTER(_P), POINTER(abi.Orthotropic),
                                                      c_double, _dp, POINTER(c_char)]),
            "ref_frame_at": (c_int, [POINTER(_P), c_double, c_double, _dp]),
            "ref_bilinear": (c_int, [POINTER(_P), _dp, _dp, c_int64, _dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    def lib_error(self):
        return self.lib.ref_last_error().decode()

    def assemble(self, prob: LaminateProblem, backend="fast", threads=1, want_stats=False):
        c = prob.to_c()
        out = RefCsr()
        st = abi.Stats()
        self._check(self.lib.ref_assemble(ctypes.byref(c), abi.BACKENDS[backend], threads,
                                          ctypes.byref(out), ctypes.byref(st)))
        try:
            rp = np.ctypeslib.as_array(out.row_ptr, shape=(out.dim + 1,)).copy()
            if out.nnz:
                cols = np.ctypeslib.as_array(out.cols, shape=(out.nnz,)).copy()
                vals = np.ctypeslib.as_array(out.values, shape=(out.nnz,)).copy()
            else:
                cols = np.zeros(0, np.int32)
                vals = np.zeros(0)
        finally:
            self.lib.ref_csr_free(ctypes.byref(out))
        res = (rp, cols, vals)
        return res + (st,) if want_stats else res

    def basis(self, degree, knots, x):
        k = np.ascontiguousarray(knots, dtype=np.float64)
        v = np.zeros(degree + 1)
        d = np.zeros(degree + 1)
        first = c_int()
        self._check(self.lib.ref_basis_eval(degree, len(k), _d(k), x, ctypes.byref(first),
                                            _d(v), _d(d)))
        return first.value, v, d

    def gauss(self, n, a=-1.0, b=1.0):
        p = np.zeros(n)
        w = np.zeros(n)
        self._check(self.lib.ref_gauss(n, a, b, _d(p), _d(w)))
        return p, w

    def stiffness(self, constants, angle=0.0):
        out = np.zeros(36)
        self._check(self.lib.ref_stiffness(ctypes.byref(abi.Orthotropic(*constants)), angle,
                                           _d(out)))
        return out.reshape(6, 6)

    def angle_decomposition(self, constants):
        out = np.zeros(180)
        self._check(self.lib.ref_angle_decomposition(ctypes.byref(abi.Orthotropic(*constants)),
                                                     _d(out)))
        return out.reshape(5, 6, 6)

    def bracket_parameters(self, constants):
        out = np.zeros(9)
        self._check(self.lib.ref_bracket_parameters(ctypes.byref(abi.Orthotropic(*constants)),
                                                    _d(out)))
        return out

    def contraction_table(self, constants, angle):
        out = np.zeros(81)
        self._check(self.lib.ref_contraction_table(ctypes.byref(abi.Orthotropic(*constants)),
                                                   angle, _d(out)))
        return out

    def thickness_operators(self, degree, knots, interfaces, pts):
        k = np.ascontiguousarray(knots, dtype=np.float64)
        f = np.ascontiguousarray(interfaces, dtype=np.float64)
        nt = len(k) - degree - 1
        q = np.zeros((len(f) - 1, 4, nt, nt))
        occ = np.zeros((nt, nt), dtype=np.int8)
        self._check(self.lib.ref_thickness_operators(degree, len(k), _d(k), len(f), _d(f), pts,
                                                     _d(q), occ.ctypes.data_as(POINTER(c_char))))
        return q, occ

    def inplane_operators(self, prob: LaminateProblem, material):
        c = prob.to_c()
        m = np.ascontiguousarray(material, dtype=np.float64).reshape(36)
        bu, bv = 2 * prob.degree_u + 1, 2 * prob.degree_v + 1
        blocks = np.zeros((4, prob.n_s, bv, bu, 3, 3))
        flags = np.zeros((prob.n_s, bv, bu), dtype=np.int8)
        st = abi.Stats()
        self._check(self.lib.ref_inplane_operators(ctypes.byref(c), _d(m), _d(blocks),
                                                   flags.ctypes.data_as(POINTER(c_char)),
                                                   ctypes.byref(st)))
        return blocks, flags

    def inplane_operators_bracket(self, prob: LaminateProblem, constants, angle):
        c = prob.to_c()
        bu, bv = 2 * prob.degree_u + 1, 2 * prob.degree_v + 1
        blocks = np.zeros((4, prob.n_s, bv, bu, 3, 3))
        flags = np.zeros((prob.n_s, bv, bu), dtype=np.int8)
        self._check(self.lib.ref_inplane_operators_bracket(
            ctypes.byref(c), ctypes.byref(abi.Orthotropic(*constants)), angle, _d(blocks),
            flags.ctypes.data_as(POINTER(c_char))))
        return blocks, flags

    def frame(self, prob: LaminateProblem, u, v):
        out = np.zeros(19)
        c = prob.to_c()
        self._check(self.lib.ref_frame_at(ctypes.byref(c), u, v, _d(out)))
        return out

    def bilinear(self, prob: LaminateProblem, v, u):
        c = prob.to_c()
        v = np.ascontiguousarray(v, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = c_double()
        self._check(self.lib.ref_bilinear(ctypes.byref(c), _d(v), _d(u), len(v),
                                          ctypes.byref(out)))
        return out.value


def csr_rel_diff(a, b):
    """frobeniusRelDiff (sparse.cpp:108-139) on (row_ptr, cols, values) tuples."""
    import scipy.sparse as sp
    n = len(a[0]) - 1
    A = sp.csr_matrix((a[2], a[1], a[0]), shape=(n, n))
    B = sp.csr_matrix((b[2], b[1], b[0]), shape=(n, n))
    d = sp.linalg.norm(A - B) if (A - B).nnz else 0.0
    den = max(np.sqrt(np.dot(a[2], a[2])), np.sqrt(np.dot(b[2], b[2])))
    return 0.0 if den == 0 else d / den


def slab_oracle_delta(prob: LaminateProblem, f_begin: int, f_end: int, row_ptr, cols, values) -> float:
    """max |K - K_oracle| / max |K_oracle| over one sampled thickness row of a
    rank's row slab: the functions of the thickness row that
    holds the slab's middle function, restricted to the slab [f_begin, f_end)
    (row_ptr / cols / values: the slab's CSR, rows from 3 f_begin, any array
    type), compared with the oracle's rows of that thickness function.  A
    pattern mismatch returns +inf."""
    import torch
    ns = prob.n_s
    if f_end <= f_begin:
        return 0.0
    t = ((f_begin + f_end) // 2) // ns
    g0, g1 = max(f_begin, t * ns), min(f_end, (t + 1) * ns)
    terms = Oracle().fast_terms(prob)
    orp, oc, ov = terms.slab(t, t + 1)
    terms.close()
    a, b = 3 * (g0 - t * ns), 3 * (g1 - t * ns)
    want = (orp[a:b + 1] - orp[a], oc[orp[a]:orp[b]], ov[orp[a]:orp[b]])
    rp = torch.as_tensor(row_ptr)
    la, lb = 3 * (g0 - f_begin), 3 * (g1 - f_begin)
    z0, z1 = int(rp[la]), int(rp[lb])
    got_rp = (rp[la:lb + 1] - z0).cpu().numpy()
    got_c = torch.as_tensor(cols)[z0:z1].cpu().numpy()
    got_v = torch.as_tensor(values)[z0:z1].cpu().numpy()
    if not (np.array_equal(got_rp, want[0]) and np.array_equal(got_c, want[1])):
        return float("inf")
    scale = float(np.abs(want[2]).max()) if len(want[2]) else 0.0
    return float(np.abs(got_v - want[2]).max()) / scale if scale else 0.0
