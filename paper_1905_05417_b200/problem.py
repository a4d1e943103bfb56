"""Host-side problem description: the Python mirror of lamfast::ProblemSetup.

``LaminateProblem`` carries exactly what the reference's ``ProblemSetup`` +
``AssemblyOptions`` carry (assembly.hpp:17-36): three open knot vectors, the
layup (interfaces + per-layer constants/angle), the extruded geometry and the
options.  ``to_c()`` produces the ``lf_problem`` descriptor of
include/lamfast_cuda.h; the same descriptor feeds the CUDA library, the C
oracle and the compiled reference, so all of them see byte-identical inputs.

The BASELINE.json configs C1-C5 and the setups used by the reference tests
are built here.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi

PI = 3.14159265358979323846  # bench.cpp:22

Constants = Tuple[float, float, float, float, float, float, float, float, float]


def orthotropic(E1, E2, E3, G12, G13, G23, nu12, nu13, nu23) -> Constants:
    return (float(E1), float(E2), float(E3), float(G12), float(G13), float(G23),
            float(nu12), float(nu13), float(nu23))


def isotropic(e: float, nu: float) -> Constants:
    """OrthotropicConstants::isotropic (materials.cpp:18-24)."""
    g = e / (2.0 * (1.0 + nu))
    return orthotropic(e, e, e, g, g, g, nu, nu, nu)


def pagano() -> Constants:
    """Reference Pagano constants (bench.cpp:104-112)."""
    return orthotropic(25.0, 1.0, 1.0, 0.2, 0.2, 0.5, 0.25, 0.25, 0.25)


def baseline_orthotropic() -> Constants:
    """BASELINE.json material: E1=25, E2=E3=1, G12=G13=0.5, G23=0.2, nu=0.25."""
    return orthotropic(25.0, 1.0, 1.0, 0.5, 0.5, 0.2, 0.25, 0.25, 0.25)


def uniform_knots(degree: int, n_elements: int) -> np.ndarray:
    """KnotVector::uniform (splines.cpp:27-35)."""
    k = [0.0] * (degree + 1)
    k += [float(i) / n_elements for i in range(1, n_elements)]
    k += [1.0] * (degree + 1)
    return np.asarray(k, dtype=np.float64)


def c0_knots(degree: int, n_elements: int) -> np.ndarray:
    """Clamped knots with every interior knot repeated `degree` times (C0),
    at k/n exactly as Layup::equalLayers places interfaces (materials.cpp:187-189)."""
    k = [0.0] * (degree + 1)
    for i in range(1, n_elements):
        k += [float(i) / n_elements] * degree
    k += [1.0] * (degree + 1)
    return np.asarray(k, dtype=np.float64)


def equal_interfaces(m: int) -> np.ndarray:
    return np.asarray([float(l) / m for l in range(m + 1)], dtype=np.float64)


@dataclass
class LaminateProblem:
    degree_u: int
    degree_v: int
    degree_t: int
    knots_u: np.ndarray
    knots_v: np.ndarray
    knots_t: np.ndarray
    interfaces: np.ndarray
    layers: List[Tuple[Constants, float]]
    geometry_kind: int = abi.LF_GEOM_PLANAR
    geometry: Sequence[float] = (1.0, 1.0)
    direction: Sequence[float] = (0.0, 0.0, 0.1)
    frames: Optional[np.ndarray] = None
    inplane_points: int = 0
    thickness_points: int = 0
    active_layers: Optional[Sequence[int]] = None
    decompose_angles: bool = False
    name: str = ""
    _keep: list = field(default_factory=list, repr=False)

    # -- sizes (splines.hpp:58-83) -------------------------------------------
    @property
    def n_u(self) -> int:
        return len(self.knots_u) - self.degree_u - 1

    @property
    def n_v(self) -> int:
        return len(self.knots_v) - self.degree_v - 1

    @property
    def n_t(self) -> int:
        return len(self.knots_t) - self.degree_t - 1

    @property
    def n_s(self) -> int:
        return self.n_u * self.n_v

    @property
    def dim(self) -> int:
        return 3 * self.n_s * self.n_t

    @property
    def n_layers(self) -> int:
        return len(self.layers)

    def distinct_configs(self) -> int:
        seen = []
        for c, a in self.layers:
            if (c, a) not in seen:
                seen.append((c, a))
        return len(seen)

    def replace(self, **kw) -> "LaminateProblem":
        d = {k: getattr(self, k) for k in self.__dataclass_fields__ if k != "_keep"}
        d.update(kw)
        return LaminateProblem(**d)

    def to_c(self) -> abi.Problem:
        """Builds the lf_problem descriptor; arrays stay alive with self."""
        keep = []

        def dptr(a):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

        p = abi.Problem()
        p.degree_u, p.degree_v, p.degree_t = self.degree_u, self.degree_v, self.degree_t
        p.n_knots_u, p.n_knots_v, p.n_knots_t = (len(self.knots_u), len(self.knots_v),
                                                 len(self.knots_t))
        p.knots_u, p.knots_v, p.knots_t = (dptr(self.knots_u), dptr(self.knots_v),
                                           dptr(self.knots_t))
        p.n_layers = len(self.layers)
        p.interfaces = dptr(self.interfaces)
        layers = (abi.Layer * max(1, len(self.layers)))()
        for k, (c, a) in enumerate(self.layers):
            layers[k].constants = abi.Orthotropic(*c)
            layers[k].angle = float(a)
        keep.append(layers)
        p.layers = ctypes.cast(layers, ctypes.POINTER(abi.Layer))
        p.geometry_kind = int(self.geometry_kind)
        g = list(self.geometry) + [0.0] * (12 - len(self.geometry))
        p.geometry = (ctypes.c_double * 12)(*g)
        p.direction = (ctypes.c_double * 3)(*self.direction)
        if self.frames is not None:
            p.frames = dptr(self.frames)
        p.inplane_points = int(self.inplane_points)
        p.thickness_points = int(self.thickness_points)
        if self.active_layers:
            act = (ctypes.c_int32 * len(self.active_layers))(*self.active_layers)
            keep.append(act)
            p.n_active_layers = len(self.active_layers)
            p.active_layers = ctypes.cast(act, ctypes.POINTER(ctypes.c_int32))
        p.decompose_angles = 1 if self.decompose_angles else 0
        p.threads = 1
        self._keep = keep
        return p


def plate(degree: int, elements_x: int, elements_y: int, angles_or_layers, *,
          lx=1.0, ly=1.0, thickness=0.1, thickness_degree: int = 2,
          thickness_knots: Optional[np.ndarray] = None, material: Optional[Constants] = None,
          name: str = "") -> LaminateProblem:
    """Flat Lx x Ly plate extruded along (0, 0, thickness), equal-thickness
    plies; thickness knots default to one C0 element per ply."""
    layers = []
    for item in angles_or_layers:
        if isinstance(item, tuple):
            layers.append(item)
        else:
            layers.append((material or baseline_orthotropic(), float(item)))
    m = len(layers)
    kt = thickness_knots if thickness_knots is not None else c0_knots(thickness_degree, m)
    return LaminateProblem(
        degree_u=degree, degree_v=degree, degree_t=thickness_degree,
        knots_u=uniform_knots(degree, elements_x), knots_v=uniform_knots(degree, elements_y),
        knots_t=kt, interfaces=equal_interfaces(m), layers=layers,
        geometry_kind=abi.LF_GEOM_PLANAR, geometry=(lx, ly), direction=(0.0, 0.0, thickness),
        name=name)


class MT19937:
    """std::mt19937 (the standardised 32-bit Mersenne Twister)."""

    def __init__(self, seed: int):
        self.mt = [0] * 624
        self.idx = 624
        self.mt[0] = seed & 0xFFFFFFFF
        for i in range(1, 624):
            self.mt[i] = (1812433253 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 30)) + i) & 0xFFFFFFFF

    def __call__(self) -> int:
        if self.idx >= 624:
            for i in range(624):
                y = (self.mt[i] & 0x80000000) | (self.mt[(i + 1) % 624] & 0x7FFFFFFF)
                v = self.mt[(i + 397) % 624] ^ (y >> 1)
                if y & 1:
                    v ^= 0x9908B0DF
                self.mt[i] = v
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= y >> 11
        y ^= (y << 7) & 0x9D2C5680
        y ^= (y << 15) & 0xEFC60000
        y ^= y >> 18
        return y & 0xFFFFFFFF


DEG0, DEG90, DEG45, DEGM45 = 0.0, 0.5 * PI, 0.25 * PI, -0.25 * PI


def baseline_config(name: str, *, plies: Optional[int] = None) -> LaminateProblem:
    """BASELINE.json configs C1..C5.  `plies` overrides the
    ply count (same family) for bounded CPU samples."""
    name = name.upper()
    if name == "C1":
        angles = [DEG0, DEG90, DEG90, DEG0]
        return plate(2, 8, 8, angles, thickness=0.1, name="C1")
    if name == "C2":
        half = [DEG0, DEG90] * 4
        angles = half + half[::-1]
        return plate(2, 32, 32, angles, thickness=0.1, name="C2")
    if name == "C3":
        m = plies or 64
        cyc = [DEG0, DEG45, DEGM45, DEG90]
        return plate(3, 64, 64, [cyc[l % 4] for l in range(m)], thickness=0.2, name="C3")
    if name == "C4":
        m = plies or 128
        soft = isotropic(0.5, 0.3)
        layers = []
        for k in range(m):
            if k % 2 == 1:
                layers.append((soft, 0.0))
            else:
                layers.append((baseline_orthotropic(), DEG0 if k % 4 == 0 else DEG90))
        return plate(2, 128, 64, layers, lx=2.0, ly=1.0, thickness=0.2, name="C4")
    if name == "C5":
        m = plies or 128
        rng = MT19937(20190514)
        cyc = [DEG0, DEG45, DEGM45, DEG90]
        angles = [cyc[rng() >> 30] for _ in range(m)]
        return plate(3, 192, 192, angles, thickness=0.25, name="C5")
    raise ValueError(f"unknown config {name}")


def cube_problem(degree: int, elems_inplane: int, elems_thickness: int, angles, *,
                 geometry: str = "flat", lx=1.0, ly=1.0, thickness=0.1,
                 material: Optional[Constants] = None) -> LaminateProblem:
    """cubeSpace + flat/skewed geometry + Pagano layup as in the reference
    tests (test_fast.cpp:23-57): uniform maximal-continuity knots everywhere."""
    layers = [(material or pagano(), float(a)) if not isinstance(a, tuple) else a
              for a in angles]
    m = len(layers)
    prob = LaminateProblem(
        degree_u=degree, degree_v=degree, degree_t=degree,
        knots_u=uniform_knots(degree, elems_inplane), knots_v=uniform_knots(degree, elems_inplane),
        knots_t=uniform_knots(degree, elems_thickness), interfaces=equal_interfaces(m),
        layers=layers, geometry_kind=abi.LF_GEOM_PLANAR, geometry=(lx, ly),
        direction=(0.0, 0.0, thickness))
    if geometry == "skewed":
        prob.geometry_kind = abi.LF_GEOM_BILINEAR
        prob.geometry = (0, 0, 0, 1.2, 0.1, 0.05, -0.1, 0.9, -0.02, 1.0, 1.1, 0.08)
        prob.direction = (0.03, -0.02, 0.2)
    return prob


def sizes(prob: LaminateProblem) -> dict:
    """Closed-form sizes of the fast-path CSR."""
    def adj_len(knots, p):
        n = len(knots) - p - 1
        firsts = [k - p for k in range(p, n) if knots[k + 1] > knots[k]]
        L = []
        for i in range(n):
            los = [f for f in firsts if f <= i <= f + p]
            L.append(max(los) + p - min(los) + 1 if los else 0)
        return np.asarray(L, dtype=np.int64)

    Lu = adj_len(prob.knots_u, prob.degree_u)
    Lv = adj_len(prob.knots_v, prob.degree_v)
    Lt = adj_len(prob.knots_t, prob.degree_t)
    S = int(Lu.sum() * Lv.sum())
    return {"n_s": prob.n_s, "n_t": prob.n_t, "dim": prob.dim, "S_s": S,
            "S_t": int(Lt.sum()), "nnz": 9 * S * int(Lt.sum())}
