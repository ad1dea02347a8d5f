"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no mesh numbering, no assembly,
no decomposition, no coarse space, no Krylov step).  It only draws the inputs
that BASELINE.json's five configs describe:

* the structured cube grid (nx, ny, nz cubes of side h; each cube is cut into
  6 tetrahedra by whoever consumes the workload),
* the present-cube mask (holes are removed cubes),
* the per-tetrahedron coefficients mu^{-1} and eps (tet id = 6*cube + s),
* the subdomain box grid, overlap, gamma, the GenEO threshold,
* the right-hand side f, i.i.d. N(0,1) per free edge (drawn for a length the
  consumer passes in, because the edge count is the consumer's business).

Cube id = ci + nx*(cj + ny*ck) (x fastest).  Every random choice comes from
``numpy.random.default_rng(seed)`` (PCG64), so both sides see bit-identical
inputs.  The recipes are stated in DESIGN.md §3 ("Input recipe").
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
import numpy as np

__all__ = ["Workload", "CONFIGS", "make", "rhs", "config_names"]


@dataclass(frozen=True)
class Workload:
    name: str
    nx: int
    ny: int
    nz: int
    h: float
    px: int                 # subdomain boxes per axis
    py: int
    pz: int
    overlap: int            # cube layers added around each owned box
    gamma: float
    threshold: float        # BASELINE "coarse threshold"; GenEO keeps lambda > 1/threshold
    cube_mask: np.ndarray = field(repr=False)   # uint8[nx*ny*nz], 1 = cube present
    mu_inv: np.ndarray = field(repr=False)      # float64[6*ncubes]
    eps: np.ndarray = field(repr=False)         # float64[6*ncubes]
    dirichlet: str = "outer"  # "outer": E x n = 0 on the box faces, natural on hole walls
    f_seed: int = 0
    holes: tuple = ()         # ((axis, lo_a, lo_b), ...) for documentation / Betti pins

    @property
    def ncubes(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def nsub(self) -> int:
        return self.px * self.py * self.pz


def rhs(n: int, seed: int) -> np.ndarray:
    """f: i.i.d. N(0,1) per free edge (BASELINE configs: "f seeded N(0,1)")."""
    return np.random.default_rng(seed).standard_normal(n)


def _cube_coords(nx, ny, nz):
    c = np.arange(nx * ny * nz)
    return c % nx, (c // nx) % ny, c // (nx * ny)


def _per_tet(per_cube: np.ndarray) -> np.ndarray:
    return np.repeat(np.asarray(per_cube, dtype=np.float64), 6)


def _c0(seed=1):
    n = 8
    nc = n ** 3
    return Workload("c0_cube8", n, n, n, 1.0 / n, 2, 2, 2, 1, 1e-2, 0.1,
                    np.ones(nc, np.uint8), np.ones(6 * nc), np.ones(6 * nc),
                    f_seed=seed)


def _channels(n, nchan, width, contrast, rng):
    """Axis-aligned channels of `width` cells crossing the whole box."""
    ci, cj, ck = _cube_coords(n, n, n)
    coords = (ci, cj, ck)
    val = np.ones(n ** 3)
    chans = []
    for _ in range(nchan):
        axis = int(rng.integers(0, 3))
        a, b = [d for d in range(3) if d != axis]
        la = int(rng.integers(0, n - width + 1))
        lb = int(rng.integers(0, n - width + 1))
        inside = ((coords[a] >= la) & (coords[a] < la + width) &
                  (coords[b] >= lb) & (coords[b] < lb + width))
        val[inside] = contrast
        chans.append((axis, la, lb))
    return val, tuple(chans)


# contrast / gamma / logrange keyword overrides build the well-conditioned
# variants of the recipes used by the literal-tolerance parity tests (same code
# paths, contrast <= 1e2, gamma = 1e-2); the defaults are BASELINE's configs.
def _c1(seed=2, n=32, p=4, contrast=1e4, gamma=1e-4):
    rng = np.random.default_rng(seed)
    mu_inv_cube, chans = _channels(n, n // 4, 2, contrast, rng)
    nc = n ** 3
    return Workload("c1_cube32_channels", n, n, n, 1.0 / n, p, p, p, 1, gamma, 0.1,
                    np.ones(nc, np.uint8), _per_tet(mu_inv_cube), np.ones(6 * nc),
                    f_seed=seed + 1000, holes=())


def _holes(n, nholes, size, rng, max_tries=1000):
    """Non-intersecting square through-holes (size x size cells), each running
    the full length of a random axis, kept >= 1 cell from the lateral faces and
    >= 1 cell apart from each other (so Betti_1 = nholes)."""
    ci, cj, ck = _cube_coords(n, n, n)
    coords = (ci, cj, ck)
    present = np.ones(n ** 3, bool)
    boxes = []
    for _ in range(max_tries):
        if len(boxes) == nholes:
            break
        axis = int(rng.integers(0, 3))
        a, b = [d for d in range(3) if d != axis]
        la = int(rng.integers(1, n - size))      # 1 .. n-size-1 keeps a wall
        lb = int(rng.integers(1, n - size))
        lo = [0, 0, 0]; hi = [n, n, n]
        lo[a], hi[a] = la, la + size
        lo[b], hi[b] = lb, lb + size
        ok = True
        for (plo, phi) in boxes:   # keep >= 1 cell gap from every earlier hole
            if all(lo[d] < phi[d] + 1 and plo[d] < hi[d] + 1 for d in range(3)):
                ok = False
                break
        if ok:
            boxes.append((lo, hi))
    if len(boxes) != nholes:
        raise RuntimeError("could not place holes")
    desc = []
    for lo, hi in boxes:
        inside = np.ones(n ** 3, bool)
        for d in range(3):
            inside &= (coords[d] >= lo[d]) & (coords[d] < hi[d])
        present &= ~inside
        desc.append((tuple(lo), tuple(hi)))
    return present.astype(np.uint8), tuple(desc)


def _c2(seed=3, n=48, p=6, hole=8, gamma=1e-6, logrange=2.0):
    rng = np.random.default_rng(seed)
    mask, holes = _holes(n, 2, hole, rng)
    ci, cj, ck = _cube_coords(n, n, n)
    s = n // p
    sub = (ci // s) + p * ((cj // s) + p * (ck // s))
    mu = 10.0 ** rng.uniform(-logrange, logrange, p ** 3)
    ep = 10.0 ** rng.uniform(-logrange, logrange, p ** 3)
    return Workload("c2_cube48_holes", n, n, n, 1.0 / n, p, p, p, 1, gamma, 0.1,
                    mask, _per_tet(1.0 / mu[sub]), _per_tet(ep[sub]),
                    f_seed=seed + 1000, holes=holes)


def _c3(seed=4, n=96, p=8, contrast=1e3, gamma=1e-3):
    rng = np.random.default_rng(seed)
    ci, cj, ck = _cube_coords(n, n, n)
    layer = (ck * 16) // n
    mu_inv = np.where(layer % 2 == 0, 1.0, contrast)
    nc = n ** 3
    eps = 10.0 ** rng.uniform(np.log10(0.5), np.log10(2.0), 6 * nc)
    return Workload("c3_cube96_layers", n, n, n, 1.0 / n, p, p, p, 2, gamma, 0.1,
                    np.ones(nc, np.uint8), _per_tet(mu_inv), eps, f_seed=seed + 1000)


def _c4(seed=5, ngpu=1, m=64, q=4, contrast=1e4, gamma=1e-2):
    rng = np.random.default_rng(seed)
    nx, ny, nz = m * ngpu, m, m
    nc = nx * ny * nz
    mu_inv = np.where(rng.random(nc) < 0.05, contrast, 1.0)
    return Workload(f"c4_weak{m}_x{ngpu}", nx, ny, nz, 1.0 / m, q * ngpu, q, q, 1, gamma, 0.1,
                    np.ones(nc, np.uint8), _per_tet(mu_inv), np.ones(6 * nc),
                    f_seed=seed + 1000)


CONFIGS = {
    "c0": _c0,
    "c1": _c1,
    "c2": _c2,
    "c3": _c3,
    "c4": _c4,
}


def config_names():
    return list(CONFIGS)


def make(name: str, **kw) -> Workload:
    """Build a config by short name ("c0".."c4").  Keyword overrides are passed
    to the recipe (e.g. ``make("c1", n=8, p=2)`` for a scaled-down c1 recipe)."""
    return CONFIGS[name](**kw)


def custom(nx, ny, nz, px, py, pz, overlap=1, gamma=1e-2, threshold=0.1,
           mask=None, mu_inv=None, eps=None, dirichlet="outer", f_seed=0,
           h=None, name="custom") -> Workload:
    """Small hand-made workloads for pins and edge cases."""
    nc = nx * ny * nz
    if mask is None:
        mask = np.ones(nc, np.uint8)
    if mu_inv is None:
        mu_inv = np.ones(6 * nc)
    if eps is None:
        eps = np.ones(6 * nc)
    if h is None:
        h = 1.0 / max(nx, ny, nz)
    return Workload(name, nx, ny, nz, float(h), px, py, pz, overlap, gamma, threshold,
                    np.asarray(mask, np.uint8), np.asarray(mu_inv, np.float64),
                    np.asarray(eps, np.float64), dirichlet=dirichlet, f_seed=f_seed)


def with_(w: Workload, **kw) -> Workload:
    return replace(w, **kw)
