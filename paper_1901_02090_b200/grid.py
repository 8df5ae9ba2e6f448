"""Grid, permeability, wells and the saddle system (host-side descriptors).

Mirrors the reference's public types (`/root/reference/pkg/src/bddcflow/
grid.py:21-357`): dof numbering is identical (interior faces only, x-faces
then y-faces then z-faces, each family x-fastest).  Mode B (`PressureDrop`,
BASELINE's boundary condition, not expressible in the reference) appends the
Dirichlet boundary faces of one axis after the interior ones: low-end faces,
then high-end faces, each in x-fastest order over the transverse axes.  No matrices are
assembled on the solve path: the device kernels apply the RT0 operators
matrix-free (csrc/stencil.cu, csrc/local.cu).  `SaddleSystem.A/.B` exist
only for API compatibility (users and tests may multiply with them) and are
built lazily on the host when first touched.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property

import numpy as np

from .errors import CompatibilityError, InvalidArgumentError


@dataclass(frozen=True)
class Grid:
    """Tensor-product grid (grid.py:21-160)."""

    dim: int
    counts: tuple
    sizes: tuple

    @property
    def n_cells(self):
        return int(np.prod(self.counts))

    @property
    def cell_volume(self):
        return float(np.prod(self.sizes))

    @cached_property
    def flux_offsets(self):
        """Offsets of the interior-face families in the flux dof numbering."""
        offs = [0]
        for a in range(self.dim):
            e = list(self.counts)
            e[a] -= 1
            offs.append(offs[-1] + int(np.prod(e)))
        return tuple(offs)

    @property
    def n_flux_dofs(self):
        return self.flux_offsets[-1]

    @property
    def total_dofs(self):
        """All face dofs (including boundary) plus cell pressures (grid.py:51-54)."""
        n = 0
        for a in range(self.dim):
            e = list(self.counts)
            e[a] += 1
            n += int(np.prod(e))
        return n + self.n_cells

    @cached_property
    def cell_coords(self):
        idx = np.arange(self.n_cells)
        out = np.empty((self.n_cells, self.dim), dtype=np.int64)
        for a in range(self.dim):
            out[:, a] = idx % self.counts[a]
            idx = idx // self.counts[a]
        return out

    def interior_face_dof(self, a, coords):
        """Dof of the a-face at face coordinate `coords` (f_a in 1..n_a-1), -1 otherwise."""
        coords = np.asarray(coords)
        ca = coords[:, a]
        ok = (ca >= 1) & (ca <= self.counts[a] - 1)
        idx = np.zeros(len(coords), dtype=np.int64)
        stride = 1
        for d in range(self.dim):
            ext = self.counts[d] - (1 if d == a else 0)
            idx += (coords[:, d] - (1 if d == a else 0)) * stride
            stride *= ext
        return np.where(ok, self.flux_offsets[a] + idx, -1)

    def cell_faces(self, a, dirichlet_axis=None):
        """(low, high) dofs of every cell's a-faces, -1 on a no-flow boundary.
        With `dirichlet_axis == a` the boundary faces of that axis are dofs too
        (numbered after the interior faces, see `boundary_face_dofs`)."""
        lo = self.interior_face_dof(a, self.cell_coords)
        hi_c = self.cell_coords.copy()
        hi_c[:, a] += 1
        hi = self.interior_face_dof(a, hi_c)
        if dirichlet_axis == a:
            blo, bhi = self.boundary_face_dofs(a)
            ca = self.cell_coords[:, a]
            lo[ca == 0] = blo
            hi[ca == self.counts[a] - 1] = bhi
        return lo, hi

    def n_boundary_faces(self, a):
        """Faces on one end of axis a."""
        return self.n_cells // self.counts[a]

    def boundary_face_dofs(self, a):
        """Dofs of the low-end and high-end a-faces (mode B numbering: after the
        interior faces, low end then high end, x-fastest over the other axes)."""
        nt = self.n_boundary_faces(a)
        base = self.n_flux_dofs
        return base + np.arange(nt), base + nt + np.arange(nt)


def build_grid(dim, counts, sizes):
    """Validate and construct a Grid (grid.py:163-175)."""
    counts = tuple(int(c) for c in counts)
    sizes = tuple(float(s) for s in sizes)
    if dim not in (2, 3):
        raise InvalidArgumentError(f"dim must be 2 or 3, got {dim}")
    if len(counts) != dim or len(sizes) != dim:
        raise InvalidArgumentError("counts/sizes length must equal dim")
    if any(c < 1 for c in counts):
        raise InvalidArgumentError(f"cell counts must be >= 1, got {counts}")
    if any(not np.isfinite(s) or s <= 0 for s in sizes):
        raise InvalidArgumentError(f"cell sizes must be > 0, got {sizes}")
    return Grid(dim, counts, sizes)


@dataclass(frozen=True)
class Permeability:
    """Per-cell permeability, one value per axis (grid.py:178-194)."""

    k: np.ndarray

    def __post_init__(self):
        k = np.asarray(self.k, dtype=np.float64)
        if not np.all(np.isfinite(k)) or np.any(k <= 0):
            raise InvalidArgumentError("permeability must be positive finite")
        object.__setattr__(self, "k", k)

    @classmethod
    def isotropic(cls, grid, values):
        values = np.broadcast_to(np.asarray(values, dtype=np.float64),
                                 (grid.n_cells,))
        return cls(np.repeat(values[:, None], grid.dim, axis=1))


@dataclass(frozen=True)
class Wells:
    src_cell: int
    sink_cell: int
    strength: float = 1.0


@dataclass(frozen=True)
class PressureDrop:
    """Mode B boundary condition (BASELINE's): pressure `p_low` on the low end and
    `p_high` on the high end of `axis`, no flow elsewhere.  The reference has no
    Dirichlet pressure (its assemble_system, grid.py:327-341, only takes wells);
    the boundary faces of `axis` become flux dofs with the momentum right-hand
    side g = +p_low (low end) and -p_high (high end) in A u + B^T p = g."""

    axis: int
    p_low: float = 1.0
    p_high: float = 0.0


class SaddleSystem:
    """Mixed system [[A, B^T],[B, 0]](u, p) = (g, f) (grid.py:230-267).

    Holds the host inputs (permeability, source vector f, and in mode B the
    pressure drop that defines g).  `D` is the per-cell pressure rescaling
    filled in by the setup (grid.py:344-357).
    """

    def __init__(self, grid, perm, f, wells=None, D=None, lumped=False, dirichlet=None):
        self.grid = grid
        self.perm = perm
        self.f = np.asarray(f, dtype=np.float64)
        self.wells = wells
        self.D = D
        self.lumped = lumped
        self.dirichlet = dirichlet

    @property
    def dirichlet_axis(self):
        return None if self.dirichlet is None else self.dirichlet.axis

    @property
    def n_flux(self):
        n = self.grid.n_flux_dofs
        if self.dirichlet is not None:
            n += 2 * self.grid.n_boundary_faces(self.dirichlet.axis)
        return n

    @property
    def g(self):
        """Momentum right-hand side (zero in mode A)."""
        g = np.zeros(self.n_flux)
        if self.dirichlet is not None:
            blo, bhi = self.grid.boundary_face_dofs(self.dirichlet.axis)
            g[blo] = self.dirichlet.p_low
            g[bhi] = -self.dirichlet.p_high
        return g

    @property
    def n_pressure(self):
        return self.grid.n_cells

    @property
    def fs(self):
        return self.f if self.D is None else self.D * self.f

    def unscale_pressure(self, p_bar):
        return p_bar if self.D is None else self.D * p_bar

    def with_rescaling(self, D):
        return SaddleSystem(self.grid, self.perm, self.f, self.wells, D=D,
                            lumped=self.lumped, dirichlet=self.dirichlet)

    # -- host matrices for API compatibility only (not used by solve) ------

    @cached_property
    def A(self):
        import scipy.sparse as sp
        g, k = self.grid, self.perm.k
        rows, cols, vals = [], [], []
        for a in range(g.dim):
            lo, hi = g.cell_faces(a, self.dirichlet_axis)
            c = g.sizes[a] ** 2 / (6.0 * g.cell_volume) / k[:, a]
            for d, o in ((lo, hi), (hi, lo)):
                m = d >= 0
                rows += [d[m]]
                cols += [d[m]]
                vals += [(3.0 if self.lumped else 2.0) * c[m]]   # grid.py:220-225
                if self.lumped:
                    continue
                mo = m & (o >= 0)
                rows += [d[mo]]
                cols += [o[mo]]
                vals += [c[mo]]
        n = self.n_flux
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows),
                                                     np.concatenate(cols))),
                             shape=(n, n)).tocsr()

    @cached_property
    def B(self):
        import scipy.sparse as sp
        g = self.grid
        rows, cols, vals = [], [], []
        cells = np.arange(g.n_cells)
        for a in range(g.dim):
            lo, hi = g.cell_faces(a, self.dirichlet_axis)
            for d, s in ((lo, 1.0), (hi, -1.0)):
                m = d >= 0
                rows += [cells[m]]
                cols += [d[m]]
                vals += [np.full(int(m.sum()), s)]
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows),
                                                     np.concatenate(cols))),
                             shape=(g.n_cells, self.n_flux)).tocsr()


def assemble_system(grid, perm, wells, lumped=False):
    """Validate inputs and form the source vector (grid.py:327-341).

    `wells` is a `Wells` (mode A, the reference's only boundary condition:
    no flow everywhere, sources at two cells) or a `PressureDrop` (mode B:
    Dirichlet pressure on both ends of one axis, zero source)."""
    if perm.k.shape != (grid.n_cells, grid.dim):
        raise InvalidArgumentError("permeability shape mismatch")
    if isinstance(wells, PressureDrop):
        if not 0 <= wells.axis < grid.dim:
            raise InvalidArgumentError(f"pressure-drop axis {wells.axis} outside 0..{grid.dim - 1}")
        if not (np.isfinite(wells.p_low) and np.isfinite(wells.p_high)):
            raise InvalidArgumentError("boundary pressures must be finite")
        return SaddleSystem(grid, perm, np.zeros(grid.n_cells), None, lumped=lumped, dirichlet=wells)
    for c in (wells.src_cell, wells.sink_cell):
        if not 0 <= c < grid.n_cells:
            raise InvalidArgumentError(f"well cell {c} outside grid")
    f = np.zeros(grid.n_cells)
    f[wells.src_cell] -= wells.strength
    f[wells.sink_cell] += wells.strength
    if abs(f.sum()) > 1e-12 * max(np.abs(f).sum(), 1.0):
        raise CompatibilityError("source terms must sum to zero")
    return SaddleSystem(grid, perm, f, wells, lumped=lumped)
