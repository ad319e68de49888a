"""Synthetic 3D lid-driven-cavity pressure matrices (the bench/test input generator).

Same numbering, slab decomposition and coefficients as the reference's
model-problem generator (assembly.py:17-243) — parity of every downstream
integer array depends on it — but built in closed form: a cell's upper
neighbours are c+1, c+d0, c+plane in that order, so walking cells in order
emits faces already sorted by (lower, upper) and no lexsort is needed at
27M cells.  Assembly stays on the host by the paper's premise; it is input
generation, not part of the accelerated path.
"""

from dataclasses import dataclass

import numpy as np

from .core import InterfaceBlock, LduMatrix


@dataclass(frozen=True)
class StructuredGrid:
    nx: int
    ny: int
    nz: int

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("grid extents must be >= 1")

    @property
    def dims(self):
        return (self.nx, self.ny, self.nz)

    @property
    def total_cells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def dimension(self) -> int:
        return sum(d > 1 for d in self.dims)

    @property
    def slab_axis(self) -> int:
        """Longest axis, ties toward z (assembly.py:48-55)."""
        d = self.dims
        return max(range(3), key=lambda ax: (d[ax], ax))

    @property
    def axis_order(self):
        slow = self.slab_axis
        fast = [ax for ax in range(3) if ax != slow]
        return (fast[0], fast[1], slow)

    @property
    def n_internal_faces(self) -> int:
        nx, ny, nz = self.dims
        return (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)


def build_grid(n_p: int) -> StructuredGrid:
    """(210 n_p)^3 benchmark cube (assembly.py:70-75)."""
    if n_p < 1:
        raise ValueError(f"n_p must be >= 1, got {n_p}")
    e = 210 * n_p
    return StructuredGrid(e, e, e)


@dataclass(frozen=True)
class MeshInterface:
    neighbor_rank: int
    cells: np.ndarray
    neighbor_cells: np.ndarray


@dataclass(frozen=True)
class SubdomainMesh:
    cpu_rank: int
    n_cells: int
    global_offset: int
    internal_faces: np.ndarray
    boundary_face_count: np.ndarray
    interfaces: tuple

    @property
    def global_cell_ids(self):
        return np.arange(self.global_offset, self.global_offset + self.n_cells, dtype=np.int64)


def slab_layers(n_layers: int, n_parts: int):
    """Balanced layer ranges, the first n_layers % n_parts get one more (assembly.py:108-117)."""
    q, rem = divmod(n_layers, n_parts)
    bounds = np.cumsum([0] + [q + (r < rem) for r in range(n_parts)])
    return [(int(bounds[r]), int(bounds[r + 1])) for r in range(n_parts)]


def _faces(d0, d1, nz):
    """Internal faces of a d0 x d1 x nz slab, sorted by (lower, upper)."""
    plane = d0 * d1
    n = plane * nz
    c = np.arange(n, dtype=np.int64)
    nb = np.empty((n, 3), dtype=np.int64)
    ok = np.empty((n, 3), dtype=bool)
    nb[:, 0] = c + 1
    nb[:, 1] = c + d0
    nb[:, 2] = c + plane
    ok[:, 0] = (c % d0) < d0 - 1
    ok[:, 1] = ((c // d0) % d1) < d1 - 1 if d1 > 1 else False
    ok[:, 2] = (c // plane) < nz - 1
    if d0 == 1:
        ok[:, 0] = False
    sel = ok.ravel()
    upper = nb.ravel()[sel]
    lower = np.repeat(c, ok.sum(axis=1))
    return lower, upper


def decompose_slab(grid: StructuredGrid, n_parts: int):
    """Contiguous slabs along the slowest axis (assembly.py:120-192)."""
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    a0, a1, a2 = grid.axis_order
    d0, d1, d2 = (grid.dims[a] for a in (a0, a1, a2))
    if n_parts > d2:
        raise ValueError(f"too many parts: {n_parts} slabs requested along an axis of {d2} cells")
    layers = slab_layers(d2, n_parts)
    plane = d0 * d1
    fp = np.arange(plane, dtype=np.int64)
    out = []
    for r, (z0, z1) in enumerate(layers):
        nz = z1 - z0
        n = plane * nz
        lower, upper = _faces(d0, d1, nz)
        c = np.arange(n, dtype=np.int64)
        bnd = np.zeros(n, dtype=np.int64)
        if d0 > 1:
            ix = c % d0
            bnd += (ix == 0)
            bnd += (ix == d0 - 1)
        if d1 > 1:
            iy = (c // d0) % d1
            bnd += (iy == 0)
            bnd += (iy == d1 - 1)
        if d2 > 1:
            gz = c // plane + z0
            bnd += (gz == 0)
            bnd += (gz == d2 - 1)
        ifaces = []
        if z0 > 0:
            prev = layers[r - 1][1] - layers[r - 1][0]
            ifaces.append(MeshInterface(r - 1, fp.copy(), fp + plane * (prev - 1)))
        if z1 < d2:
            ifaces.append(MeshInterface(r + 1, fp + plane * (nz - 1), fp.copy()))
        out.append(SubdomainMesh(r, n, plane * z0, np.column_stack((lower, upper)), bnd,
                                 tuple(ifaces)))
    return out


def assemble_poisson(part: SubdomainMesh):
    """Unit 7-point Laplacian: diag = faces of the cell, couplings -1 (assembly.py:195-222)."""
    n = part.n_cells
    lower = np.ascontiguousarray(part.internal_faces[:, 0])
    upper = np.ascontiguousarray(part.internal_faces[:, 1])
    diag = part.boundary_face_count.astype(np.int64) + np.bincount(lower, minlength=n) \
        + np.bincount(upper, minlength=n)
    blocks = []
    for itf in part.interfaces:
        diag = diag + np.bincount(itf.cells, minlength=n)
        blocks.append(InterfaceBlock(itf.neighbor_rank, itf.cells, itf.neighbor_cells,
                                     np.full(len(itf.cells), -1.0)))
    nf = len(lower)
    m = LduMatrix(n, lower, upper, diag.astype(np.float64), np.full(nf, -1.0), np.full(nf, -1.0))
    return m, blocks


def perturb_coefficients(m: LduMatrix, ifaces, step: int):
    """Pseudo-timestep change: diag * (1 + step/100) from the pristine base (assembly.py:225-243)."""
    if step < 1:
        raise ValueError(f"step must be >= 1, got {step}")
    return LduMatrix(m.n_cells, m.lower_addr, m.upper_addr, m.diag * (1.0 + step / 100.0),
                     m.lower_val, m.upper_val), ifaces


def perturb_diag_into(base_diag: np.ndarray, step: int, out: np.ndarray) -> np.ndarray:
    """Producer variant writing the step's diagonal into a preallocated (pinned)
    array; bit-identical to perturb_coefficients."""
    if step < 1:
        raise ValueError(f"step must be >= 1, got {step}")
    return np.multiply(base_diag, 1.0 + step / 100.0, out=out)
