"""Create-once repartitioning of per-rank LDU matrices onto GPU parts.

Drop-in for the reference's repart.py (same names, arguments, errors).  The
owner-side fusion — localization, row-major ordering, LDU->row-major scatter
map, halo columns — is one O(nnz) native build (lrb_plan_build_ldu, C++), and
its result is uploaded once into a SELL-32 device part; only values move
afterwards (update.py).  Integer outputs are bit-identical to the reference's
lexsort/searchsorted pipeline (tests/test_plan_golden.py).
"""

from dataclasses import dataclass, field

import numpy as np

from .core import DeviceCooMatrix, DistributedCooMatrix, InterfaceBlock, LduMatrix, \
    PartitionMap, gpu_owner
from .device import DevicePart, Plan, Team, device_count
from .solver import HaloPlan, build_halo_plan
from .transport import CAT_DEVICE_DIRECT, CAT_RANK, CommGroup, DeviceBuffer, RankContext, split_active


@dataclass(frozen=True)
class SparsityPattern:
    """Global-index pattern of one source rank (repart.py:26-39)."""

    local_rows: np.ndarray
    local_cols: np.ndarray
    nonlocal_rows: np.ndarray
    nonlocal_cols: np.ndarray
    row_lo: int
    row_hi: int

    @property
    def n_entries(self) -> int:
        return len(self.local_rows) + len(self.nonlocal_rows)


@dataclass(frozen=True)
class UpdatePattern:
    """Who sends how many coefficients to which owner offset (repart.py:42-79)."""

    send_target: np.ndarray
    send_length: np.ndarray
    recv_offsets: tuple

    def __post_init__(self):
        for k, offs in enumerate(self.recv_offsets):
            if offs[0] != 0 or (np.diff(offs) <= 0).any():
                raise ValueError(f"update pattern: owner {k} segments must be "
                                 "contiguous, disjoint and non-empty")

    @property
    def n_cpu(self) -> int:
        return len(self.send_target)

    @property
    def alpha(self) -> int:
        return len(self.send_target) // len(self.recv_offsets)

    def total(self, k: int) -> int:
        return int(self.recv_offsets[k][-1])

    def segments(self, k: int):
        a = self.alpha
        o = self.recv_offsets[k]
        return [(a * k + i, int(o[i]), int(o[i + 1] - o[i])) for i in range(a)]


class ScatterMap:
    """Bijection buffer position -> (local | non-local, slot) (repart.py:82-106).

    Built from explicit arrays (validated like the reference), or backed by a
    native plan, in which case the arrays are exported on first access.
    """

    def __init__(self, to_local=None, index=None, n_local=0, n_nonlocal=0, plan=None):
        self._plan = plan
        if plan is not None:
            self.n_local, self.n_nonlocal = plan.nnz_local, plan.nnz_nonlocal
            self._to_local = self._index = None
            return
        self.n_local, self.n_nonlocal = int(n_local), int(n_nonlocal)
        self._to_local = np.asarray(to_local, dtype=bool)
        self._index = np.asarray(index, dtype=np.int64)
        if len(self._to_local) != len(self._index):
            raise ValueError("scatter map arrays must have equal length")
        if len(self._index) != self.n_local + self.n_nonlocal:
            raise ValueError("scatter map must cover every destination slot")
        hl = np.bincount(self._index[self._to_local], minlength=self.n_local)
        hn = np.bincount(self._index[~self._to_local], minlength=self.n_nonlocal)
        if len(hl) != self.n_local or (hl != 1).any():
            raise ValueError("scatter map is not a bijection onto local slots")
        if len(hn) != self.n_nonlocal or (hn != 1).any():
            raise ValueError("scatter map is not a bijection onto non-local slots")

    def _materialize(self):
        if self._to_local is None:
            self._to_local, self._index = self._plan.scatter()

    @property
    def to_local(self) -> np.ndarray:
        self._materialize()
        return self._to_local

    @property
    def index(self) -> np.ndarray:
        self._materialize()
        return self._index

    def __len__(self) -> int:
        return self.n_local + self.n_nonlocal


@dataclass
class RepartitionedSystem:
    """Create-once state of one rank (repart.py:109-134)."""

    ctx: RankContext
    pm: PartitionMap
    comm: CommGroup
    update_pattern: UpdatePattern
    fingerprint: tuple
    matrix: object = None
    scatter: ScatterMap = None
    device: DeviceBuffer = None
    halo: HaloPlan = None
    # every rank of an owner group holds the owner's device part (to copy its
    # own segment straight into it); only the owner allocated it
    part: DevicePart = field(default=None, repr=False)
    team: Team = field(default=None, repr=False)

    @property
    def is_owner(self) -> bool:
        return self.matrix is not None

    @property
    def gpu_rank(self):
        return self.ctx.rank // self.pm.alpha if self.is_owner else None

    @property
    def segment(self) -> int:
        return self.ctx.rank % self.pm.alpha


def sparsity_fingerprint(m: LduMatrix, ifaces) -> tuple:
    return (m.n_cells, m.n_faces,
            tuple((b.neighbor_rank, len(b)) for b in sorted(ifaces, key=lambda b: b.neighbor_rank)))


# ---------------------------------------------------------------------------
# source-side description of the packed buffer
# ---------------------------------------------------------------------------
class _Source:
    """One rank's LDU addressing and interface provenance in pack order."""

    __slots__ = ("rank", "lo", "hi", "n", "lower", "upper", "ifc_row", "ifc_col", "n_entries")

    def __init__(self, m: LduMatrix, ifaces, pm: PartitionMap, rank: int):
        lo, hi = pm.cpu_range(rank)
        if hi - lo != m.n_cells:
            raise ValueError(f"rank {rank} holds {m.n_cells} cells but owns "
                             f"{hi - lo} in the partition map")
        rows, cols = [], []
        for b in sorted(ifaces, key=lambda b: b.neighbor_rank):
            if b.neighbor_rank == rank:
                raise ValueError(f"inconsistent interface: rank {rank} lists itself as neighbor")
            nlo, nhi = pm.cpu_range(b.neighbor_rank)
            if len(b) and (int(b.cols_remote.max()) >= nhi - nlo or int(b.rows.max()) >= m.n_cells):
                raise ValueError(f"inconsistent interface: entry of rank {rank} toward "
                                 f"rank {b.neighbor_rank} is out of range")
            rows.append(b.rows)
            cols.append(b.cols_remote + nlo)
        if rows:
            ir, ic = np.concatenate(rows), np.concatenate(cols)
            # provenance order of the packed interface values: (column owner, row,
            # column) (repart.py:262-264); the concatenation is already in that
            # order unless a neighbour is listed twice
            own = pm.col_owner_cpu(ic)
            key_sorted = (np.diff(own) > 0) | ((np.diff(own) == 0) & (
                (np.diff(ir) > 0) | ((np.diff(ir) == 0) & (np.diff(ic) > 0))))
            if not key_sorted.all():
                o = np.lexsort((ic, ir, own))
                ir, ic = ir[o], ic[o]
                own = own[o]
            dup = (np.diff(ir) == 0) & (np.diff(ic) == 0)
            if dup.any():
                raise ValueError("inconsistent interface: duplicate coupling entry")
        else:
            ir = ic = np.zeros(0, np.int64)
        self.rank, self.lo, self.hi, self.n = rank, lo, hi, m.n_cells
        self.lower, self.upper = m.lower_addr, m.upper_addr
        self.ifc_row, self.ifc_col = ir, ic
        self.n_entries = m.n_cells + 2 * m.n_faces + len(ir)


def _pieces(m: LduMatrix, ifaces):
    """Coefficient pieces in pack order [diag | upper | lower | ifaces] (update.py:40-45)."""
    return [m.diag, m.upper_val, m.lower_val] + \
        [b.values for b in sorted(ifaces, key=lambda b: b.neighbor_rank)]


def _owner_plan(sources, pm: PartitionMap, k: int) -> Plan:
    lo, hi = pm.gpu_range(k)
    src_rows = np.array([s.lo for s in sources] + [sources[-1].hi], dtype=np.int64)
    face_off = np.concatenate(([0], np.cumsum([len(s.lower) for s in sources]))).astype(np.int64)
    ifc_off = np.concatenate(([0], np.cumsum([len(s.ifc_row) for s in sources]))).astype(np.int64)
    cat = (lambda xs: np.concatenate(xs) if len(xs) > 1 else np.asarray(xs[0]))
    return Plan.from_ldu(pm.total_cells, lo, hi, src_rows, face_off,
                         cat([s.lower for s in sources]), cat([s.upper for s in sources]),
                         ifc_off, cat([s.ifc_row for s in sources]),
                         cat([s.ifc_col for s in sources]), pm.gpu_offsets)


def _matrix_from_plan(plan: Plan, part: DevicePart, pm: PartitionMap, k: int):
    lo, hi = pm.gpu_range(k)
    loc_ptr, loc_col, nl_ptr, nl_col, halo = plan.csr()
    n = hi - lo
    local = DeviceCooMatrix(n, n, loc_ptr, loc_col, part, "local")
    non_local = DeviceCooMatrix(n, len(halo), nl_ptr, nl_col, part, "non_local")
    return DistributedCooMatrix(owner_gpu_rank=k, row_offset=lo, local=local,
                                non_local=non_local, halo_cols=halo)


def _group_barrier(ctx: RankContext, pm: PartitionMap, tag: str):
    """Barrier among the alpha ranks fused onto one owner."""
    k = ctx.rank // pm.alpha
    ctx.world._barrier(ctx.rank, ("owner-group", tag, k, pm.n_cpu, pm.alpha), pm.alpha)


def repartition(m: LduMatrix, ifaces, pm: PartitionMap, ctx: RankContext) -> RepartitionedSystem:
    """Create the repartitioned system (repart.py:321-354); collective over the world.

    Owners come back with the fused matrix on their GPU (initial values
    scattered), the scatter map, the device buffer and the halo plan;
    inactive ranks keep the update pattern, fingerprint and a handle to their
    owner's part (no device allocation of their own).
    """
    src = _Source(m, ifaces, pm, ctx.rank)
    counts = ctx.allgather(src.n_entries)
    up = build_update_pattern(pm, counts)
    k = gpu_owner(ctx.rank, pm)
    owner = pm.alpha * k
    ctx.send(owner, src)
    # bytes of the reference's pattern message (4 int64 arrays + row_lo/hi,
    # repart.py:185-187); _Source itself travels by reference
    n_loc = m.n_cells + 2 * m.n_faces
    ctx.world._account(CAT_RANK, 16 * n_loc + 16 * (src.n_entries - n_loc) + 16, messages=0)
    comm = split_active(ctx, pm)
    system = RepartitionedSystem(ctx=ctx, pm=pm, comm=comm, update_pattern=up,
                                 fingerprint=sparsity_fingerprint(m, ifaces))
    if ctx.rank == owner:
        sources = [ctx.recv(r) for r in range(owner, owner + pm.alpha)]
        plan = _owner_plan(sources, pm, k)
        part = DevicePart(plan, k % device_count())
        ctx.world._count_allocation(ctx.rank)
        system.part = part
        system.matrix = _matrix_from_plan(plan, part, pm, k)
        system.scatter = ScatterMap(plan=plan)
        system.device = DeviceBuffer(ctx.world, ctx.rank, plan.n_buf, part=part)
        for r in range(owner + 1, owner + pm.alpha):
            ctx.send(r, part)
    else:
        system.part = ctx.recv(owner)
    # initial fill is always direct (repart.py:349-350)
    pieces = _pieces(m, ifaces)
    system.part.update_segment(system.segment, pieces)
    ctx.world._account(CAT_DEVICE_DIRECT, 8 + 8 * src.n_entries)
    _group_barrier(ctx, pm, "create")
    if system.is_owner:
        system.device.transfer_count += pm.alpha
        system.device.transfer_bytes += 8 * up.total(k)
        system.part.join()
        system.halo = build_halo_plan(system.matrix, pm, comm)
        parts = comm.allgather(system.part)
        team = Team(parts) if comm.group_rank == 0 else None
        system.team = comm.bcast(team, 0)
        system.matrix._team = system.team
        system.matrix._part = system.part
        system.matrix._gpu_rank = k
    return system


# ---------------------------------------------------------------------------
# low-level API of the reference (repart.py:143-304), same contracts
# ---------------------------------------------------------------------------
def extract_sparsity(m: LduMatrix, ifaces, pm: PartitionMap, my_rank: int) -> SparsityPattern:
    """Global-index local pattern + interface pattern (repart.py:143-174)."""
    src = _Source(m, ifaces, pm, my_rank)
    lo, hi = src.lo, src.hi
    plan = Plan.from_ldu(pm.total_cells, lo, hi, np.array([lo, hi]), np.array([0, len(src.lower)]),
                         src.lower, src.upper, np.array([0, 0]), np.zeros(0, np.int64),
                         np.zeros(0, np.int64), np.array([0, pm.total_cells]))
    loc_ptr, loc_col, _, _, _ = plan.csr()
    rows = np.repeat(np.arange(lo, hi, dtype=np.int64), np.diff(loc_ptr))
    nr = src.ifc_row + lo
    nc = src.ifc_col
    o = np.lexsort((nc, nr))
    return SparsityPattern(local_rows=rows, local_cols=loc_col + lo,
                           nonlocal_rows=nr[o], nonlocal_cols=nc[o], row_lo=lo, row_hi=hi)


def exchange_patterns(sp: SparsityPattern, pm: PartitionMap, ctx: RankContext):
    """Ship patterns to owner alpha*floor(r/alpha); owners get them ascending (repart.py:177-194)."""
    owner = pm.alpha * gpu_owner(ctx.rank, pm)
    ctx.send(owner, sp)
    if ctx.rank != owner:
        return []
    return [ctx.recv(r) for r in range(owner, owner + pm.alpha)]


def _check_tiling(received, pm: PartitionMap, gpu_rank: int):
    lo, hi = pm.gpu_range(gpu_rank)
    if len(received) != pm.alpha:
        raise ValueError(f"owner {gpu_rank} expected {pm.alpha} patterns, got {len(received)}")
    prev = lo
    for sp in received:
        if sp.row_lo != prev or sp.row_hi > hi:
            raise ValueError("received patterns must tile I_GPU in ascending source order")
        prev = sp.row_hi
    if prev != hi:
        raise ValueError("received patterns must tile I_GPU in ascending source order")
    return lo, hi


def _patterns_of(plan: Plan, lo: int):
    loc_ptr, loc_col, nl_ptr, nl_col, halo = plan.csr()
    rows = np.arange(lo, lo + plan.n, dtype=np.int64)
    local = (np.repeat(rows, np.diff(loc_ptr)), loc_col + lo)
    nonlocal_ = (np.repeat(rows, np.diff(nl_ptr)), halo[nl_col])
    return local, nonlocal_


def fuse_patterns(received, pm: PartitionMap, gpu_rank: int):
    """Fused row-major local / non-local global patterns (repart.py:197-236)."""
    lo, hi = _check_tiling(received, pm, gpu_rank)
    rows = np.concatenate([sp.local_rows for sp in received] + [sp.nonlocal_rows for sp in received])
    cols = np.concatenate([sp.local_cols for sp in received] + [sp.nonlocal_cols for sp in received])
    plan = Plan.from_coo(pm.total_cells, lo, hi, rows, cols)
    return _patterns_of(plan, lo)


def build_update_pattern(pm: PartitionMap, counts) -> UpdatePattern:
    counts = np.asarray(counts, dtype=np.int64)
    if len(counts) != pm.n_cpu:
        raise ValueError(f"need one count per CPU rank ({pm.n_cpu}), got {len(counts)}")
    offs = []
    for k in range(pm.n_gpu):
        o = np.zeros(pm.alpha + 1, dtype=np.int64)
        np.cumsum(counts[pm.alpha * k: pm.alpha * (k + 1)], out=o[1:])
        offs.append(o)
    return UpdatePattern(send_target=np.arange(pm.n_cpu, dtype=np.int64) // pm.alpha,
                         send_length=counts.copy(), recv_offsets=tuple(offs))


def pack_order_pairs(sp: SparsityPattern, pm: PartitionMap):
    """(row, col) of each packed slot: diag, upper, lower, ifaces (repart.py:253-270)."""
    r, c = sp.local_rows, sp.local_cols
    d = r[r == c]
    up = r < c
    o = np.lexsort((sp.nonlocal_cols, sp.nonlocal_rows, pm.col_owner_cpu(sp.nonlocal_cols)))
    return (np.concatenate((d, r[up], c[up], sp.nonlocal_rows[o])),
            np.concatenate((d, c[up], r[up], sp.nonlocal_cols[o])))


def build_scatter_map(received, local_pattern, nonlocal_pattern, pm: PartitionMap) -> ScatterMap:
    """Buffer position -> value slot (repart.py:273-304), via the native plan."""
    lo, hi = received[0].row_lo, received[-1].row_hi
    pairs = [pack_order_pairs(sp, pm) for sp in received]
    seg = np.concatenate(([0], np.cumsum([len(p[0]) for p in pairs]))).astype(np.int64)
    plan = Plan.from_coo(pm.total_cells, lo, hi, np.concatenate([p[0] for p in pairs]),
                         np.concatenate([p[1] for p in pairs]), seg)
    (lr, lc), (nr, nc) = _patterns_of(plan, lo)
    if not (np.array_equal(lr, local_pattern[0]) and np.array_equal(lc, local_pattern[1])
            and np.array_equal(nr, nonlocal_pattern[0]) and np.array_equal(nc, nonlocal_pattern[1])):
        raise RuntimeError("scatter map: buffer entries do not match the fused pattern slots")
    return ScatterMap(plan=plan)


# ---------------------------------------------------------------------------
# text dumps for test fixtures (repart.py:357-369): same line formats
# ---------------------------------------------------------------------------
def dump_sparsity(sp: SparsityPattern) -> str:
    """``rows lo hi`` then one ``local r c`` / ``nonlocal r c`` line per entry."""
    out = [f"rows {sp.row_lo} {sp.row_hi}\n"]
    for tag, rows, cols in (("local", sp.local_rows, sp.local_cols),
                            ("nonlocal", sp.nonlocal_rows, sp.nonlocal_cols)):
        out.extend(f"{tag} {r} {c}\n" for r, c in zip(rows.tolist(), cols.tolist()))
    return "".join(out)


def dump_scatter(sm: ScatterMap) -> str:
    """One ``b -> local|nonlocal slot`` line per receive-buffer position."""
    tags = ("nonlocal", "local")
    return "".join(f"{b} -> {tags[int(t)]} {i}\n"
                   for b, (t, i) in enumerate(zip(sm.to_local.tolist(), sm.index.tolist())))
