"""Row-slab decomposition plan for multi-GPU solves.

The 2D unknowns are lexicographic with x fastest (reference src/assembly.cpp:255),
so a contiguous band of iy rows is a contiguous slice of every vector.  Each rank
owns one band per level; every level operator is a Kronecker sum of banded 1D
factors (half-bandwidth ``band``), so an apply on a band needs ``band`` halo rows
from each neighbour and nothing else.

Level hierarchy (reference src/precond.cpp:115-124): n_{l+1} = n_l // 2 while
n_l > coarsest.  The transfers couple rows as follows (0-based indices):

* linear z (src/precond.cpp:57-76): coarse q <- fine rows 2q, 2q+1, 2q+2;
  fine i <- coarse (i-1)/2 (odd i) or i/2-1, i/2 (even i);
* Bezier z (src/precond.cpp:34-55): coarse q <- fine rows 2q-1 .. 2q+3;
  fine i <- coarse (i-3)/2 .. (i+1)/2 (odd i) or i/2-1, i/2 (even i).

Boundaries are chosen on the gather level (the first agglomerated MG level) and
doubled going up, so with fine band [2Q_r, 2Q_{r+1}) the coarse band
[Q_r, Q_{r+1}) is produced locally from the fine band plus at most two halo
rows (``TRANSFER_HALO``).  Levels at or below the gather level are small; their
restricted right-hand side is allgathered and the rest of the V-cycle (and the
coarsest direct solve) runs redundantly on every rank.  The deflation coarse
grid (per_dim // 2, Bezier z) shares its bounds with MG level 1; its E solve is
done redundantly on the allgathered coarse vector.

The plan is pure host logic: it is shared by the device implementation's
launcher and by the CPU emulation in tests/slab_emulation.py, which checks it
with a world_size-2 gloo run against the single-domain solve.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

# (top, bottom) halo rows of the INPUT of each transfer, per kind
TRANSFER_HALO = {
    ("restrict", "linear"): (0, 1),   # coarse q reads fine 2q .. 2q+2
    ("prolong", "linear"): (1, 0),    # fine [2Q_r, 2Q_{r+1}) reads coarse Q_r-1 .. Q_{r+1}-1
    ("restrict", "bezier"): (1, 2),   # coarse q reads fine 2q-1 .. 2q+3
    ("prolong", "bezier"): (1, 1),    # fine reads coarse Q_r-1 .. Q_{r+1}
}


def level_sizes(per_dim: int, coarsest: int = 32) -> List[int]:
    """MG level sizes per dimension (src/precond.cpp:115-124)."""
    sizes = [per_dim]
    while sizes[-1] > coarsest:
        sizes.append(sizes[-1] // 2)
    return sizes


@dataclass
class LevelSlabs:
    n: int                 # rows (and columns) of the level grid
    bounds: List[int]      # world_size + 1 row boundaries (distributed levels)
    band: int              # half-bandwidth of the level operator = stencil halo rows
    distributed: bool      # False: held whole and processed redundantly on every rank

    def rows(self, rank: int) -> Tuple[int, int]:
        if not self.distributed:
            return 0, self.n
        return self.bounds[rank], self.bounds[rank + 1]

    def count(self, rank: int) -> int:
        r0, r1 = self.rows(rank)
        return r1 - r0


@dataclass
class SlabPlan:
    world_size: int
    levels: List[LevelSlabs]          # MG hierarchy, levels[0] = fine grid
    coarse: LevelSlabs                # deflation coarse grid (per_dim // 2)
    gather_level: int                 # first agglomerated MG level (>= 1)
    notes: List[str] = field(default_factory=list)

    @property
    def fine(self) -> LevelSlabs:
        return self.levels[0]

    def halo(self, what: str, level: int = 0, kind: str = "linear") -> Tuple[int, int]:
        """(top, bottom) halo rows an operation needs on its input at ``level``."""
        if what in ("apply", "resid", "jacobi", "resnorm"):
            b = self.levels[level].band
            return b, b
        if what == "e_apply":
            b = self.coarse.band
            return b, b
        return TRANSFER_HALO[(what, kind)]

    def gather_bytes(self, level: int) -> int:
        """Bytes every rank receives when a complex level vector is allgathered."""
        n = self.levels[level].n if level >= 0 else self.coarse.n
        return 16 * n * n

    def halo_bytes(self, level: int, rows: int) -> int:
        return 16 * rows * self.levels[level].n

    def per_iteration(self, smooth_steps: int = 1, cycles: int = 1) -> dict:
        """Communication of one GMRES iteration of the DC_MG chain on this plan
        (op = P MG^-1 A, one-reduction Arnoldi, true-residual monitor)."""
        if self.world_size == 1:
            return {"allreduce": 0, "allgather": 0, "halo_exchange": 0}
        g = self.gather_level
        halo = 1  # A v on the fine level
        for l in range(g):
            # residual, restriction input, prolongation input (distributed
            # coarse level only), post-smoothing sweeps, pre-sweeps after the
            # first (the first starts from zero and needs no apply)
            halo += cycles * (2 + (1 if l + 1 < g else 0) + smooth_steps + (smooth_steps - 1))
        # later cycles start the FINE level from a nonzero iterate (coarser
        # levels always start from zero, src/precond.cpp:150): one more exchange
        halo += cycles - 1
        halo += 2  # projection: A w, Bezier restriction input (E solution is gathered)
        halo += 1  # monitor: A x
        return {"allreduce": 3, "allgather": cycles + 1, "halo_exchange": halo}


def _split(n: int, parts: int) -> List[int]:
    return [(r * n + parts // 2) // parts for r in range(parts + 1)]


def plan(per_dim: int, bands: List[int], world_size: int, coarse_band: int, coarsest: int = 32,
         agglomerate_at: int = 200, min_rows: int = 8) -> SlabPlan:
    """Plan the row slabs of a 2D DC_MG solve.

    ``bands[l]``: half-bandwidth of MG level l; ``coarse_band``: of E.
    Levels with n <= ``agglomerate_at`` (and every level whose smallest slab would
    fall below ``max(min_rows, halo)`` rows) are agglomerated."""
    sizes = level_sizes(per_dim, coarsest)
    if len(bands) != len(sizes):
        raise ValueError(f"bands has {len(bands)} entries for {len(sizes)} levels")
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    L = len(sizes)
    notes = []
    if L == 1:
        raise ValueError("a single-level hierarchy has nothing to distribute")
    # gather level g: first level that is small enough to agglomerate; the
    # distributed levels 0..g-1 must each leave every rank >= need rows
    g = 1
    while g < L - 1 and sizes[g] > agglomerate_at:
        g += 1
    while g > 1:
        q = _split(sizes[g], world_size)
        ok = True
        for l in range(g):
            f = 1 << (g - l)
            b = [v * f for v in q[:-1]] + [sizes[l]]
            need = max(min_rows, bands[l] + 2)
            if min(b[r + 1] - b[r] for r in range(world_size)) < need:
                ok = False
        if ok:
            break
        g -= 1
        notes.append(f"gather level lowered to {g}: slabs too thin")
    q = _split(sizes[g], world_size)
    levels = []
    for l, n in enumerate(sizes):
        if l <= g:
            f = 1 << (g - l)
            b = [v * f for v in q[:-1]] + [n]
        else:
            b = [0] * world_size + [n]
        levels.append(LevelSlabs(n, b, bands[l], l < g))
    if world_size > 1:
        need0 = max(bands[0], 2)
        if min(levels[0].count(r) for r in range(world_size)) < need0:
            raise ValueError(f"per_dim {per_dim} too small for {world_size} slabs")
    coarse = LevelSlabs(per_dim // 2, list(levels[1].bounds), coarse_band, False)
    return SlabPlan(world_size, levels, coarse, g, notes)
