"""Multi-GPU M2L: targets sharded by contiguous Morton ranges, NCCL halo.

The reference has no distributed execution; its only
parallelism is disjoint target chunks over threads sharing the multipole
array (engine.py:145-155).  The B200 build scales the same way across GPUs
(SURVEY.md §8e): every level's occupied cells are ordered by Morton key and
split into one contiguous range per rank; a rank computes the locals of its
own targets only (owners write them, no reduction), and the one exchange step
per level is the source-multipole halo — rows a rank's far lists read but
another rank owns — moved with one ``all_to_all_single`` (NCCL over NVLink on
GPUs, gloo on CPU in the tests).  Range boundaries are aligned to sibling
groups (multiples of 8 in Morton order) so the halo is the 2-cell shell of
SURVEY.md §8e.

Overlap: a rank's owned targets split into *interior* ones,
whose far sources are all owned here, and *boundary* ones.  A step starts the
halo exchange (asynchronous collective on the communicator's stream), runs the
interior targets' M2L on the compute stream meanwhile, waits for the exchange
and then runs the boundary targets — correct by construction (stream order
only, no device-side waiting), so the exchange can never be starved of SMs.

One process per GPU; ``torch.distributed`` provides the plumbing.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def morton_keys(ijk) -> np.ndarray:
    """3-D Morton (Z-order) keys, x in the most significant bit of each triple."""
    ijk = np.asarray(ijk, dtype=np.int64).reshape(-1, 3)
    key = np.zeros(len(ijk), dtype=np.int64)
    for b in range(21):
        for a in range(3):
            key |= ((ijk[:, a] >> b) & 1) << (3 * b + (2 - a))
    return key


def partition_rows(cells_ijk, world: int) -> list[np.ndarray]:
    """Split a level's rows (lexicographic order = reference row order) into
    `world` contiguous Morton ranges of ~equal size, boundaries on sibling
    groups.  Returns the sorted row indices owned by each rank."""
    cells = np.asarray(cells_ijk, dtype=np.int64).reshape(-1, 3)
    n = len(cells)
    order = np.argsort(morton_keys(cells), kind="stable")
    parent = morton_keys(cells[order] >> 1)
    # candidate cut points: starts of sibling groups (parent key changes)
    starts = np.concatenate([[0], np.nonzero(np.diff(parent))[0] + 1, [n]])
    out = []
    prev = 0
    for r in range(1, world + 1):
        target = (n * r) // world
        if r == world:
            cut = n
        else:
            cut = int(starts[np.searchsorted(starts, target)]) if n else 0
            cut = max(cut, prev)
        out.append(np.sort(order[prev:cut]))
        prev = cut
    return out


def split_interior(cells_ijk, level: int, rows, owner) -> tuple[np.ndarray, np.ndarray]:
    """Split target `rows` of a level into (interior, boundary): interior
    targets have every far source (octree.py:148-178: children of the parent's
    neighbours with t.t > 3) owned by the same rank as the target.

    `owner[r]` is the rank owning row r.  Exact: the 216 candidates of each
    target are enumerated like the classifier does."""
    cells = np.asarray(cells_ijk, dtype=np.int64).reshape(-1, 3)
    rows = np.asarray(rows, dtype=np.int64)
    owner = np.asarray(owner, dtype=np.int64)
    if len(rows) == 0:
        return rows.copy(), rows.copy()
    side = 1 << level
    grid = np.full((side, side, side), -1, dtype=np.int64)
    grid[cells[:, 0], cells[:, 1], cells[:, 2]] = owner
    t_ijk = cells[rows]
    me = owner[rows]
    base = 2 * ((t_ijk >> 1) - 1)
    ok = np.ones(len(rows), dtype=bool)
    for dx in range(6):
        for dy in range(6):
            for dz in range(6):
                src = base + np.array([dx, dy, dz])
                inside = np.all((src >= 0) & (src < side), axis=1)
                t = t_ijk - src
                far = (t * t).sum(axis=1) > 3
                sel = inside & far
                o = np.full(len(rows), -1, dtype=np.int64)
                s_in = src[sel]
                o[sel] = grid[s_in[:, 0], s_in[:, 1], s_in[:, 2]]
                ok &= (o < 0) | (o == me)
    return rows[ok], rows[~ok]


def owner_of_rows(parts, n_rows: int) -> np.ndarray:
    """Row -> owning rank from partition_rows' output."""
    owner = np.full(n_rows, -1, dtype=np.int64)
    for r, rows in enumerate(parts):
        owner[np.asarray(rows, dtype=np.int64)] = r
    return owner


@dataclass
class HaloPlan:
    """Rows this rank sends to / receives from every peer (sorted per peer)."""

    send_rows: list  # per peer: np.ndarray of rows owned here, needed there
    recv_rows: list  # per peer: np.ndarray of rows owned there, needed here

    @property
    def send_counts(self):
        return [len(r) for r in self.send_rows]

    @property
    def recv_counts(self):
        return [len(r) for r in self.recv_rows]


def build_halo(owned_by_rank: list, needed_here: np.ndarray, needed_by_rank: list, rank: int) -> HaloPlan:
    """Halo plan from every rank's owned rows and every rank's needed source rows."""
    world = len(owned_by_rank)
    n = max([int(o.max()) + 1 for o in owned_by_rank if len(o)] + [int(x.max()) + 1 for x in needed_by_rank if len(x)]
            + [1])
    owner = np.full(n, -1, dtype=np.int64)
    for r, rows in enumerate(owned_by_rank):
        owner[rows] = r
    recv = []
    need = np.asarray(needed_here, dtype=np.int64)
    for q in range(world):
        recv.append(np.sort(need[(owner[need] == q)]) if q != rank else np.zeros(0, np.int64))
    send = []
    mine = owner == rank
    for q in range(world):
        if q == rank:
            send.append(np.zeros(0, np.int64))
            continue
        nq = np.asarray(needed_by_rank[q], dtype=np.int64)
        send.append(np.sort(nq[mine[nq]]))
    return HaloPlan(send, recv)


def setup_level(dist, cells_ijk, needed_fn):
    """Collective setup for one level.

    needed_fn(owned_rows) -> sorted source rows read by those targets
    (e.g. the handler's ``plan_level_cells_subset``).  Returns
    (owned_rows, halo_plan)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    parts = partition_rows(cells_ijk, world)
    owned = parts[rank]
    needed = np.asarray(needed_fn(owned), dtype=np.int64)
    gathered = [None] * world
    dist.all_gather_object(gathered, needed)
    return owned, build_halo(parts, needed, gathered, rank)


def exchange_halo(dist, mpoles, halo: HaloPlan, group=None):
    """Fill the halo rows of this rank's (full-size) multipole array from
    their owners: one all_to_all_single of packed rows (NCCL on CUDA tensors).
    Rows owned here are left untouched."""
    import torch

    dev = mpoles.device
    send_idx = torch.as_tensor(np.concatenate(halo.send_rows) if halo.send_rows else np.zeros(0, np.int64),
                               device=dev)
    recv_idx = torch.as_tensor(np.concatenate(halo.recv_rows) if halo.recv_rows else np.zeros(0, np.int64),
                               device=dev)
    send = mpoles.index_select(0, send_idx).contiguous()
    recv = torch.empty((len(recv_idx),) + tuple(mpoles.shape[1:]), dtype=mpoles.dtype, device=dev)
    if mpoles.is_complex():  # NCCL/gloo all_to_all on real views
        dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), halo.recv_counts,
                               halo.send_counts, group=group)
    else:
        dist.all_to_all_single(recv, send, halo.recv_counts, halo.send_counts, group=group)
    if len(recv_idx):
        mpoles.index_copy_(0, recv_idx, recv)
    return mpoles


class PreparedHalo:
    """Device-resident index tensors of a HaloPlan (built once, reused every step)."""

    def __init__(self, halo: HaloPlan, device):
        import torch

        self.halo = halo
        cat = lambda rows: np.concatenate(rows) if rows else np.zeros(0, np.int64)  # noqa: E731
        self.send_idx = torch.as_tensor(cat(halo.send_rows), device=device)
        self.recv_idx = torch.as_tensor(cat(halo.recv_rows), device=device)
        self.send_counts = halo.send_counts
        self.recv_counts = halo.recv_counts

    def exchange(self, dist, mpoles, group=None):
        return self.start(dist, mpoles, group=group).finish()

    def start(self, dist, mpoles, group=None) -> "_PendingHalo":
        """Launch the exchange asynchronously (the collective runs on the
        communicator's stream after the packing on the current stream);
        ``finish()`` makes the current stream wait and scatters the rows."""
        import torch

        send = mpoles.index_select(0, self.send_idx)
        recv = torch.empty((len(self.recv_idx),) + tuple(mpoles.shape[1:]), dtype=mpoles.dtype, device=mpoles.device)
        if mpoles.is_complex():
            work = dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), self.recv_counts,
                                          self.send_counts, group=group, async_op=True)
        else:
            work = dist.all_to_all_single(recv, send, self.recv_counts, self.send_counts, group=group, async_op=True)
        return _PendingHalo(work, mpoles, self.recv_idx, recv, send)


class _PendingHalo:
    def __init__(self, work, mpoles, recv_idx, recv, send):
        self.work, self.mpoles, self.recv_idx, self.recv, self._send = work, mpoles, recv_idx, recv, send

    def finish(self):
        self.work.wait()
        if len(self.recv_idx):
            self.mpoles.index_copy_(0, self.recv_idx, self.recv)
        return self.mpoles


def overlapped_step(dist, mpoles: dict, halos: dict, apply_interior, apply_boundary, group=None):
    """One sharded M2L step with the halo exchange overlapped by the interior
    targets: start every level's exchange, apply the interior targets, finish
    the exchanges, apply the boundary targets."""
    pending = [halos[lvl].start(dist, mpoles[lvl], group=group) for lvl in sorted(halos)]
    apply_interior()
    for p in pending:
        p.finish()
    apply_boundary()


# ---------------------------------------------------------------------------
# Shard-local sharded M2L (owned rows + compacted halo per rank)
# ---------------------------------------------------------------------------


def device_far_lists(cells_ijk, level: int, target_rows, device: int = 0):
    """CSR far lists of ``target_rows`` of a level (sources = every occupied
    cell, global row numbers) from the device classifier
    (cfm_classify_targets_*; the lists of octree.py:148-178).  Returns
    (offsets[n + 1], src[P] int64, t[P, 3] int8)."""
    import ctypes

    from . import _native

    lib = _native.load()
    c = np.ascontiguousarray(cells_ijk, dtype=np.int32).reshape(-1, 3)
    rows = np.ascontiguousarray(target_rows, dtype=np.int64)
    off = np.zeros(len(rows) + 1, np.int64)
    tot = ctypes.c_int64()
    _native.check(lib.cfm_classify_targets_count(int(device), int(level), len(c), c.ctypes.data, len(rows),
                                                 rows.ctypes.data, off.ctypes.data, ctypes.byref(tot)))
    src = np.empty(tot.value, np.int32)
    t = np.empty((tot.value, 3), np.int8)
    if tot.value:
        _native.check(lib.cfm_classify_targets_fill(int(device), int(level), len(c), c.ctypes.data, len(rows),
                                                    rows.ctypes.data, off.ctypes.data, src.ctypes.data,
                                                    t.ctypes.data))
    return off, src.astype(np.int64), t


def native_pack(src, rows_dev, out):
    """out[k] = src[rows[k]] on the device (cfm_gather_rows, the halo pack kernel)."""
    import torch

    from . import _native

    row_doubles = src.shape[1] * (2 if src.is_complex() else 1)
    _native.check(_native.load().cfm_gather_rows(src.device.index, src.data_ptr(), row_doubles, rows_dev.data_ptr(),
                                                 len(rows_dev), out.data_ptr(),
                                                 ctypes_stream(torch.cuda.current_stream(src.device))))
    return out


def ctypes_stream(stream):
    import ctypes

    return ctypes.c_void_p(stream.cuda_stream)


@dataclass
class ShardLevel:
    """One level on one rank.  Local row space: [owned rows (ascending global
    row), halo rows grouped by owning peer (peer ascending, rows ascending)],
    so the all_to_all receive buffer IS the halo block of the local array."""

    level: int
    owned: np.ndarray        # global rows owned here (ascending)
    halo: np.ndarray         # global rows received, in local order
    send_local: np.ndarray   # local rows (< n_owned) packed for the peers, peer-major
    send_counts: list
    recv_counts: list
    pairs: int
    interior_pairs: int
    boundary_pairs: int

    @property
    def n_owned(self) -> int:
        return len(self.owned)

    @property
    def n_local(self) -> int:
        return len(self.owned) + len(self.halo)


class ShardedM2L:
    """Targets of every level sharded by contiguous Morton range (SURVEY.md
    §8e), shard-local level arrays (owned rows + the compacted halo), one
    halo all_to_all per level per step, overlapped by the interior targets.

    ``h_boundary`` / ``h_interior``: two precomputed handlers of the same
    variant (each holds one plan per level).  ``lists_fn(cells, level, rows)``
    gives CSR far lists of target rows in global rows (default: the device
    classifier); ``pack_fn(src, rows_dev, out)`` packs send rows (default:
    the cfm_gather_rows kernel).  Results equal the single-GPU apply bitwise:
    every target sums its own pairs in the same order on its owner."""

    def __init__(self, dist, h_boundary, h_interior, cells: dict, device=None, lists_fn=None, pack_fn=None,
                 complex_data: bool | None = None, group=None):
        import torch

        self.dist, self.group = dist, group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.h_bnd, self.h_int = h_boundary, h_interior
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        dev_index = self.device.index if self.device.type == "cuda" else 0
        self.lists_fn = lists_fn or (lambda c, lvl, rows: device_far_lists(c, lvl, rows, dev_index))
        self.pack_fn = pack_fn or native_pack
        self.staged = dist.get_backend(group) == "gloo" and self.device.type == "cuda"
        self.levels: dict[int, ShardLevel] = {}
        self.int_levels, self.bnd_levels = [], []
        self._send_idx = {}
        for lvl in sorted(cells):
            self._setup_level(lvl, np.asarray(cells[lvl]), complex_data)

    def _setup_level(self, lvl, cells, complex_data):
        import torch

        parts = partition_rows(cells, self.world)
        owned = parts[self.rank]
        off, src, t = self.lists_fn(cells, lvl, owned)
        need = np.unique(src)
        owner = owner_of_rows(parts, len(cells))
        halo_need = need[owner[need] != self.rank]
        gathered = [None] * self.world
        self.dist.all_gather_object(gathered, halo_need, group=self.group)
        recv = [np.sort(halo_need[owner[halo_need] == q]) if q != self.rank else np.zeros(0, np.int64)
                for q in range(self.world)]
        halo = np.concatenate(recv) if recv else np.zeros(0, np.int64)
        send = []
        for q in range(self.world):
            if q == self.rank:
                send.append(np.zeros(0, np.int64))
                continue
            nq = np.asarray(gathered[q], dtype=np.int64)
            send.append(np.sort(nq[owner[nq] == self.rank]))
        g2l = np.full(len(cells), -1, np.int64)
        g2l[owned] = np.arange(len(owned))
        g2l[halo] = len(owned) + np.arange(len(halo))
        send_local = g2l[np.concatenate(send)] if send else np.zeros(0, np.int64)
        src_l = g2l[src]
        counts = np.diff(off)
        tgt_l = np.arange(len(owned), dtype=np.int64)
        # interior targets: every source owned here (none in the halo block)
        halo_pairs = np.add.reduceat((src_l >= len(owned)).astype(np.int64), off[:-1]) if len(src_l) else \
            np.zeros(len(owned), np.int64)
        halo_pairs = np.where(counts > 0, halo_pairs, 0)
        inner = halo_pairs == 0
        n_local = len(owned) + len(halo)
        sl = ShardLevel(lvl, owned, halo, send_local, [len(s) for s in send], [len(r) for r in recv],
                        int(off[-1]), 0, 0)
        for hh, mask, lst, attr in ((self.h_int, inner, self.int_levels, "interior_pairs"),
                                    (self.h_bnd, ~inner, self.bnd_levels, "boundary_pairs")):
            sel = np.nonzero(mask & (counts > 0))[0]
            if len(sel) == 0:
                continue
            c = counts[sel]
            o = np.zeros(len(sel) + 1, np.int64)
            np.cumsum(c, out=o[1:])
            take = np.repeat(off[sel], c) + (np.arange(int(o[-1])) - np.repeat(o[:-1], c))
            hh.plan_level_csr(lvl, tgt_l[sel], o, src_l[take], t[take], n_local, complex_data)
            setattr(sl, attr, int(o[-1]))
            lst.append(lvl)
        self.levels[lvl] = sl
        self._send_idx[lvl] = torch.as_tensor(send_local, dtype=torch.int64, device=self.device)

    # -------------------------------------------------------------- arrays
    def allocate(self, size: int, dtype):
        """Zeroed shard-local (mpoles, locals) per level: n_local rows each."""
        import torch

        return {lvl: (torch.zeros((sl.n_local, size), dtype=dtype, device=self.device),
                      torch.zeros((sl.n_local, size), dtype=dtype, device=self.device))
                for lvl, sl in self.levels.items()}

    @property
    def pairs(self) -> int:
        return sum(sl.pairs for sl in self.levels.values())

    # -------------------------------------------------------------- step
    def _start(self, lvl, mp):
        import torch

        sl = self.levels[lvl]
        send = torch.empty((len(sl.send_local),) + tuple(mp.shape[1:]), dtype=mp.dtype, device=mp.device)
        if len(sl.send_local):
            self.pack_fn(mp, self._send_idx[lvl], send)
        recv = mp[sl.n_owned:]
        real = (lambda x: torch.view_as_real(x)) if mp.is_complex() else (lambda x: x)
        if self.staged:  # gloo cannot move CUDA tensors: stage the packed rows through the host
            h_send = send.cpu()
            h_recv = torch.empty(recv.shape, dtype=recv.dtype)
            self.dist.all_to_all_single(real(h_recv), real(h_send), sl.recv_counts, sl.send_counts,
                                        group=self.group)
            recv.copy_(h_recv)
            return None, send
        work = self.dist.all_to_all_single(real(recv), real(send), sl.recv_counts, sl.send_counts,
                                           group=self.group, async_op=True)
        return work, send

    def step(self, arrays: dict) -> int:
        """One M2L step of this rank: exchange every level's halo (async),
        interior targets meanwhile, then the boundary targets.  ``arrays``:
        level -> (mpoles_local, locals_local).  Returns the counted flops."""
        pending = [self._start(lvl, arrays[lvl][0]) for lvl in sorted(self.levels)]
        flops = 0
        if self.int_levels:
            flops += self.h_int.apply_levels({l: arrays[l] for l in self.int_levels})
        for work, _ in pending:
            if work is not None:
                work.wait()
        if self.bnd_levels:
            flops += self.h_bnd.apply_levels({l: arrays[l] for l in self.bnd_levels})
        return flops

    def launches(self) -> int:
        n = 0
        for hh, lv in ((self.h_int, self.int_levels), (self.h_bnd, self.bnd_levels)):
            if lv and hasattr(hh, "last_apply_stats"):
                n += hh.last_apply_stats()[1]
        return n + sum(1 for sl in self.levels.values() if len(sl.send_local))
