"""ORACLE -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker (or as the
CPU baseline being timed).  The product path (paper_1210_7292_b200) never
imports it.

CPU restatement (numpy) of the reference's M2L path, written independently of
the product code, each piece citing the reference it follows
(/root/reference/pkg/src/chebfmm):

  cheb_roots / nodes           interp.py:45-70, 155-161, 206-211
  canonicalize, perm tables    symmetry.py:63-111
  far lists                    octree.py:148-178 (+ transfer_vector :50-61, _is_near :64-65)
  operator assembly            kernels.py:75-97, 142-179
  truncated SVD / ACA          lowrank.py:47-62, 65-184
  precompute                   m2l.py:136-273
  apply (plain/sym/shared/blocked, flop model)   m2l.py:279-452

Parity is PINNED: tests/test_oracle_golden.py checks every function here
against tests/golden/*.npz, which tests/golden/make_golden.py produced by
executing the reference itself.  The reference pins no golden vectors of its
own, so those executed fixtures are the pin.

Two apply forms are provided: ``apply_faithful`` mirrors the reference's
per-pair / 128-column-flush loops (and is what the CPU baseline times), and
``apply_fast`` is a vectorized regrouping (per transfer vector) used for the
larger parity checks; tests cross-check the two.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

VARIANTS = ("na", "nasym", "nablk", "sa", "sarcmp", "ia", "iasym", "iablk")
AXIS_ORDERS = [(1, 2, 3), (1, 3, 2), (2, 1, 3), (2, 3, 1), (3, 1, 2), (3, 2, 1)]


# ------------------------------------------------------------------ interpolation
def cheb_roots(order: int) -> np.ndarray:
    """interp.py:45-70: cos((2i-1) pi / 2l), largest first, mirrored halves."""
    out = np.empty(order)
    h = order // 2
    i = np.arange(1, h + 1)
    out[:h] = np.cos((2 * i - 1) * np.pi / (2 * order))
    if order % 2:
        out[h] = 0.0
    out[order - h:] = -out[h - 1::-1]
    return out


@lru_cache(maxsize=None)
def components(order: int) -> np.ndarray:
    j = np.arange(order**3)
    return np.stack([j % order, (j // order) % order, j // order**2])


def nodes3d(order: int) -> np.ndarray:
    return cheb_roots(order)[components(order)].T.copy()


# ------------------------------------------------------------------ symmetry
def canonicalize(t):
    """symmetry.py:63-75 -> (t_sym, flips, axis_order(1-based))."""
    flips = tuple(c < 0 for c in t)
    a = [abs(int(c)) for c in t]
    order = tuple(int(i) + 1 for i in sorted(range(3), key=lambda i: (-a[i], i)))
    return tuple(a[i - 1] for i in order), flips, order


def perm_id(flips, order) -> int:
    return (int(flips[0]) | int(flips[1]) << 1 | int(flips[2]) << 2) * 6 + AXIS_ORDERS.index(tuple(order))


@lru_cache(maxsize=None)
def perm_table(flips, axis_order, order: int) -> np.ndarray:
    """symmetry.py:86-102."""
    comp = components(order).copy()
    for ax in range(3):
        if flips[ax]:
            comp[ax] = order - 1 - comp[ax]
    comp = comp[[i - 1 for i in axis_order]]
    return comp[0] + comp[1] * order + comp[2] * order**2


@lru_cache(maxsize=None)
def inv_table(flips, axis_order, order: int) -> np.ndarray:
    tab = perm_table(flips, axis_order, order)
    inv = np.empty_like(tab)
    inv[tab] = np.arange(tab.size)
    return inv


def cone_of(vectors):
    """Sorted cone representatives and t -> (rep index, flips, order) (symmetry.py:114-137)."""
    assign = {}
    reps = set()
    for t in vectors:
        t = tuple(int(c) for c in t)
        ts, fl, od = canonicalize(t)
        reps.add(ts)
        assign[t] = (ts, fl, od)
    cone = sorted(reps)
    idx = {r: i for i, r in enumerate(cone)}
    return cone, {t: (idx[ts], fl, od) for t, (ts, fl, od) in assign.items()}


def full_far_field():
    r = range(-3, 4)
    return [(a, b, c) for a in r for b in r for c in r if a * a + b * b + c * c > 3]


# ------------------------------------------------------------------ octree lists
def level_cells_from_points(points, center, half_width, depth):
    """Occupied cells per level, lexicographically sorted (octree.py:93-127)."""
    pts = np.asarray(points, dtype=float)
    low = np.asarray(center, dtype=float) - half_width
    ref = (pts - low) / (2.0 * half_width)
    side = 1 << depth
    ijk = np.minimum((ref * side).astype(np.int64), side - 1)
    out = {}
    keys = np.unique((ijk[:, 0] << 42) | (ijk[:, 1] << 21) | ijk[:, 2])
    cur = np.stack([keys >> 42, (keys >> 21) & ((1 << 21) - 1), keys & ((1 << 21) - 1)], axis=1)
    out[depth] = cur
    for lvl in range(depth - 1, -1, -1):
        par = cur >> 1
        k = np.unique((par[:, 0] << 42) | (par[:, 1] << 21) | par[:, 2])
        cur = np.stack([k >> 42, (k >> 21) & ((1 << 21) - 1), k & ((1 << 21) - 1)], axis=1)
        out[lvl] = cur
    return out


def far_lists(cells: np.ndarray, level: int, targets=None):
    """Far lists of every occupied cell of a level in the reference's order:
    targets by row (lexicographic ijk), sources by ijk (octree.py:148-178).
    Returns CSR (tgt_rows, offsets, src_rows, t) over targets with non-empty lists
    (engine.py:114-119 drops the empty ones).  ``targets`` restricts the
    targets to a sorted subset of rows (sampled parity at full size)."""
    all_cells = np.asarray(cells, dtype=np.int64).reshape(-1, 3)
    n = len(all_cells)
    sel = np.arange(n) if targets is None else np.asarray(targets, dtype=np.int64)
    side = 1 << level
    if level < 2 or n == 0:
        z = np.zeros(0, np.int64)
        return z, np.zeros(1, np.int64), z, np.zeros((0, 3), np.int64)
    key = (all_cells[:, 0] * side + all_cells[:, 1]) * side + all_cells[:, 2]
    cells = all_cells[sel]
    order = np.argsort(key)
    skey = key[order]
    # 216 candidate offsets in lexicographic order of the source ijk
    d = np.arange(6)
    cand = np.stack(np.meshgrid(d, d, d, indexing="ij"), axis=-1).reshape(-1, 3)  # lex (x, y, z)
    base = 2 * ((cells >> 1) - 1)  # (n, 3)
    src_ijk = base[:, None, :] + cand[None, :, :]  # (n, 216, 3)
    t = cells[:, None, :] - src_ijk
    inb = np.all((src_ijk >= 0) & (src_ijk < side), axis=-1)
    far = np.sum(t * t, axis=-1) > 3
    skeys = (src_ijk[..., 0] * side + src_ijk[..., 1]) * side + src_ijk[..., 2]
    pos = np.searchsorted(skey, np.where(inb, skeys, -1))
    pos_c = np.minimum(pos, n - 1)
    occ = inb & (skey[pos_c] == skeys)
    keep = occ & far
    counts = keep.sum(axis=1)
    rows = np.nonzero(counts)[0]
    off = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(counts[rows], out=off[1:])
    src_rows = order[pos_c[rows][keep[rows]]]
    return sel[rows].astype(np.int64), off, src_rows.astype(np.int64), t[rows][keep[rows]].astype(np.int64)


def csr_to_batch(tgt, off, src, t):
    return [(int(tgt[i]), [(int(src[q]), tuple(int(c) for c in t[q])) for q in range(off[i], off[i + 1])])
            for i in range(len(tgt))]


# ------------------------------------------------------------------ kernels / operators
def laplace_profile(r):
    return 1.0 / (4.0 * np.pi * r)


def helmholtz_profile(k):
    def prof(r):
        return np.exp(1j * k * r) / (4.0 * np.pi * r)
    return prof


def assemble(profile, t, width, order) -> np.ndarray:
    """kernels.py:142-179 (target cell at w*t, source cell at the origin)."""
    half = 0.5 * width
    nd = nodes3d(order)
    x = np.asarray((width * t[0], width * t[1], width * t[2]), dtype=float) + half * nd
    y = np.asarray((0.0, 0.0, 0.0)) + half * nd
    r = np.sqrt(np.sum((x[:, None, :] - y[None, :, :]) ** 2, axis=-1))
    return profile(r)


def eps_rank(s, eps) -> int:
    if s.size == 0 or s[0] == 0.0:
        return 0
    return int(np.count_nonzero(s > eps * s[0]))


def tsvd(a, eps):
    """lowrank.py:53-62 -> (left, right) with A ~ left right^H."""
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    r = eps_rank(s, eps)
    return u[:, :r] * s[:r], vh[:r].conj().T


def aca_svd(evaluate, m, n, eps):
    """lowrank.py:65-184 (ACA with row probing, then QR + SVD recompression)."""
    cols = np.arange(n)
    rows = np.arange(m)
    us, vs = [], []
    urow, ucol = set(), set()
    nrm = 0.0
    nxt = 0
    conv = False
    for _ in range(min(m, n)):
        row = None
        for c in [nxt] + [r for r in range(m) if r not in urow][:4]:
            if c in urow:
                continue
            tr = np.asarray(evaluate(c, cols)).copy()
            for u, v in zip(us, vs):
                tr -= u[c] * v
            if np.max(np.abs(tr)) > 0.0:
                nxt, row = c, tr
                break
        if row is None:
            conv = bool(us)
            break
        urow.add(nxt)
        mk = row.copy()
        if ucol:
            mk[sorted(ucol)] = 0.0
        j = int(np.argmax(np.abs(mk)))
        piv = row[j]
        if piv == 0.0:
            conv = False
            break
        ucol.add(j)
        vn = row / piv
        un = np.asarray(evaluate(rows, j)).copy()
        for u, v in zip(us, vs):
            un -= v[j] * u
        cross = sum(np.vdot(u, un) * np.vdot(v, vn) for u, v in zip(us, vs))
        inc = float(np.real(np.vdot(un, un)) * np.real(np.vdot(vn, vn)))
        nrm = max(nrm + 2.0 * float(np.real(cross)) + inc, 0.0)
        us.append(un)
        vs.append(vn)
        if inc <= eps**2 * nrm:
            conv = True
            break
        cm = np.abs(un)
        cm[sorted(urow)] = 0.0
        nxt = int(np.argmax(cm))
    else:
        conv = True
    if not conv:
        dense = np.asarray(evaluate(np.arange(m)[:, None], np.arange(n)[None, :]))
        return tsvd(dense, eps)
    if not us:
        dt = np.asarray(evaluate(0, 0)).dtype
        return np.zeros((m, 0), dt), np.zeros((n, 0), dt)
    U = np.column_stack(us)
    V = np.column_stack([v.conj() for v in vs])
    qu, ru = np.linalg.qr(U)
    qv, rv = np.linalg.qr(V)
    uc, s, vch = np.linalg.svd(ru @ rv.conj().T)
    r = eps_rank(s, eps)
    return qu @ (uc[:, :r] * s[:r]), qv @ vch[:r].conj().T


# ------------------------------------------------------------------ handler port
class OracleM2L:
    """CPU port of M2LHandler (m2l.py:90-536) for checking and baseline timing."""

    def __init__(self, variant, profile, dtype, order, eps, homogeneity=None, compression="svd", block_size=128):
        assert variant in VARIANTS
        self.variant = variant
        self.profile = profile
        self.dtype = np.dtype(dtype)
        self.order = order
        self.size = order**3
        self.eps = eps
        self.degree = homogeneity
        self.compression = compression
        self.block_size = block_size
        self.sym = variant in ("nasym", "nablk", "iasym", "iablk")
        self.blk = variant in ("nablk", "iablk")
        self.dense = variant in ("na", "nasym", "nablk")
        self.shared = variant in ("sa", "sarcmp")
        self.groups = {}
        self.level_group = {}
        self.level_scale = {}
        self.ops = {}
        self.flops = {}
        self.factorization_calls = 0

    # m2l.py:136-169
    def precompute(self, level_transfers, level_widths):
        levels = sorted(l for l, ts in level_transfers.items() if ts)
        if not levels:
            return self
        if self.degree is not None:
            union = sorted({tuple(int(c) for c in t) for l in levels for t in level_transfers[l]})
            ref = levels[0]
            self.groups["ref"] = (union, level_widths[ref])
            for l in levels:
                self.level_group[l] = "ref"
                self.level_scale[l] = (level_widths[l] / level_widths[ref]) ** self.degree
            self._build("ref")
        else:
            for l in levels:
                self.groups[l] = (sorted(tuple(int(c) for c in t) for t in level_transfers[l]), level_widths[l])
                self.level_group[l] = l
                self.level_scale[l] = 1.0
                self._build(l)
        return self

    def _op(self, t, width):
        return assemble(self.profile, t, width, self.order).astype(self.dtype, copy=False)

    def _build(self, key):
        transfers, width = self.groups[key]
        cone, assign = cone_of(transfers)
        vectors = cone if self.sym else transfers
        if self.dense:
            self.ops[key] = {"cone": cone, "assign": assign, "op": {t: self._op(t, width) for t in vectors}}
        elif self.shared:
            self.ops[key] = {"cone": cone, "assign": assign, "sa": self._shared(transfers, width)}
        else:
            facs = {}
            for t in vectors:
                self.factorization_calls += 1
                if self.compression == "svd":
                    facs[t] = tsvd(self._op(t, width), self.eps)
                else:
                    half = 0.5 * width
                    nd = nodes3d(self.order)
                    xn = np.asarray((width * t[0], width * t[1], width * t[2])) + half * nd
                    yn = half * nd

                    def ev(i, j, xn=xn, yn=yn):
                        d = xn[np.asarray(i)] - yn[np.asarray(j)]
                        return self.profile(np.sqrt(np.sum(d**2, axis=-1)))

                    facs[t] = aca_svd(ev, self.size, self.size, self.eps)
            self.ops[key] = {"cone": cone, "assign": assign, "op": facs}

    def _shared(self, transfers, width):
        n = self.size
        blocks = {t: self._op(t, width) for t in transfers}
        row = np.hstack([blocks[t] for t in transfers])
        col = np.vstack([blocks[t] for t in transfers])
        if self.compression == "svd":
            u_row, s_row, vh_row = np.linalg.svd(row, full_matrices=False)
            _, s_col, vh_col = np.linalg.svd(col, full_matrices=False)
            r = max(eps_rank(s_row, self.eps), eps_rank(s_col, self.eps))
            u, sig, vh, b = u_row[:, :r], s_row[:r], vh_row[:r], vh_col[:r].conj().T
        else:  # m2l.py:241-255: ACA on the concatenations
            L, R = aca_svd(lambda i, j: row[np.asarray(i), np.asarray(j)], n, row.shape[1], self.eps)
            _, Rc = aca_svd(lambda i, j: col[np.asarray(i), np.asarray(j)], col.shape[0], n, self.eps)
            sig = np.linalg.norm(L, axis=0)
            u = L / sig
            vh = R.conj().T
            b = Rc
        self.factorization_calls += 2
        cores = {t: ("dense", (sig[:, None] * vh[:, k * n:(k + 1) * n]) @ b) for k, t in enumerate(transfers)}
        if self.variant == "sarcmp":
            for t, (_, c) in list(cores.items()):
                L, R = tsvd(c, self.eps)
                self.factorization_calls += 1
                if L.shape[1] * (u.shape[1] + b.shape[1]) < u.shape[1] * b.shape[1]:
                    cores[t] = ("factored", (L, R))
        return {"u": u, "b": b, "cores": cores, "rank": max(u.shape[1], b.shape[1])}

    def level_ranks(self, level):
        key = self.level_group.get(level)
        if key is None:
            return []
        transfers, _ = self.groups[key]
        d = self.ops[key]
        if self.dense:
            return [self.size] * len(transfers)
        if self.shared:
            sa = d["sa"]
            return [sa["rank"] if sa["cores"][t][0] == "dense" else sa["cores"][t][1][0].shape[1] for t in transfers]
        if self.sym:
            return [d["op"][d["cone"][d["assign"][t][0]]][0].shape[1] for t in transfers]
        return [d["op"][t][0].shape[1] for t in transfers]

    # ---- faithful apply (m2l.py:279-452)
    def apply_faithful(self, level, batch, mpoles, locals_out) -> int:
        self.flush_log = []
        if not batch:
            return 0
        key = self.level_group[level]
        scale = self.level_scale[level]
        d = self.ops[key]
        n = self.size
        acc_dt = np.result_type(self.dtype, mpoles.dtype)
        flops = 0
        if self.shared:
            sa = d["sa"]
            u, b, cores = sa["u"], sa["b"], sa["cores"]
            r_u, r_b = u.shape[1], b.shape[1]
            srcs = sorted({s for _, far in batch for s, _ in far})
            if not srcs:
                return 0
            pos = {s: i for i, s in enumerate(srcs)}
            wt = b.conj().T @ mpoles[srcs].T
            flops += 2 * n * r_b * len(srcs)
            for tgt, far in batch:
                if not far:
                    continue
                acc = np.zeros(r_u, dtype=acc_dt)
                for s, t in far:
                    kind, c = cores[tuple(t)]
                    w = wt[:, pos[s]]
                    if kind == "dense":
                        acc += c @ w
                        flops += 2 * r_u * r_b
                    else:
                        L, R = c
                        acc += L @ (R.conj().T @ w)
                        flops += 2 * L.shape[1] * (r_u + r_b)
                locals_out[tgt] += scale * (u @ acc)
                flops += 2 * n * r_u
        elif self.blk:
            cone, assign = d["cone"], d["assign"]
            cap = self.block_size
            bufs, pend, cnt = {}, {}, {}

            def flush(ri):
                nonlocal flops
                c = cnt[ri]
                if c == 0:
                    return
                op = d["op"][cone[ri]]
                W = bufs[ri][:, :c]
                if self.dense:
                    F = op @ W
                    flops += 2 * n * n * c
                else:
                    L, R = op
                    F = L @ (R.conj().T @ W)
                    flops += 4 * n * L.shape[1] * c
                for col, (tgt, tab) in enumerate(pend[ri]):
                    locals_out[tgt] += scale * F[tab, col]
                self.flush_log.append((tuple(cone[ri]), c))  # block_stats["flushes"] (m2l.py:428)
                cnt[ri] = 0
                pend[ri] = []

            for tgt, far in batch:
                for s, t in far:
                    ri, fl, od = assign[tuple(t)]
                    if ri not in bufs:
                        bufs[ri] = np.empty((n, cap), dtype=acc_dt)
                        pend[ri] = []
                        cnt[ri] = 0
                    bufs[ri][:, cnt[ri]] = mpoles[s][inv_table(fl, od, self.order)]
                    pend[ri].append((tgt, perm_table(fl, od, self.order)))
                    cnt[ri] += 1
                    if cnt[ri] == cap:
                        flush(ri)
            for ri in sorted(bufs):
                flush(ri)
        else:
            cone, assign = d["cone"], d["assign"]
            for tgt, far in batch:
                if not far:
                    continue
                acc = np.zeros(n, dtype=acc_dt)
                for s, t in far:
                    t = tuple(t)
                    if self.sym:
                        ri, fl, od = assign[t]
                        op = d["op"][cone[ri]]
                        u = mpoles[s][inv_table(fl, od, self.order)]
                        if self.dense:
                            out = op @ u
                            flops += 2 * n * n
                        else:
                            out = op[0] @ (op[1].conj().T @ u)
                            flops += 4 * n * op[0].shape[1]
                        acc += out[perm_table(fl, od, self.order)]
                    else:
                        op = d["op"][t]
                        if self.dense:
                            acc += op @ mpoles[s]
                            flops += 2 * n * n
                        else:
                            acc += op[0] @ (op[1].conj().T @ mpoles[s])
                            flops += 4 * n * op[0].shape[1]
                locals_out[tgt] += scale * acc
        self.flops[level] = self.flops.get(level, 0) + flops
        return flops

    # ---- vectorized apply: same math regrouped per transfer vector
    def apply_fast(self, level, tgt, off, src, t, mpoles, locals_out) -> int:
        key = self.level_group[level]
        scale = self.level_scale[level]
        d = self.ops[key]
        n = self.size
        acc_dt = np.result_type(self.dtype, mpoles.dtype)
        tgt = np.asarray(tgt, np.int64)
        off = np.asarray(off, np.int64)
        src = np.asarray(src, np.int64)
        t = np.asarray(t, np.int64).reshape(-1, 3)
        pair_tgt = np.repeat(tgt, np.diff(off))
        code = (t[:, 0] + 3) * 49 + (t[:, 1] + 3) * 7 + (t[:, 2] + 3)
        acc = np.zeros((locals_out.shape[0], n if not self.shared else d["sa"]["u"].shape[1]), dtype=acc_dt)
        flops = 0
        if self.shared:
            sa = d["sa"]
            u, b = sa["u"], sa["b"]
            usrc = np.unique(src)
            wt = np.zeros((mpoles.shape[0], b.shape[1]), dtype=acc_dt)
            wt[usrc] = (b.conj().T @ mpoles[usrc].T).T
            flops += 2 * n * b.shape[1] * len(usrc)
        for c in np.unique(code):
            sel = code == c
            tv = (int(c) // 49 - 3, (int(c) // 7) % 7 - 3, int(c) % 7 - 3)
            ps, pt = src[sel], pair_tgt[sel]
            if self.shared:
                kind, core = d["sa"]["cores"][tv]
                W = wt[ps]
                if kind == "dense":
                    F = W @ core.T
                    flops += 2 * core.shape[0] * core.shape[1] * len(ps)
                else:
                    L, R = core
                    F = (W @ R.conj()) @ L.T
                    flops += 2 * L.shape[1] * (L.shape[0] + R.shape[0]) * len(ps)
                np.add.at(acc, pt, F)
                continue
            if self.sym:
                ri, fl, od = d["assign"][tv]
                op = d["op"][d["cone"][ri]]
                W = mpoles[ps][:, inv_table(fl, od, self.order)]
                tab = perm_table(fl, od, self.order)
            else:
                op = d["op"][tv]
                W = mpoles[ps]
                tab = None
            if self.dense:
                F = W @ op.T
                flops += 2 * n * n * len(ps)
            else:
                F = (W @ op[1].conj()) @ op[0].T
                flops += 4 * n * op[0].shape[1] * len(ps)
            if tab is not None:
                F = F[:, tab]
            np.add.at(acc, pt, F)
        ut = np.unique(pair_tgt)
        if self.shared:
            u = d["sa"]["u"]
            locals_out[ut] += scale * (acc[ut] @ u.T)
            flops += 2 * n * u.shape[1] * int(np.count_nonzero(np.diff(off)))
        else:
            locals_out[ut] += scale * acc[ut]
        self.flops[level] = self.flops.get(level, 0) + flops
        return flops


def rel_l2(a, b) -> float:
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0))
