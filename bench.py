"""M2L throughput benchmark (BASELINE.json metric: M2L cell-pair interactions/s,
fp64, with the fraction of the FP64-tensor roofline).

Workload (BASELINE config 2, the largest single-GPU config the metric is
quoted on): N = 10^7 points uniform in the unit cube (seeded), octree height 7
(reference depth 6, leaf level 6: 262,144 cells, all occupied), Chebyshev
order l = 5, Laplace kernel 1/(4 pi r), symmetry-blocked full-rank M2L
(variant nablk) over every level >= 2: 52,337,880 cell pairs per step.
Multipoles are seeded U[-1,1] (M2L is linear; SURVEY.md §8d allows seeded
multipoles for configs 2/4).

A step = one M2L application of all levels (what the reference times with
engine.py:212-214).  `value` is measured with device-resident expansions
(CUDA events on the launching stream, L2 flushed between steps); `e2e` runs
the same step through the handler with pinned HOST buffers (copies in the
timed region).  `--impl reference` times the CPU port of the reference
(oracle/, kind "port") on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))

METRIC = "M2L cell-pair interactions/sec (fp64)"
FP64_PEAK_FILE = ROOT / "profiles" / "fp64_peak.json"

CONFIGS = {
    # name: (n_points, depth, order, geometry, variant, eps)   (BASELINE.json configs; height H = depth + 1)
    "cfg1": (10_000, 3, 4, "cube", "nablk", 1e-5),
    "cfg2": (10_000_000, 6, 5, "cube", "nablk", 1e-5),
    "cfg2_ia": (10_000_000, 6, 5, "cube", "iablk", 1e-5),
    "cfg3": (8_000_000, 5, 9, "sphere", "nablk", 1e-8),
    "cfg3_sa": (8_000_000, 5, 9, "sphere", "sa", 1e-8),
    "cfg4": (100_000_000, 7, 7, "cube", "nablk", 1e-7),
    "cfg5": (2_000_000, 5, 5, "sphere", "iablk", 1e-4),   # Helmholtz k = 8 pi, complex128, non-directional
}
HELMHOLTZ = {"cfg5": 8 * np.pi}


def fp64_peak():
    if FP64_PEAK_FILE.exists():
        d = json.loads(FP64_PEAK_FILE.read_text())
        return float(d["dmma_tflops"]), "measured (profiles/fp64_peak.json, DMMA m8n8k4 microbenchmark)"
    return 37.1, "fallback (148 SM x 128 flop/clk x 1.965 GHz)"


def bench_points(cfg):
    """Seeded synthetic particles of a config (chunks of 10^7 with per-chunk
    seeds) and its bounding cube (center, half width)."""
    from geometry import cube_points, sphere_points

    n, depth, order, geom, _, _ = CONFIGS[cfg]
    chunk = 10_000_000
    base = 2 if geom == "cube" else (5 if cfg == "cfg5" else 3)  # cfg3 / cfg5 = the golden fixtures' points
    parts = []
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        seed = base + 1000 * (i // chunk)
        parts.append(cube_points(m, seed=seed) if geom == "cube" else sphere_points(m, seed=seed))
    pts = parts[0] if len(parts) == 1 else np.concatenate(parts)
    center, half = ((0.5, 0.5, 0.5), 0.5) if geom == "cube" else ((0.0, 0.0, 0.0), 1.0)
    return pts, center, half


def level_cells(cfg):
    """Occupied cells per level (lexicographic = reference row order), numpy."""
    n, depth, order, geom, _, _ = CONFIGS[cfg]
    pts, center, half = bench_points(cfg)
    side = 1 << depth
    low = np.asarray(center) - half
    width = 2.0 * half
    keys = []
    for i in range(0, len(pts), 10_000_000):
        ijk = np.minimum(((pts[i:i + 10_000_000] - low) / width * side).astype(np.int64), side - 1)
        keys.append(np.unique((ijk[:, 0] << 42) | (ijk[:, 1] << 21) | ijk[:, 2]))
    del pts
    key = np.unique(np.concatenate(keys))
    out = {}
    cur = np.stack([key >> 42, (key >> 21) & 0x1FFFFF, key & 0x1FFFFF], 1)
    out[depth] = cur
    for lvl in range(depth - 1, 1, -1):
        p = cur >> 1
        k = np.unique((p[:, 0] << 42) | (p[:, 1] << 21) | p[:, 2])
        cur = np.stack([k >> 42, (k >> 21) & 0x1FFFFF, k & 0x1FFFFF], 1)
        out[lvl] = cur
    widths = {lvl: width / (1 << lvl) for lvl in out}
    return out, widths


def gpu_level_cells(cfg, device):
    """Same cells from the GPU octree build (paper_1210_7292_b200.octree)."""
    from paper_1210_7292_b200.octree import build_tree_gpu

    n, depth, order, geom, _, _ = CONFIGS[cfg]
    pts, center, half = bench_points(cfg)
    import torch

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = build_tree_gpu(pts, center, half, depth, device=device)
    cells = {l: tree.cells(l) for l in range(2, depth + 1)}
    ms = (time.perf_counter() - t0) * 1e3
    widths = {l: 2.0 * half / (1 << l) for l in cells}
    return cells, widths, ms


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def reference_batches(cells, device):
    """The level batches exactly as the reference's FmmPlan._level_data builds
    them (engine.py:113-119): [(target_row, [(source_row, (t0, t1, t2)), ...]),
    ...] for every target with a non-empty far list, in row order.  The lists
    come from the device classifier (bit-exact with octree.py:148-178); the t
    tuples are shared per distinct vector (the reference allocates one per
    pair; the values are identical)."""
    import ctypes

    from paper_1210_7292_b200 import _native

    lib = _native.load()
    tvec = [(c // 49 - 3, (c // 7) % 7 - 3, c % 7 - 3) for c in range(343)]
    out = {}
    for lvl, c in cells.items():
        c = np.ascontiguousarray(c, dtype=np.int32)
        n = len(c)
        off = np.zeros(n + 1, np.int64)
        tot = ctypes.c_int64()
        _native.check(lib.cfm_classify_count(device, int(lvl), n, c.ctypes.data, off.ctypes.data, ctypes.byref(tot)))
        src = np.empty(tot.value, np.int32)
        t = np.empty((tot.value, 3), np.int8)
        _native.check(lib.cfm_classify_fill(device, int(lvl), n, c.ctypes.data, off.ctypes.data, src.ctypes.data,
                                            t.ctypes.data, None, None))
        code = ((t[:, 0].astype(np.int32) + 3) * 49 + (t[:, 1] + 3) * 7 + (t[:, 2] + 3)).tolist()
        pairs = list(zip(src.tolist(), map(tvec.__getitem__, code)))
        del code
        o = off.tolist()
        out[lvl] = [(i, pairs[o[i]:o[i + 1]]) for i in range(n) if o[i + 1] > o[i]]
        del pairs
    return out


def reference_api_e2e(h, cells, levels, size, dtype, steps, device):
    """M2L of all levels through the reference's own call, as FmmPlan._m2l
    issues it (engine.py:140-157): apply_level(level, batch, mpoles, locals)
    with the Python batch and fresh np.zeros (pageable) level arrays
    (engine.py:98-120).  Times the first call (plans built) and the steady
    state (plans cached under the batch content)."""
    import torch

    t0 = time.perf_counter()
    batches = reference_batches({l: cells[l] for l in levels}, device)
    build_s = time.perf_counter() - t0
    rng = np.random.default_rng(7)
    mp = {}
    for l in levels:
        m = rng.uniform(-1, 1, (len(cells[l]), size))
        mp[l] = m if dtype == np.float64 else m + 1j * rng.uniform(-1, 1, m.shape)
    pairs = sum(len(f) for l in levels for _, f in batches[l])

    def run():
        loc = {l: np.zeros((len(cells[l]), size), dtype=dtype) for l in levels}
        torch.cuda.synchronize()
        tic = time.perf_counter()
        for l in levels:
            h.apply_level(l, batches[l], mp[l], loc[l])
        return time.perf_counter() - tic, loc

    first_s, _ = run()
    times = [run()[0] for _ in range(max(1, steps))]
    s = statistics.median(times)
    bytes_step = sum(3 * len(cells[l]) * size * np.dtype(dtype).itemsize for l in levels)
    return {"value": pairs / s, "unit": "pairs/s", "ms_per_step": s * 1e3, "first_call_ms": first_s * 1e3,
            "pairs_per_step": pairs, "steps": len(times), "batch_build_s_untimed": build_s,
            "h2d_bytes_per_step": bytes_step * 2 // 3, "d2h_bytes_per_step": bytes_step // 3,
            "plan_cache_hit": bool(h.last_plan_cache_hit),
            "path": "B200M2LHandler.apply_level(level, batch, mpoles, locals) per level with the reference's "
                    "Python batch and np.zeros level arrays (pageable), as FmmPlan._m2l calls it; timed region = "
                    "batch->CSR (C), plan lookup, H2D, kernels, D2H; first_call_ms also builds the plans"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


_PORT = {}


def _port_setup(cfg):
    """Oracle port of the reference handler for a config, precomputed once in the
    parent process (forked workers share it)."""
    from oracle import oracle as O

    if cfg in _PORT:
        return _PORT[cfg]
    cells, widths = cached_level_cells(cfg)
    _, depth, order, _, variant, eps = CONFIGS[cfg]
    full = O.full_far_field()
    if cfg in HELMHOLTZ:
        prof, dt, deg = O.helmholtz_profile(HELMHOLTZ[cfg]), np.complex128, None
    else:
        prof, dt, deg = O.laplace_profile, np.float64, -1.0
    orc = O.OracleM2L(variant, prof, dt, order, eps, deg).precompute({l: full for l in cells}, widths)
    rng = np.random.default_rng(7)
    mp = rng.uniform(-1, 1, (len(cells[depth]), order**3))
    if cfg in HELMHOLTZ:
        mp = mp + 1j * rng.uniform(-1, 1, mp.shape)
    _PORT[cfg] = (orc, mp)
    return _PORT[cfg]


def _port_worker(job):
    """One worker of the CPU port: faithful apply (m2l.py:279-452) on a chunk
    of targets; returns (pairs, seconds) of the timed apply only."""
    from threadpoolctl import threadpool_limits

    from oracle import oracle as O

    cfg, rows, blas_threads = job
    cells, _ = cached_level_cells(cfg)
    orc, mp = _port_setup(cfg)
    lvl = CONFIGS[cfg][1]
    tgt, off, src, t = O.far_lists(cells[lvl], lvl, targets=rows)
    loc = np.zeros_like(mp)
    batch = O.csr_to_batch(tgt, off, src, t)
    with threadpool_limits(limits=blas_threads):
        tic = time.perf_counter()
        orc.apply_faithful(lvl, batch, mp, loc)
        dt = time.perf_counter() - tic
    return int(off[-1]), dt


_LEVEL_CACHE = {}


def cached_level_cells(cfg):
    if cfg not in _LEVEL_CACHE:
        _LEVEL_CACHE[cfg] = level_cells(cfg)
    return _LEVEL_CACHE[cfg]


def cpu_port_sample(cfg, n_targets, workers):
    """Time the oracle's faithful port of the reference apply on the first
    n_targets targets of the deepest level (reference row order), split into
    contiguous target chunks over `workers` processes (the reference's own
    parallel mode splits targets over threads, engine.py:145-155)."""
    import multiprocessing as mp_

    _, depth, _, _, _, _ = CONFIGS[cfg]
    cached_level_cells(cfg)  # build once in the parent; forked workers share it
    _port_setup(cfg)
    n_targets = min(n_targets, len(_LEVEL_CACHE[cfg][0][depth]))
    rows = np.arange(n_targets)
    chunks = [c for c in np.array_split(rows, workers) if len(c)]
    if workers == 1:
        res = [_port_worker((cfg, chunks[0], 1))]
    else:
        ctx = mp_.get_context("fork")
        with ctx.Pool(len(chunks)) as pool:
            res = pool.map(_port_worker, [(cfg, c, 1) for c in chunks])
    pairs = sum(r[0] for r in res)
    dt = max(r[1] for r in res)
    return pairs / dt, pairs, dt


def workload_name(cfg, variant=None):
    """The workload string both arms print in config.workload."""
    n, depth, order, geom, v0, eps = CONFIGS[cfg]
    return (f"{cfg}: N={n:.0e} {geom}, height {depth + 1} (levels 2-{depth}), l={order}, "
            f"{'Helmholtz k=8pi complex128' if cfg in HELMHOLTZ else 'Laplace'}, variant {variant or v0}, eps={eps:g}")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    threads = os.cpu_count() or 1
    n_deep = len(cached_level_cells(cfg)[0][CONFIGS[cfg][1]])
    n_t = min(args.cpu_targets * threads, n_deep)
    vals = []
    for i in range(args.warmup + args.steps):
        v, pairs, dt = cpu_port_sample(cfg, n_t, threads)
        if i >= args.warmup:
            vals.append((v, pairs, dt))
    v = statistics.median(x[0] for x in vals)
    pairs = vals[0][1]
    lvl = CONFIGS[cfg][1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(x[2] for x in vals),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128" if cfg in HELMHOLTZ else "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg, args.variant), "sample": f"first {n_t} targets of level {lvl}"},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{pairs} pairs: first {n_t} level-{lvl} targets (full far lists), faithful "
                                   f"port of m2l.py _apply_blocked (oracle/oracle.py), {threads} processes x 1 "
                                   f"BLAS thread, time = slowest worker"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class Ctx:
    """Per-process run context: rank layout, device, process group, L2 flush buffer."""

    def __init__(self, args):
        import torch

        self.ws, self.rank, self.local = dist_env()
        self.shared_gpu = os.environ.get("CFM_BENCH_SHARE_GPU") == "1"
        self.dist = None
        if self.ws > 1:
            import torch.distributed as dist

            # CFM_BENCH_SHARE_GPU=1: every rank on cuda:0 with a gloo group (a
            # functional multi-rank run on a 1-GPU box; not a scaling number)
            dist.init_process_group("gloo" if self.shared_gpu else "nccl")
            self.dist = dist
        self.device_index = 0 if self.shared_gpu else self.local
        torch.cuda.set_device(self.device_index)
        self.dev = torch.device("cuda", self.device_index)
        self.flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=self.dev)  # 256 MB > 126 MB L2

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def reduce(self, x, op="sum", dtype=None):
        if self.dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=dtype or (torch.float64 if isinstance(x, float) else torch.int64), device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return t.item()


def _kernel_of(cfg):
    from paper_1210_7292_b200 import helmholtz_kernel, laplace_kernel

    return helmholtz_kernel(HELMHOLTZ[cfg]) if cfg in HELMHOLTZ else laplace_kernel()


def measure(ctx, cfg, variant=None, steps=10, warmup=3, e2e_steps=None, want_handler=False):
    """One configuration: GPU tree -> precompute -> device lists + plans ->
    `steps` timed M2L steps (L2 flushed before each, CUDA events on the
    launching stream, max over ranks) -> the same step end to end from pinned
    host buffers.  N > 1: shard-local arrays (owned rows + halo), the halo
    exchanged every step (distributed.ShardedM2L)."""
    import torch

    from paper_1210_7292_b200 import ChebyshevGrid, full_far_field_vectors, make_handler

    n, depth, order, geom, v0, eps = CONFIGS[cfg]
    variant = variant or v0
    size = order**3
    cplx = cfg in HELMHOLTZ
    dt = torch.complex128 if cplx else torch.float64
    cells, widths, tree_ms = gpu_level_cells(cfg, ctx.device_index)
    levels = sorted(cells)
    full = full_far_field_vectors()
    budget = 4_000_000_000 if variant in ("sa", "sarcmp") else 2_000_000_000

    def new_handler():
        hh = make_handler(variant, _kernel_of(cfg), ChebyshevGrid(order), eps, device=ctx.device_index,
                          budget_bytes=budget)
        hh.precompute({l: full for l in levels}, widths)
        return hh

    t0 = time.perf_counter()
    h = new_handler()
    pre_s = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh, stats = None, {}
    if ctx.ws == 1:
        for l in levels:
            stats[l] = h.plan_level_cells(l, cells[l].astype(np.int32))
        pairs_local = sum(st["pairs"] for st in stats.values())
    else:
        from paper_1210_7292_b200.distributed import ShardedM2L

        sh = ShardedM2L(ctx.dist, h, new_handler(), {l: cells[l] for l in levels}, device=ctx.dev,
                        complex_data=cplx)
        pairs_local = sh.pairs
    torch.cuda.synchronize()
    plan_s = time.perf_counter() - t0
    pairs_total = int(ctx.reduce(pairs_local))

    # seeded U[-1,1] multipoles of the whole level (identical for every N); a
    # rank keeps its owned rows, the halo arrives through the exchange
    gen = torch.Generator(device=ctx.dev).manual_seed(11)
    arrays = {}
    for l in levels:
        glob = torch.rand((len(cells[l]), size), dtype=dt, device=ctx.dev, generator=gen) * 2 - (1 + 1j if cplx else 1)
        if sh is None:
            arrays[l] = (glob, torch.zeros_like(glob))
        else:
            sl = sh.levels[l]
            mp = torch.zeros((sl.n_local, size), dtype=dt, device=ctx.dev)
            mp[: sl.n_owned] = glob[torch.as_tensor(sl.owned, device=ctx.dev)]
            arrays[l] = (mp, torch.zeros_like(mp))
        del glob
    torch.cuda.empty_cache()
    flops = [0]

    def step():
        if sh is None:
            flops[0] = h.apply_levels(arrays)
            return h.last_apply_stats()[1]
        flops[0] = sh.step(arrays)
        return sh.launches()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ctx.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    launches = 0
    with ClockSampler(ctx.device_index) as clk:
        for i in range(steps):
            ctx.flush.fill_(float(i))
            torch.cuda.synchronize()
            ev[i][0].record()
            launches += step()
            ev[i][1].record()
            torch.cuda.synchronize()
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]
    total_ms = ctx.reduce(float(sum(step_ms)), "max")
    med_ms = ctx.reduce(float(statistics.median(step_ms)), "max")
    real_flops = int(ctx.reduce(int(flops[0]))) * (4 if cplx else 1)

    # end to end: the same step from pinned host buffers (H2D multipoles +
    # locals, kernels, D2H locals in the timed region).  N = 1: through the
    # handler's host-buffer pipeline; N > 1: each rank moves its owned rows.
    e2e_steps = e2e_steps or steps
    if sh is None:
        h_mp = {l: torch.empty(arrays[l][0].shape, dtype=dt, pin_memory=True) for l in levels}
        h_loc = {l: torch.zeros(arrays[l][0].shape, dtype=dt, pin_memory=True) for l in levels}
        for l in levels:
            h_mp[l].copy_(arrays[l][0].cpu())
        np_arr = {l: (h_mp[l].numpy(), h_loc[l].numpy()) for l in levels}

        def e2e_step():
            h.apply_levels(np_arr)

        h2d = sum(2 * a[0].numel() * a[0].element_size() for a in arrays.values())
        d2h = sum(a[0].numel() * a[0].element_size() for a in arrays.values())
    else:
        own = {l: sh.levels[l].n_owned for l in levels}
        h_mp = {l: torch.empty((own[l], size), dtype=dt, pin_memory=True) for l in levels}
        h_loc = {l: torch.zeros((own[l], size), dtype=dt, pin_memory=True) for l in levels}
        for l in levels:
            h_mp[l].copy_(arrays[l][0][: own[l]].cpu())

        def e2e_step():
            for l in levels:
                arrays[l][0][: own[l]].copy_(h_mp[l], non_blocking=True)
                arrays[l][1][: own[l]].copy_(h_loc[l], non_blocking=True)
            sh.step(arrays)
            for l in levels:
                h_loc[l].copy_(arrays[l][1][: own[l]], non_blocking=True)
            torch.cuda.synchronize()

        h2d = int(ctx.reduce(sum(2 * own[l] * size * (16 if cplx else 8) for l in levels)))
        d2h = int(ctx.reduce(sum(own[l] * size * (16 if cplx else 8) for l in levels)))
    e2e_step()
    torch.cuda.synchronize()
    ctx.barrier()
    tic = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = ctx.reduce((time.perf_counter() - tic) / e2e_steps, "max")

    peak, peak_src = fp64_peak()
    achieved = real_flops / ctx.ws / (med_ms * 1e-3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            tr = json.loads(prof.read_text()).get(cfg, {}).get(variant)
            traffic = tr["dram_bytes"] if isinstance(tr, dict) else tr
        except Exception:
            traffic = None
    rec = {
        "config": cfg, "variant": variant, "workload": workload_name(cfg, variant),
        "value": pairs_total * steps / (total_ms * 1e-3), "unit": "pairs/s", "ms_per_step": total_ms / steps,
        "steps": steps, "warmup": warmup, "pairs_per_step": pairs_total,
        "dtype": "c128" if cplx else "f64",
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": f"M2L step over levels {levels[0]}-{levels[-1]} "
                               f"({pairs_total} pairs x {real_flops / max(pairs_total, 1):.0f} flop avg, "
                               f"reference accounting{' x4 complex' if cplx else ''})",
                     "peak_source": peak_src, "dominant_ms": med_ms},
        "e2e": {"value": pairs_total / e2e_s, "unit": "pairs/s", "ms_per_step": e2e_s * 1e3,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "path": ("B200M2LHandler.apply_levels with pinned host numpy buffers (C ABI; H2D multipoles + "
                         "locals, kernels, D2H locals in the timed region)") if sh is None else
                        ("per rank: H2D of its owned multipole + local rows, halo exchange + apply "
                         "(ShardedM2L.step), D2H of its owned locals")},
        "gpu_launches": launches, "clocks": clk.summary(),
        "precompute_s": pre_s, "plan_s": plan_s, "tree_build_ms": tree_ms,
        "levels": {str(l): int(ctx.reduce(stats[l]["pairs"] if sh is None else sh.levels[l].pairs)) for l in levels},
        "l2": "flushed between steps (256 MB write)", "multipoles": "seeded U[-1,1]",
    }
    if sh is None:
        slots = sum(st["slots"] for st in stats.values())
        rec["tile_fill"] = pairs_local / max(slots, 1)
        rec["plan_modes"] = {str(l): stats[l].get("mode") for l in levels}
    else:
        rec["shard"] = {str(l): {"owned": sh.levels[l].n_owned, "halo": len(sh.levels[l].halo),
                                 "interior_pairs": sh.levels[l].interior_pairs,
                                 "boundary_pairs": sh.levels[l].boundary_pairs} for l in levels}
        rec["local_array_bytes"] = int(sum(2 * a[0].numel() * a[0].element_size() for a in arrays.values()))
    out = (rec, h, cells, levels) if want_handler else (rec,)
    del arrays, sh
    torch.cuda.empty_cache()
    return out


def classifier_record(ctx, cells, level):
    """Row a1 on its own: device far-list classification of one level
    (HBM-bound integer work), device outputs, L2 flushed, CUDA events."""
    import ctypes

    import torch

    from paper_1210_7292_b200 import _native

    lib = _native.load()
    dev = ctx.dev
    deep_cells = torch.from_numpy(cells.astype(np.int32)).to(dev)
    ncell = len(cells)
    offs = torch.empty(ncell + 1, dtype=torch.int64, device=dev)
    tot = ctypes.c_int64()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _native.check(lib.cfm_classify_count_device(ctx.device_index, level, ncell, deep_cells.data_ptr(),
                                                offs.data_ptr(), ctypes.byref(tot), stream))
    src_d = torch.empty(tot.value, dtype=torch.int32, device=dev)
    code_d = torch.empty(tot.value, dtype=torch.int16, device=dev)
    ms_c = []
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.flush.fill_(float(i))
        e0.record()
        _native.check(lib.cfm_classify_fill_device(ctx.device_index, level, ncell, deep_cells.data_ptr(),
                                                   offs.data_ptr(), src_d.data_ptr(), code_d.data_ptr(), stream))
        e1.record()
        torch.cuda.synchronize()
        ms_c.append(e0.elapsed_time(e1))
    cl_ms = min(ms_c[1:])
    # algorithmic bytes of the fill pass: occupancy grid memset + scatter, cells
    # read, offsets read, per pair 4 B source row + 2 B t-code written
    S3 = (1 << level) ** 3
    cl_bytes = S3 * 4 + ncell * (4 + 12 + 12 + 8) + tot.value * 6
    peak_hbm = 6551.4
    try:
        peak_hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    return {"level": level, "pairs": tot.value, "fill_ms": cl_ms, "pairs_per_s": tot.value / (cl_ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": cl_bytes / (cl_ms * 1e-3) / 1e9, "peak": peak_hbm,
                         "unit": "GB/s", "frac": cl_bytes / (cl_ms * 1e-3) / 1e9 / peak_hbm},
            "note": "cfm_classify_fill_device (grid build + 216-candidate enumeration + canonical codes), "
                    "device outputs, L2 flushed"}


SUB_DEFAULT = {1: "cfg2_ia,cfg3,cfg3_sa,cfg5,cfg4", "multi": "cfg4"}


def run_b200(args):
    import torch

    ctx = Ctx(args)
    cfg = args.config
    rec, h, cells, levels = measure(ctx, cfg, args.variant, args.steps, args.warmup, want_handler=True)
    variant = rec["variant"]
    size = CONFIGS[cfg][2] ** 3

    extras = {}
    if ctx.rank == 0:
        extras["classifier"] = classifier_record(ctx, cells[levels[-1]], levels[-1])
    # the reference's own call path (apply_level with the Python batch and
    # pageable np.zeros level arrays, engine.py:140-157), single GPU
    if ctx.ws == 1 and not args.no_reference_api:
        extras["e2e_reference_api"] = reference_api_e2e(
            h, cells, levels, size, np.complex128 if cfg in HELMHOLTZ else np.float64, 3, ctx.device_index)
    del h
    torch.cuda.empty_cache()

    subs = {}
    sub_list = args.subconfigs if args.subconfigs is not None else SUB_DEFAULT[1 if ctx.ws == 1 else "multi"]
    for name in [s for s in sub_list.split(",") if s]:
        sub_steps = min(args.steps, 3 if name == "cfg4" else 10)
        r = measure(ctx, name, None, sub_steps, max(3, args.warmup if name != "cfg4" else 3), e2e_steps=
                    min(sub_steps, 3))[0]
        subs[name] = r

    cpu = None
    if ctx.rank == 0 and ctx.ws == 1 and not args.no_cpu:
        v, pairs, dt_s = cpu_port_sample(cfg, args.cpu_targets, 1)
        deep = CONFIGS[cfg][1]
        cpu = {"value": v, "unit": "pairs/s", "cores": 1, "kind": "port",
               "sample": f"{pairs} pairs ({args.cpu_targets} level-{deep} targets, full far lists), faithful port "
                         f"of m2l.py _apply_blocked, 1 thread, {dt_s:.1f} s"}

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": rec["value"], "unit": "pairs/s", "n_gpus": ctx.ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": rec["dtype"], "data": "synthetic",
            "config": {"workload": rec["workload"], "pairs_per_step": rec["pairs_per_step"],
                       "precompute_s": rec["precompute_s"], "plan_s": rec["plan_s"],
                       "tree_build_ms": rec["tree_build_ms"], "levels": rec["levels"],
                       "tile_fill": rec.get("tile_fill"), "plan_modes": rec.get("plan_modes"),
                       "parallelism": (f"{ctx.ws} ranks: targets sharded by Morton range, shard-local arrays, "
                                       f"{'gloo (shared GPU)' if ctx.shared_gpu else 'NCCL'} halo all_to_all per "
                                       f"level") if ctx.ws > 1 else "1 GPU",
                       "l2": rec["l2"], "multipoles": rec["multipoles"]},
            "roofline": rec["roofline"], "e2e": rec["e2e"], "gpu_launches": rec["gpu_launches"],
            "clocks": rec["clocks"],
        }
        if "shard" in rec:
            line["config"]["shard"] = rec["shard"]
            line["config"]["local_array_bytes_rank0"] = rec["local_array_bytes"]
        if cpu:
            line["cpu_baseline"] = cpu
        line.update(extras)
        if subs:
            line["configs"] = subs
        print(json.dumps(line), flush=True)
    if ctx.dist is not None:
        ctx.dist.destroy_process_group()


def respawn(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-launch this
    script under torch.distributed.run with N ranks (127.0.0.1 rendezvous);
    rank 0 prints the line."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--variant", default=None)
    ap.add_argument("--cpu-targets", type=int, default=8192,
                    help="CPU-port sample size in deepest-level targets (per process for --impl reference)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-reference-api", action="store_true", help="skip the apply_level(batch) e2e measurement")
    ap.add_argument("--subconfigs", default=None,
                    help="comma list of extra configs measured after the main line (default: cfg2_ia,cfg3,"
                         "cfg3_sa,cfg5,cfg4 at N=1, cfg4 at N>1; '' for none)")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "0"))
    if ws == 0 and args.gpus > 1:
        sys.exit(respawn(args))
    if ws and ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch N ranks for --gpus N")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
