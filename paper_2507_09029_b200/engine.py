"""Owner-subset sync behind the reference's `aggregate` (engine.py:60-79).

    aggregate(grads, assignment) -> AggregatedGradient(gbar, divisor)

keeps the reference signature, argument meaning and errors: `grads` is a list
of N flat gradients (CUDA tensors -- or numpy arrays, which are copied to the
device and the mean copied back), `gbar` is a fresh buffer, `divisor` is the
assignment's float64 divisor, ProtocolError on a wrong count or an uncovered
leak.  Underneath, one launch of libsdp's k_owner_sync reads each element from
its owners only, in ascending worker order, and divides by the owner count.

`owner_sync` is the B200-native form of the same step: the
mean is written back into every owner's replica (and an optional bf16
training copy) -- what an all-reduce over the owner subset leaves behind --
optionally fused with the SGD-Nesterov update (optim.py:78-84).
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._device import device, ptr, sdp_dtype, stream_ptr, upload_struct
from .errors import ConfigError, NumericalError, ProtocolError, UsageError
from .storage import dispatch_order, leader_cta

TILE = 2048              # elements per sync tile (8 KB of fp32 per replica); measured
                         # best on B200 for 11M..268M buffers (tools/sync_probe.py)
TILE_DTYPE = np.dtype([("owner_bits", "<u8"), ("tile_index", "<u4"), ("len_flags", "<u4")])
CTAS_PER_SM = 4          # 64 regs x 256 threads -> 4 resident CTAs per SM


@dataclass
class AggregatedGradient:
    gbar: object
    divisor: object


def _sm_count() -> int:
    n = C.c_int(0)
    N.call("sdp_device_sm_count", C.byref(n))
    return int(n.value)


def auto_tile(d: int, sms: int, avg_owners: float = 4.0) -> int:
    """2048-element tiles; 1024 when that leaves fewer than two full waves of
    resident CTAs (small buffers are latency-bound: more, shorter CTAs); 4096
    for large buffers with ~2 owners per element, where a 2048-tile CTA moves
    too few bytes (same-box A/B, 256 MiB P=2: 0.977 vs 0.893-0.95)."""
    if -(-d // TILE) < 2 * sms * CTAS_PER_SM:
        return TILE // 2
    if avg_owners < 2.5 and d * avg_owners * 10 >= BIG_TRAFFIC / 2:
        return 2 * TILE
    return TILE


def gpu_of_worker(n_workers: int, world: int) -> np.ndarray:
    """Contiguous placement of N logical workers on `world` GPUs: w -> w*G//N."""
    return np.array([w * world // n_workers for w in range(n_workers)], dtype=np.int64)


def tile_leaders(tiles: np.ndarray, gpu_of: np.ndarray, world: int) -> np.ndarray:
    """Rank that reduces each tile: the owner GPUs of the tile take turns
    (tile t -> the (t mod k)-th of its k owner GPUs), so one of the reads is
    always local and every owner GPU leads an equal share; uncovered tiles are
    dealt round-robin."""
    n = len(tiles)
    out = np.empty(n, dtype=np.int64)
    bits = tiles["owner_bits"].astype(np.uint64)
    # owner-GPU set per tile as a bitmask over ranks
    gmask = np.zeros(n, dtype=np.int64)
    for w, g in enumerate(gpu_of):
        on = ((bits >> np.uint64(w)) & np.uint64(1)).astype(bool)
        gmask[on] |= 1 << int(g)
    for m in np.unique(gmask):
        sel = np.nonzero(gmask == m)[0]
        gpus = [g for g in range(world) if m >> g & 1]
        out[sel] = [gpus[t % len(gpus)] for t in sel] if gpus else sel % world
    return out


BIG_TRAFFIC = 1.5e9  # bytes per launch above which one CTA per tile wins
def direct_wins(d: int, owned_frac: float, mixed_frac: float = 0.0) -> tuple[bool, bool]:
    """(small, mixed): whether the one-round-trip kernel (SDP_SYNC_DIRECT,
    which also reads the non-owned replica bytes) beats the tiled one for
    every launch of the plan, and whether the streaming form does for its
    plain `aggregate` launches.  Same-box A/Bs:
    * small buffers (profiles/r2_small_buffers_direct_ab.jsonl, graph-
      amortised cold): up to 1 MiB at any P (10-20 %), up to 2 MiB at
      P = N/2, up to 16 MiB when every worker owns (nearly) everything;
    * width-wise (flat-layout) plans with >= 30 % mixed tiles, in the
      streaming form (SDP_SYNC_STREAM, owner-filtered lines, prefetched
      masks; profiles/r2_direct_ab.jsonl): C3 73.6 -> 57.4 us, the c=512
      neuron sweep 196 -> 172 us, GPT-2 channel units 796 -> 679 us -- in
      the mean-only form; with the per-owner write-back it lost (C3 128 ->
      147 us), so those launches stay tiled, as do the block plans."""
    small = d <= 1 << 18 or (d <= 1 << 19 and owned_frac >= 0.5) or (d <= 1 << 22 and owned_frac >= 0.99)
    return small, (not small) and mixed_frac >= 0.3


def plan_grid(n_tiles: int, sms: int, resident: bool, traffic: float = 0.0) -> int:
    """Grid of the sync launch (tools/grid_ab.py, same-box A/B, fraction of the
    measured copy peak):

        workload (P=4)     traffic   one tile/CTA   capped grid (8 waves)
        ResNet-18          0.64 GB      0.898           0.947
        sweep 256 MiB      2.7 GB       1.004           0.949
        GPT-2 124M         6.5 GB       0.976           0.941

    so one CTA per tile above BIG_TRAFFIC, a grid capped at 8 waves of
    resident CTAs below it, and a persistent grid for co-residency (the
    cross-rank barrier)."""
    if resident:
        return max(1, min(n_tiles, sms * CTAS_PER_SM))
    if traffic >= BIG_TRAFFIC:
        return max(1, min(n_tiles, 2**31 - 1))
    return max(1, min(n_tiles, sms * CTAS_PER_SM * 8))


def cta_major(tiles: np.ndarray, grid: int, tiles_per_cta: int) -> np.ndarray:
    """Descriptor table where CTA b's tiles (b, b+grid, b+2*grid, ...) are
    contiguous, so one bulk copy stages them; holes have length 0."""
    table = np.zeros(grid * tiles_per_cta, dtype=TILE_DTYPE)
    for k in range(tiles_per_cta):
        sel = tiles[k * grid:(k + 1) * grid]
        table[np.arange(len(sel)) * tiles_per_cta + k] = sel
    return table


class SyncPlan:
    """Tile plan of one assignment: which tiles have a single owner set, which
    rank leads each tile, and the CTA-major descriptor table k_owner_sync
    stages into shared memory.

    world/rank: multi-GPU split (tiles led by `rank`); gpu_of_worker maps the
    logical workers to ranks (contiguous placement, SURVEY.md §7 hard part 6).
    """

    def __init__(self, assignment, world: int = 1, rank: int = 0, tile: int | None = None,
                 resident: bool = False, max_grid: int | None = None,
                 force_grid: int | None = None, tile_lo: int | None = None,
                 tile_hi: int | None = None, owner_mask: torch.Tensor | None = None,
                 order: str = "mixed_first", direct: bool | None = None,
                 stream: bool | None = None):
        """direct: use the small-buffer kernel (SDP_SYNC_DIRECT) -- by default
        where direct_wins() says so, for world-1, non-resident, unchunked
        plans with N <= 8 workers."""
        self.assignment = assignment
        dev = assignment.device
        d = assignment.topology.total
        owned_total = assignment.owned_total()
        if tile is None:
            tile = auto_tile(d, _sm_count(), owned_total / max(1, d))
        self.tile = tile
        self.world, self.rank = world, rank
        # a permuted layout (layout.SyncLayout) brings its own per-element owner mask
        self.owner_mask = assignment.owner_mask if owner_mask is None else owner_mask
        n_tiles = (d + tile - 1) // tile
        raw = torch.empty(max(1, n_tiles) * TILE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        owned = torch.zeros(max(1, n_tiles), dtype=torch.int64, device=dev)
        N.call("sdp_plan_tiles", ptr(self.owner_mask), assignment.mask_bytes, d, tile,
               ptr(raw), ptr(owned), stream_ptr(dev))
        tiles = raw.cpu().numpy().view(TILE_DTYPE)[:n_tiles].copy()
        # exact sum of |O_j| per tile (popcounts reduced in k_plan_tiles)
        self.tile_owned = owned.cpu().numpy()[:n_tiles]
        self.all_tiles = tiles
        self.n_uniform = int(((tiles["len_flags"] & N.TILE_UNIFORM) != 0).sum())
        nw = assignment.n_workers
        self.gpu_of_worker = gpu_of_worker(nw, world)
        self.leaders = (tile_leaders(tiles, self.gpu_of_worker, world) if world > 1
                        else np.zeros(len(tiles), dtype=np.int64))
        self.order = order
        mine = tiles[self.leaders == rank] if world > 1 else tiles
        if tile_lo is not None or tile_hi is not None:  # a chunk of the vector (pipelined host path)
            lo, hi = tile_lo or 0, n_tiles if tile_hi is None else tile_hi
            mine = mine[(mine["tile_index"] >= lo) & (mine["tile_index"] < hi)]
        # dispatch order of the tiles (CTA b takes b, b + grid, ...): the
        # lane-per-element mixed tiles are the slow ones, so they go out in the
        # first wave instead of forming the tail (same-box A/B, tools/c3_ab.py:
        # C3 sync layout 63.6 -> 60.1 us, C2 unchanged)
        mine = mine[dispatch_order(mine, order)]
        self.n_tiles = len(mine)
        # every CTA must be co-resident for the cross-rank flag barrier
        self.grid = plan_grid(self.n_tiles, _sm_count(), resident or world > 1,
                              traffic=10.0 * owned_total / world)
        if max_grid:
            self.grid = max(1, min(self.grid, max_grid))
        self.tiles_per_cta = max(1, -(-self.n_tiles // self.grid))
        if force_grid:
            self.grid = int(force_grid)  # all ranks launch the same grid (pairwise barrier)
            self.tiles_per_cta = max(1, -(-self.n_tiles // self.grid))
        self.mine = mine
        self.table = upload_struct(cta_major(mine, self.grid, self.tiles_per_cta), dev)
        mixed_frac = 1.0 - self.n_uniform / max(1, len(tiles))
        eligible = world == 1 and not resident and tile_lo is None and tile_hi is None \
            and nw <= 8 and assignment.mask_bytes == 1
        small, mixed = direct_wins(d, owned_total / max(1, d * nw), mixed_frac)
        # direct / stream given: that kernel for every launch (tests, A/B);
        # by default the small-buffer kernel for every launch of a small plan
        # and the streaming one for the mean-only launches of a mixed plan
        self.direct = eligible and (small if direct is None else bool(direct))
        self.stream = eligible and bool(stream)
        self.stream_mean = eligible and mixed and direct is None and stream is None
        self.owned_elems = int(self.tile_owned[mine["tile_index"].astype(np.int64)].sum())

    def leader_cta(self) -> np.ndarray:
        """CTA index that reduces each tile on its leader rank (same grid on
        every rank); the local-update phase of a compact trainer runs a tile's
        optimizer step in that CTA index after the pairwise exit barrier."""
        return leader_cta(self.all_tiles, self.leaders, self.world, self.grid, self.order)

    def worker_ranges(self, w: int) -> list[tuple[int, int]]:
        """Element ranges (start, length) of worker w's replica the kernel reads:
        the tiles whose owner union contains w, merged into maximal runs."""
        if not hasattr(self, "_ranges"):
            self._ranges = {}
        if w not in self._ranges:
            t = self.all_tiles
            on = ((t["owner_bits"] >> np.uint64(w)) & np.uint64(1)).astype(bool)
            idx = t["tile_index"][on].astype(np.int64)
            lens = (t["len_flags"][on] & N.TILE_LEN_MASK).astype(np.int64)
            out = []
            for i, ln in zip(idx, lens):
                s = int(i) * self.tile
                if out and out[-1][0] + out[-1][1] == s:
                    out[-1][1] += int(ln)
                else:
                    out.append([s, int(ln)])
            self._ranges[w] = [tuple(x) for x in out]
        return self._ranges[w]

    def args(self, dtype: int) -> N.SyncArgs:
        a = self.assignment
        s = N.SyncArgs()
        s.dtype = dtype
        s.n_workers = a.n_workers
        s.mask_bytes = a.mask_bytes
        s.tile = self.tile
        s.total = a.topology.total
        s.owner_mask = self.owner_mask.data_ptr()
        s.tiles = self.table.data_ptr()
        s.n_tiles = self.grid * self.tiles_per_cta
        s.tiles_per_cta = self.tiles_per_cta
        s.grid = self.grid
        s.rank = self.rank
        s.world = 1
        return s


def _as_replica_list(grads, n: int, d: int):
    if torch.is_tensor(grads) and grads.dim() == 2:
        if grads.shape != (n, d):
            raise ProtocolError(f"aggregate received {grads.shape[0]} gradients for {n} workers")
        return [grads[i] for i in range(n)]
    if len(grads) != n:
        raise ProtocolError(f"aggregate received {len(grads)} gradients for {n} workers")
    return list(grads)


def _aligned(t: torch.Tensor) -> bool:
    return t.is_contiguous() and t.data_ptr() % 16 == 0


def _device_readable(t: torch.Tensor) -> bool:
    """Host tensor in page-locked memory mapped at the same address on the
    device (libsdp sdp_host_ptr_on_device)."""
    if t.device.type != "cpu" or t.numel() == 0:
        return False
    ok = C.c_int(0)
    N.call("sdp_host_ptr_on_device", C.c_void_p(t.data_ptr()), C.byref(ok))
    return bool(ok.value)


class PreparedSync:
    """A fully bound k_owner_sync launch (args built once): the steady-state
    form used by training loops and the benchmark -- one ctypes call per step."""

    def __init__(self, replicas, assignment, **kw):
        self._keep = (replicas, kw)
        self.args = _bind(replicas, assignment, **kw)
        self.status = kw.get("status")
        self.device = assignment.device
        self._fn = N.lib().sdp_owner_sync
        self._ref = C.byref(self.args)

    def launch(self, stream=None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self._fn(self._ref, C.c_void_p(s.cuda_stream))
        if rc:
            N.check(rc, "sdp_owner_sync")


def owner_sync(replicas, assignment, **kw) -> torch.Tensor | None:
    """One launch of k_owner_sync over co-resident replicas (one GPU, N logical
    workers).  Returns the device status word tensor (not synchronised).

    out / out_bf16: the mean (dtype / bf16); writeback: mean into every owner's
    replica; shadows_bf16: per-worker bf16 training copies;
    nesterov: {"theta": t, "velocity": v, "lr": float, "momentum": float,
               "theta_bf16": optional} applies optim.py:81-84 in the epilogue.
    """
    if kw.get("status") is None and (kw.get("check_uncovered") or kw.get("check_finite")):
        kw["status"] = torch.zeros(1, dtype=torch.int32, device=assignment.device)
    a = _bind(replicas, assignment, **kw)
    N.check(N.lib().sdp_owner_sync(C.byref(a), stream_ptr(assignment.device)), "sdp_owner_sync")
    return kw.get("status")


def _bind(replicas, assignment, *, out: torch.Tensor | None = None,
          out_bf16: torch.Tensor | None = None, writeback: bool = True,
          shadows_bf16=None, check_uncovered: bool = False, check_finite: bool = False,
          nesterov: dict | None = None, adam: dict | None = None,
          status: torch.Tensor | None = None, plan: SyncPlan | None = None,
          zero_copy: bool = False, compact=None, local_update: dict | None = None) -> N.SyncArgs:
    """zero_copy: replicas (and `out`) may be pinned host tensors, which the
    kernel reads (writes) over PCIe through their unified addresses.
    compact: a storage.CompactLayout of `plan` -- replica / shadow w holds only
    the tiles w owns (length compact.length(w)).
    local_update: {"states": device sdp_worker_state array, "updates": device
    sdp_update_desc table, "per_cta": int} -- the Nesterov / Adam of `nesterov`
    / `adam` (their scalars) applied to each worker's own state after the sync
    (SDP_SYNC_LOCAL_UPDATE) instead of to one flat theta."""
    n, d = assignment.n_workers, assignment.topology.total
    reps = _as_replica_list(replicas, n, d) if compact is None else list(replicas)
    if compact is not None and len(reps) != n:
        raise ProtocolError(f"owner sync received {len(reps)} replicas for {n} workers")
    dt = reps[0].dtype
    dev = assignment.device

    def placed(t):
        return t.device == dev or (zero_copy and _device_readable(t))

    for w, r in enumerate(reps):
        size = d if compact is None else compact.length(w)
        if r.dtype != dt or r.numel() != size or not placed(r) or not _aligned(r):
            raise UsageError("replicas must be contiguous, 16-byte aligned, same dtype, "
                             f"[{size}] on {dev}" + (" or pinned host memory" if zero_copy else ""))
    if out is not None and not placed(out):
        raise UsageError(f"out must be on {dev}" + (" or in pinned host memory" if zero_copy else ""))
    plan = plan or assignment.sync_plan()
    a = plan.args(sdp_dtype(dt))
    flags = 0
    # small buffers: the one-round-trip kernel (its extra reads of non-owned
    # replica bytes would cross PCIe on the zero-copy path: device only)
    # small buffers: the one-round-trip kernel; a mixed-tile (width-wise flat)
    # plan in the plain `aggregate` form (mean out only -- its per-owner
    # write-back / optimizer epilogue measured slower there): the streaming one
    pure_mean = not writeback and nesterov is None and adam is None
    if compact is None and local_update is None and not zero_copy:
        if plan.stream or (plan.stream_mean and pure_mean):
            flags |= N.SYNC_DIRECT | N.SYNC_STREAM
        elif plan.direct:
            flags |= N.SYNC_DIRECT
    if writeback:
        flags |= N.SYNC_WRITEBACK
    if check_uncovered:
        flags |= N.SYNC_CHECK_UNCOVERED
    if check_finite:
        flags |= N.SYNC_CHECK_FINITE
    for w, r in enumerate(reps):
        a.replicas[w] = r.data_ptr()
    if shadows_bf16 is not None:
        for w, sh in enumerate(shadows_bf16):
            a.shadow_bf16[w] = None if sh is None else sh.data_ptr()
    a.out = None if out is None else out.data_ptr()
    a.out_bf16 = None if out_bf16 is None else out_bf16.data_ptr()
    if nesterov is not None and adam is not None:
        raise UsageError("choose one fused optimizer")
    opt = nesterov if nesterov is not None else adam
    if opt is not None and local_update is None:
        keys = ("theta", "velocity") if nesterov is not None else ("theta", "m", "v")
        for k in keys:
            t = opt.get(k)
            if not torch.is_tensor(t) or t.dtype != dt or t.numel() != d or t.device != dev or not _aligned(t):
                raise UsageError(f"fused optimizer buffer {k!r} must be a contiguous, 16-byte aligned [{d}] "
                                 f"{dt} tensor on {dev} (the replicas' dtype)")
        tb = opt.get("theta_bf16")
        if tb is not None and (tb.dtype != torch.bfloat16 or tb.numel() != d or tb.device != dev
                               or not tb.is_contiguous()):
            raise UsageError(f"theta_bf16 must be a contiguous [{d}] bfloat16 tensor on {dev}")
    for nm, t, want in (("out", out, dt), ("out_bf16", out_bf16, torch.bfloat16)):
        if t is not None and (t.dtype != want or t.numel() != d or not t.is_contiguous()):
            raise UsageError(f"{nm} must be a contiguous [{d}] {want} tensor")
    if shadows_bf16 is not None:
        for w, sh in enumerate(shadows_bf16):
            size = d if compact is None else compact.length(w)
            if sh is not None and (sh.dtype != torch.bfloat16 or sh.numel() != size or sh.device != dev
                                   or not sh.is_contiguous()):
                raise UsageError(f"bf16 shadows must be contiguous [{size}] bfloat16 tensors on {dev}")
    if local_update is not None and nesterov is None and adam is None:
        raise UsageError("local_update needs the nesterov= or adam= scalars")
    flat_opt = local_update is None
    if nesterov is not None:
        flags |= N.SYNC_NESTEROV
        if flat_opt:
            a.theta = nesterov["theta"].data_ptr()
            a.velocity = nesterov["velocity"].data_ptr()
            tb = nesterov.get("theta_bf16")
            a.theta_bf16 = None if tb is None else tb.data_ptr()
        a.lr = float(nesterov["lr"])
        a.momentum = float(nesterov.get("momentum", 0.9))
    if adam is not None:
        # optim.Adam (optim.py:90-109): t is the step count after increment --
        # a host int ("t"), or a device int32 ("step") the kernel reads at run
        # time together with adam_bias_table(...) ("bias_table"): graph replay
        flags |= N.SYNC_ADAM
        b1, b2 = float(adam.get("beta1", 0.9)), float(adam.get("beta2", 0.999))
        step = adam.get("step")
        if step is not None:
            tab = adam["bias_table"]
            a.adam_step = step.data_ptr()
            a.adam_bias_table = tab.data_ptr()
            a.adam_table_len = tab.numel() // 2
            t = 1  # host scalars unused
        else:
            t = int(adam["t"])
        if flat_opt:
            a.theta = adam["theta"].data_ptr()
            a.velocity = adam["m"].data_ptr()
            a.second_moment = adam["v"].data_ptr()
            tb = adam.get("theta_bf16")
            a.theta_bf16 = None if tb is None else tb.data_ptr()
        a.lr = float(adam["lr"])
        a.beta1, a.beta2 = b1, b2
        a.one_minus_beta1, a.one_minus_beta2 = 1 - b1, 1 - b2
        a.bias1, a.bias2 = 1 - b1 ** t, 1 - b2 ** t
        a.eps = float(adam.get("eps", 1e-8))
    if compact is not None:
        a.slots = compact.slots.data_ptr()
        a.slot_stride = compact.slot_stride
    if local_update is not None:
        flags |= N.SYNC_LOCAL_UPDATE
        a.states = local_update["states"].data_ptr()
        a.updates = local_update["updates"].data_ptr()
        a.updates_per_cta = int(local_update["per_cta"])
    a.status = None if status is None else status.data_ptr()
    a.flags = flags
    return a


def adam_bias_rows(beta1: float = 0.9, beta2: float = 0.999, max_len: int = 1 << 20) -> np.ndarray:
    """[L, 2] float64: the Adam bias corrections (1 - beta1**t, 1 - beta2**t)
    for t = 0 .. L-1, computed exactly as the reference does (Python float
    pow, optim.py:107-108), up to the first t where both are exactly 1.0 --
    the kernel clamps larger steps to that row."""
    rows = []
    t = 0
    while True:
        c1, c2 = 1 - beta1 ** t, 1 - beta2 ** t
        rows.append((c1, c2))
        if (c1 == 1.0 and c2 == 1.0) or len(rows) >= max_len:
            break
        t += 1
    return np.array(rows, dtype=np.float64)


def adam_bias_table(beta1: float = 0.9, beta2: float = 0.999, dev=None) -> torch.Tensor:
    """adam_bias_rows on the device, flattened (sdp_sync_args.adam_bias_table)."""
    return torch.from_numpy(adam_bias_rows(beta1, beta2).reshape(-1)).to(device(dev))


def aggregate(grads, assignment) -> AggregatedGradient:
    """Masked averaging gbar_j = sum_i m_ij g_ij / sum_i m_ij (engine.py:60-79).

    Workers are accumulated in ascending id order from +0; uncovered entries get
    0.  float64 inputs reproduce the reference bit for bit; float32 inputs follow
    the same recurrence in fp32.  numpy inputs are copied to the device and the
    mean is returned as numpy (the host-buffer end-to-end path).  `assignment`
    may be this package's device MaskAssignment or the reference's own (numpy)
    one, so engine.run (engine.py:222) can call this unchanged.
    """
    from . import masking
    if masking.is_reference_assignment(assignment):
        # the reference's own MaskAssignment (engine.run hands us that one):
        # packed onto the device once, cached per object; the result carries
        # the reference's frozen divisor, as engine.py:79 returns it
        ref = assignment
        out = aggregate(grads, masking.from_reference(ref))
        return AggregatedGradient(gbar=out.gbar, divisor=ref.divisor)
    n, d = assignment.n_workers, assignment.topology.total
    if not torch.is_tensor(grads) and len(grads) != n:
        raise ProtocolError(f"aggregate received {len(grads)} gradients for {n} workers")
    host = not torch.is_tensor(grads) and len(grads) > 0 and isinstance(grads[0], np.ndarray)
    dev = assignment.device
    check = assignment.uncovered_params > 0
    if host:
        dt = torch.float64 if grads[0].dtype == np.float64 else torch.float32
        hosts = [torch.from_numpy(np.ascontiguousarray(g, dtype=dt_np(dt))) for g in grads]
        if all(h.numel() == d and _aligned(h) and _device_readable(h) for h in hosts):
            return _aggregate_host_zero_copy(hosts, assignment, check)
    if host:
        return _aggregate_host_staged([h.numpy() for h in hosts], assignment, check)
    else:
        reps = _as_replica_list(grads, n, d)
        dt = reps[0].dtype
        reps = [r if _aligned(r) and r.dtype == dt else r.contiguous().clone() for r in reps]
    gbar = torch.empty(d, dtype=dt, device=dev)
    status = owner_sync(reps, assignment, out=gbar, writeback=False, check_uncovered=check)
    if check and int(status.item()) & N.STATUS_UNCOVERED_LEAK:
        raise ProtocolError("a gradient reached a parameter with zero mask coverage")
    if host:
        out_np, out = _RESULTS.get(d, dt)
        out.copy_(gbar, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return AggregatedGradient(gbar=out_np, divisor=assignment.host_divisor())
    return AggregatedGradient(gbar=gbar, divisor=assignment.divisor)


class _PinnedResults:
    """Pinned host buffers for host-path aggregate results.  A buffer is handed
    out again only once every array built on it has been dropped by the caller
    (numpy views collapse their base onto the buffer, so its reference count
    is exact), which keeps the reference's fresh-result semantics
    (engine.py:60-79) while steady-state calls skip cudaHostAlloc (~30 ms for
    44 MB).  The caller receives a fresh view made INSIDE the lock, so the
    buffer's count has already risen when a concurrent caller looks at it:
    two callers never share a buffer."""

    def __init__(self, cap: int = 4):
        self.cap = cap
        self.bufs: dict = {}
        self.lock = threading.Lock()

    def get(self, d: int, dt: torch.dtype) -> tuple[np.ndarray, torch.Tensor]:
        with self.lock:
            base, t = self._get(d, dt)
            return base[:], t  # the lease: a view holding a reference to the buffer

    @staticmethod
    def _alloc(d: int, dt: torch.dtype) -> torch.Tensor:
        return torch.empty(d, dtype=dt, pin_memory=True)

    def _get(self, d: int, dt: torch.dtype) -> tuple[np.ndarray, torch.Tensor]:
        lst = self.bufs.setdefault((d, dt), [])
        for entry in lst:
            if sys.getrefcount(entry[0]) == 2:  # the pool's tuple + the call's argument: no lease out
                return entry
        t = self._alloc(d, dt)
        entry = (t.numpy(), t)
        lst.append(entry)
        if len(lst) > self.cap:
            lst.pop(0)  # in use by the caller: it keeps the buffer alive, the pool forgets it
        return entry


_RESULTS = _PinnedResults()
_STREAMS: dict = {}


def _copy_streams(dev: torch.device):
    """The H2D and D2H streams of the host pipeline (created once per device)."""
    if dev not in _STREAMS:
        _STREAMS[dev] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _STREAMS[dev]


def _aggregate_host_zero_copy(hosts, assignment, check: bool) -> AggregatedGradient:
    """Host-buffer aggregate over pinned inputs: ONE k_owner_sync launch reads
    the owners' gradients straight from pinned host memory over PCIe (only the
    tiles each worker owns an element of) and writes the mean straight into a
    pinned result buffer -- no device staging copies, no device replicas, no
    pipeline bubbles (B200: 5.08 ms vs 5.33 ms for the best copy pipeline at
    ResNet-18, N = 8, P = 4; tools/e2e_probe.py)."""
    d = assignment.topology.total
    dev = assignment.device
    dt = hosts[0].dtype
    out_np, out = _RESULTS.get(d, dt)
    status = owner_sync(hosts, assignment, out=out, writeback=False, check_uncovered=check,
                        zero_copy=True)
    torch.cuda.current_stream(dev).synchronize()
    if check and int(status.item()) & N.STATUS_UNCOVERED_LEAK:
        raise ProtocolError("a gradient reached a parameter with zero mask coverage")
    return AggregatedGradient(gbar=out_np, divisor=assignment.host_divisor())


# pageable host path (tools/pageable_probe.py, profiles/r2_pageable_staging_ab.jsonl:
# C4, 16 threads: 128 MB x 2 slots 67 ms, 64 MB x 3 slots 82 ms, 32 MB 120 ms;
# a 16-thread pageable -> pinned memcpy alone peaks at 56 GB/s on the box)
STAGE_CHUNK_BYTES = 128 << 20  # bytes staged per pipeline chunk (all workers together)
STAGE_SLOTS = 2                # pinned staging slots in flight
STAGE_PIECE = 4 << 20         # bytes per host-thread memcpy piece
_STAGING: dict = {}
_COPY_POOL = None


def _copy_pool():
    """Host threads for the pageable -> pinned staging copies (numpy copies
    release the GIL)."""
    global _COPY_POOL
    if _COPY_POOL is None:
        import concurrent.futures
        _COPY_POOL = concurrent.futures.ThreadPoolExecutor(max_workers=max(1, min(16, os.cpu_count() or 1)))
    return _COPY_POOL


def _staging(dev, dt: torch.dtype, elems: int):
    """Pinned staging slots (cached per device and dtype, grown on demand)."""
    key = (dev, dt)
    st = _STAGING.get(key)
    if st is None or st[0].numel() < STAGE_SLOTS * elems:
        buf = torch.empty(STAGE_SLOTS * elems, dtype=dt, pin_memory=True)
        st = (buf, buf.numpy(), [torch.cuda.Event() for _ in range(STAGE_SLOTS)], [False] * STAGE_SLOTS)
        _STAGING[key] = st
    return st


_STAGE_LOCK = threading.Lock()


def _aggregate_host_staged(grads, assignment, check: bool) -> AggregatedGradient:
    with _STAGE_LOCK:  # one caller at a time owns the staging slots
        return _host_staged(grads, assignment, check)


def _host_staged(grads, assignment, check: bool, pinned=None, chunk_bytes: int | None = None) -> AggregatedGradient:
    """Host-buffer aggregate over ordinary (pageable) numpy arrays -- what a
    reference caller passes (engine.run hands over flat_gradient outputs).
    The vector is cut into tile-range chunks of ~STAGE_CHUNK_BYTES of input;
    per chunk, a pool of host threads copies every worker's owned ranges into
    a pinned staging slot (a single-threaded driver staging copy ran ~4x
    slower), the copy engine moves the slot to the device replicas, the owner
    sync runs on the chunk, and the mean's D2H goes into a pinned result --
    host copies of chunk c+1 overlap the H2D / sync / D2H of chunk c.  With
    the uncovered-leak check every worker's full range is staged (the kernel
    reads all workers at zero-coverage entries).

    pinned: the inputs as pinned host tensors -- then the copy engine moves
    each chunk's owned ranges straight from them (no staging copies)."""
    n, d = assignment.n_workers, assignment.topology.total
    dev = assignment.device
    dt = pinned[0].dtype if pinned is not None else (torch.float64 if grads[0].dtype == np.float64 else torch.float32)
    esz = 8 if dt == torch.float64 else 4
    full = assignment.sync_plan()
    tile = full.tile
    n_tiles = len(full.all_tiles)
    ranges = [[(0, d)] if check else full.worker_ranges(w) for w in range(n)]
    staged = sum(ln for rs in ranges for _, ln in rs)
    k = max(1, min(n_tiles, -(-staged * esz // (chunk_bytes or STAGE_CHUNK_BYTES))))
    bounds = [n_tiles * c // k for c in range(k + 1)]
    chunks = []
    for c in range(k):
        lo_e, hi_e = bounds[c] * tile, min(d, bounds[c + 1] * tile)
        pieces, off = [], 0
        for w in range(n):
            for s, ln in ranges[w]:
                a, b = max(s, lo_e), min(s + ln, hi_e)
                if a < b:
                    pieces.append((w, a, b, off))
                    off += b - a
        chunks.append((lo_e, hi_e, pieces, off))
    slot_elems = max(1, max(ch[3] for ch in chunks))
    if pinned is None:
        buf, buf_np, evs, used = _staging(dev, dt, slot_elems)
    reps = [torch.empty(d, dtype=dt, device=dev) for _ in range(n)]
    gbar = torch.empty(d, dtype=dt, device=dev)
    out_np, out = _RESULTS.get(d, dt)
    cur = torch.cuda.current_stream(dev)
    s_in, s_out = _copy_streams(dev)
    s_in.wait_stream(cur)
    pool = _copy_pool()
    piece = max(1, STAGE_PIECE // esz)
    status = torch.zeros(1, dtype=torch.int32, device=dev) if check else None
    for c, (lo_e, hi_e, pieces, _) in enumerate(chunks):
        if pinned is not None:
            ev_in = torch.cuda.Event()
            with torch.cuda.stream(s_in):
                for w, a, b, off in pieces:
                    reps[w][a:b].copy_(pinned[w][a:b], non_blocking=True)
                ev_in.record(s_in)
            cur.wait_event(ev_in)
        else:
            slot = c % STAGE_SLOTS
            if used[slot]:
                evs[slot].synchronize()  # the slot's previous H2D has drained
            base = slot * slot_elems
            jobs = [(w, a0, min(a0 + piece, b), off + (a0 - a))
                    for w, a, b, off in pieces for a0 in range(a, b, piece)]
            list(pool.map(lambda j: np.copyto(buf_np[base + j[3]:base + j[3] + j[2] - j[1]],
                                              grads[j[0]][j[1]:j[2]]), jobs))
            with torch.cuda.stream(s_in):
                for w, a, b, off in pieces:
                    reps[w][a:b].copy_(buf[base + off:base + off + b - a], non_blocking=True)
                evs[slot].record(s_in)
                used[slot] = True
            cur.wait_event(evs[slot])
        plan = assignment.sync_plan(tile=tile, tile_lo=bounds[c], tile_hi=bounds[c + 1])
        owner_sync(reps, assignment, out=gbar, writeback=False, plan=plan, check_uncovered=check, status=status)
        ev_c = torch.cuda.Event()
        ev_c.record(cur)
        s_out.wait_event(ev_c)
        with torch.cuda.stream(s_out):
            out[lo_e:hi_e].copy_(gbar[lo_e:hi_e], non_blocking=True)
    s_out.synchronize()
    if check and int(status.item()) & N.STATUS_UNCOVERED_LEAK:
        raise ProtocolError("a gradient reached a parameter with zero mask coverage")
    for r in reps + [gbar]:
        r.record_stream(s_in)
    return AggregatedGradient(gbar=out_np, divisor=assignment.host_divisor())


def dt_np(dt: torch.dtype):
    return np.float64 if dt == torch.float64 else np.float32


class SgdNesterov:
    """optim.SgdNesterov (optim.py:71-87) over a device theta, on libsdp's
    k_nesterov: v = mu v + g; theta -= lr (g + mu v).  Like the reference
    (optim.py:78-80) a non-finite gradient raises NumericalError BEFORE theta
    or the velocity is touched: libsdp's k_check_finite scans the gradient
    first and the update kernel runs only if it is finite.

    The velocity takes theta's dtype and device on the first update unless
    `dtype` is given (the reference's theta is float64); every update checks
    that theta, velocity and gradient agree in dtype, size and device."""

    kind = "sgd-nesterov"

    def __init__(self, dim: int, momentum: float = 0.9, dtype=None, device_=None):
        self.dim = int(dim)
        self.momentum = momentum
        self._device = device_
        self.velocity = None if dtype is None else torch.zeros(dim, dtype=dtype, device=device(device_))

    def _check(self, theta: torch.Tensor, grad: torch.Tensor, theta_bf16) -> None:
        if self.velocity is None:
            self.velocity = torch.zeros(self.dim, dtype=theta.dtype, device=theta.device)
        _check_update_args("SgdNesterov", self.dim, theta, grad, {"velocity": self.velocity}, theta_bf16)

    def update(self, theta: torch.Tensor, grad: torch.Tensor, lr: float,
               theta_bf16: torch.Tensor | None = None) -> None:
        self._check(theta, grad, theta_bf16)
        s = stream_ptr(theta.device)
        _raise_if_nonfinite(grad, s)
        N.call("sdp_nesterov_update", sdp_dtype(theta.dtype), theta.numel(), ptr(theta),
               ptr(self.velocity), ptr(grad), float(lr), float(self.momentum), ptr(theta_bf16),
               None, s)

    def state_elements(self) -> int:
        return self.dim


class Adam:
    """optim.Adam (optim.py:90-112) over a device theta, on libsdp's k_adam:
    numpy's evaluation order, float64 bit-identical to the reference.  Like
    the reference a non-finite gradient raises NumericalError before the step
    counter, the moments or theta change.  The moments take theta's dtype and
    device on the first update unless `dtype` is given."""

    kind = "adam"

    def __init__(self, dim: int, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                 dtype=None, device_=None):
        self.dim = int(dim)
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.t = 0
        self.m = self.v = None
        if dtype is not None:
            self.m = torch.zeros(dim, dtype=dtype, device=device(device_))
            self.v = torch.zeros_like(self.m)

    def update(self, theta: torch.Tensor, grad: torch.Tensor, lr: float,
               theta_bf16: torch.Tensor | None = None) -> None:
        if self.m is None:
            self.m = torch.zeros(self.dim, dtype=theta.dtype, device=theta.device)
            self.v = torch.zeros_like(self.m)
        _check_update_args("Adam", self.dim, theta, grad, {"m": self.m, "v": self.v}, theta_bf16)
        s = stream_ptr(theta.device)
        _raise_if_nonfinite(grad, s)
        self.t += 1
        N.call("sdp_adam_update", sdp_dtype(theta.dtype), theta.numel(), ptr(theta), ptr(self.m), ptr(self.v),
               ptr(grad), float(lr), float(self.beta1), float(self.beta2), float(self.eps), self.t,
               ptr(theta_bf16), s)

    def state_elements(self) -> int:
        return 2 * self.dim


def make_optimizer(kind: str, dim: int, momentum: float = 0.9):
    """optim.make_optimizer (optim.py:115-120) for device thetas."""
    if kind == "sgd-nesterov":
        return SgdNesterov(dim, momentum=momentum)
    if kind == "adam":
        return Adam(dim)
    raise ConfigError(f"unknown optimizer kind {kind!r}")


def _check_update_args(name: str, dim: int, theta, grad, states: dict, theta_bf16) -> None:
    """Every buffer of an optimizer update: contiguous [dim], theta's dtype and
    device (the kernels cast every pointer to theta's element type)."""
    for nm, t in (("theta", theta), *states.items(), ("grad", grad)):
        if not torch.is_tensor(t) or t.dtype != theta.dtype or t.numel() != dim \
                or t.device != theta.device or not t.is_contiguous():
            raise UsageError(f"{name}: {nm} must be a contiguous [{dim}] {theta.dtype} tensor on "
                             f"{theta.device} (got {getattr(t, 'dtype', type(t))}, "
                             f"{getattr(t, 'numel', lambda: '?')()} elements, {getattr(t, 'device', '?')})")
    if theta.dtype not in (torch.float32, torch.float64) or theta.device.type != "cuda":
        raise UsageError(f"{name}: theta must be a float32 / float64 CUDA tensor")
    if theta_bf16 is not None and (theta_bf16.dtype != torch.bfloat16 or theta_bf16.numel() != dim
                                   or theta_bf16.device != theta.device or not theta_bf16.is_contiguous()):
        raise UsageError(f"{name}: theta_bf16 must be a contiguous [{dim}] bfloat16 tensor")


def _raise_if_nonfinite(grad: torch.Tensor, stream) -> None:
    """optim.py:78-80 / :102-103: NumericalError before anything is updated."""
    status = torch.zeros(1, dtype=torch.int32, device=grad.device)
    N.call("sdp_check_finite", sdp_dtype(grad.dtype), grad.numel(), ptr(grad), ptr(status), stream)
    if int(status.item()) & N.STATUS_NONFINITE:
        raise NumericalError("aggregated gradient contains non-finite values")
