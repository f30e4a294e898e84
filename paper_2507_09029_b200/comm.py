"""Multi-GPU owner-subset sync: one process per GPU, replicas peer-mapped over
NVLink, no NCCL on the data path.

Placement: the N logical workers sit contiguously on the G ranks
(worker w on rank w*G//N, SURVEY.md §7 hard part 6), so at N = G each GPU is
one worker and at G < N several workers share an HBM.

Bootstrap (once): every rank allocates its local workers' replicas (+ bf16
shadows) and a signal pad, exports CUDA-IPC handles, and all-gathers them
through torch.distributed (the only collective, plumbing only); each rank
then opens its peers' handles.  After that a sync step is ONE k_owner_sync
launch per rank: the rank reduces the tiles it leads (engine.tile_leaders),
reading every owner's replica -- local or over NVLink -- in ascending worker
order, and writes the mean into every owner's replica and bf16 shadow.
Per-CTA release/acquire flag barriers on the signal pads bracket the launch
(entry: every peer's gradients are ready; exit: every peer's writes into my
replicas have landed), with a spin timeout that reports instead of hanging.

The exchange logic (`exchange_handles`, `rank_layout`) is CUDA-free so the
N > 1 host path is tested with gloo on CPU (tests/test_multirank.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .engine import SyncPlan, gpu_of_worker
from .errors import CudaError, ProtocolError

PAD_WORDS_PER_CTA = 8  # >= world (<= 8 ranks)
IPC_HANDLE_BYTES = 64  # SDP_IPC_HANDLE_BYTES


@dataclass
class RankLayout:
    world: int
    rank: int
    n_workers: int
    gpu_of: np.ndarray

    @property
    def local_workers(self) -> list[int]:
        return [w for w in range(self.n_workers) if int(self.gpu_of[w]) == self.rank]


def rank_layout(n_workers: int, world: int, rank: int) -> RankLayout:
    if not 1 <= world <= 8:
        raise ProtocolError(f"the peer-mapped sync supports 1..8 ranks, got {world}")
    if world > n_workers:
        raise ProtocolError(f"{world} ranks for {n_workers} workers: a rank would hold no replica")
    return RankLayout(world, rank, n_workers, gpu_of_worker(n_workers, world))


def exchange_handles(local: dict, all_gather) -> list[dict]:
    """All-gather every rank's {name: (handle_bytes, offset)} export table.

    `all_gather(obj) -> list[obj]` is torch.distributed.all_gather_object bound
    to the process group (or a fake in tests)."""
    tables = all_gather({k: (bytes(h), int(off)) for k, (h, off) in local.items()})
    for r, t in enumerate(tables):
        for k, (h, _) in t.items():
            if len(h) != IPC_HANDLE_BYTES:
                raise ProtocolError(f"rank {r} sent a malformed IPC handle for {k}")
    return tables


def ipc_export(t: torch.Tensor) -> tuple[bytes, int]:
    h = (C.c_uint8 * 64)()
    off = C.c_uint64(0)
    N.call("sdp_ipc_export", C.c_void_p(t.data_ptr()), h, C.byref(off))
    return bytes(h), int(off.value)


def ipc_import(handle: bytes, offset: int) -> int:
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p(0)
    N.call("sdp_ipc_import", h, C.c_uint64(offset), C.byref(p))
    return int(p.value)


def bind_rank_args(plan: SyncPlan, dtype: int, rep_ptr, sh_ptr, pad_ptr, status_ptr: int,
                   timeout_cycles: int = 20_000_000_000) -> N.SyncArgs:
    """k_owner_sync arguments of one rank: every worker's replica address (local
    or peer-mapped), the ranks' signal pads, and the rank's own tile table."""
    a = plan.args(dtype)
    for w in range(plan.assignment.n_workers):
        a.replicas[w] = rep_ptr[w]
        a.shadow_bf16[w] = sh_ptr[w] or None
    a.world = plan.world
    a.rank = plan.rank
    for r in range(plan.world):
        a.signal_pads[r] = pad_ptr[r]
    a.flags = N.SYNC_WRITEBACK
    a.status = status_ptr
    a.timeout_cycles = timeout_cycles
    return a


class PeerGroup:
    """Peer-mapped replicas of one assignment across the ranks of a process group."""

    def __init__(self, assignment, rank: int, world: int, device, all_gather,
                 dtype=torch.float32, shadows: bool = True, max_grid: int | None = None,
                 timeout_cycles: int = 20_000_000_000, owner_mask: torch.Tensor | None = None,
                 compact: bool = False):
        """compact: every worker's replica (and shadow) holds only the tiles it
        owns (storage.CompactLayout); the kernel finds each owner's copy of a
        tile through the slot table (sdp_sync_args.slots)."""
        self.assignment = assignment
        self.layout = rank_layout(assignment.n_workers, world, rank)
        self.device = torch.device(device)
        d = assignment.topology.total
        # owner_mask: the sync-space mask of a layout.SyncLayout when replicas are
        # kept window-class-major (width-wise assignments)
        self.plan = SyncPlan(assignment, world=world, rank=rank, resident=True, max_grid=max_grid,
                             owner_mask=owner_mask)
        # every rank must launch the same grid for the pairwise per-CTA barrier
        self.grid = max(all_gather(self.plan.grid))
        if self.plan.grid != self.grid:
            self.plan = SyncPlan(assignment, world=world, rank=rank, resident=True,
                                 force_grid=self.grid, owner_mask=owner_mask)
        self.compact = None
        if compact:
            from .storage import CompactLayout
            self.compact = CompactLayout(self.plan)
        size = {w: (self.compact.length(w) if self.compact else d) for w in self.layout.local_workers}
        self.replicas = {w: torch.zeros(size[w], dtype=dtype, device=self.device) for w in self.layout.local_workers}
        self.shadows = ({w: torch.zeros(size[w], dtype=torch.bfloat16, device=self.device)
                         for w in self.layout.local_workers} if shadows else {})
        self.pad = torch.zeros(self.grid * PAD_WORDS_PER_CTA, dtype=torch.int32, device=self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._imported: list[int] = []
        exports = {f"rep{w}": ipc_export(t) for w, t in self.replicas.items()}
        exports.update({f"sh{w}": ipc_export(t) for w, t in self.shadows.items()})
        exports["pad"] = ipc_export(self.pad)
        tables = exchange_handles(exports, all_gather)
        self.rep_ptr = [0] * assignment.n_workers
        self.sh_ptr = [0] * assignment.n_workers
        self.pad_ptr = [0] * world
        for r, table in enumerate(tables):
            for key, (h, off) in table.items():
                if r == rank:
                    p = {"pad": self.pad.data_ptr()}.get(key)
                    if p is None:
                        w = int(key[3:] if key.startswith("rep") else key[2:])
                        p = (self.replicas if key.startswith("rep") else self.shadows)[w].data_ptr()
                else:
                    p = ipc_import(h, off)
                    self._imported.append(p)
                if key == "pad":
                    self.pad_ptr[r] = p
                elif key.startswith("rep"):
                    self.rep_ptr[int(key[3:])] = p
                else:
                    self.sh_ptr[int(key[2:])] = p
        self.epoch = 0
        self.args = bind_rank_args(self.plan, N.DTYPE_F32 if dtype == torch.float32 else N.DTYPE_F64,
                                   self.rep_ptr, self.sh_ptr, self.pad_ptr, self.status.data_ptr(),
                                   timeout_cycles)
        # barrier epochs live on the device (one per CTA), so a launch recorded
        # in a CUDA graph replays with fresh flag values every time
        self.epochs = torch.zeros(self.grid, dtype=torch.int32, device=self.device)
        self.args.epoch_counters = self.epochs.data_ptr()
        if self.compact is not None:
            self.args.slots = self.compact.slots.data_ptr()
            self.args.slot_stride = self.compact.slot_stride
        self._fn = N.lib().sdp_owner_sync

    def launch(self, stream=None) -> None:
        """One synchronised owner-subset sync step (asynchronous on the stream;
        capturable in a CUDA graph — every rank must replay its graph in step)."""
        self.epoch += 1
        self.args.epoch = self.epoch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = self._fn(C.byref(self.args), C.c_void_p(s.cuda_stream))
        if rc:
            N.check(rc, "sdp_owner_sync")

    def check(self) -> None:
        st = int(self.status.item())
        if st & N.STATUS_BARRIER_TIMEOUT:
            raise CudaError(f"rank {self.layout.rank}: cross-GPU barrier timed out (a peer stalled)")

    def close(self) -> None:
        for p in self._imported:
            N.call("sdp_ipc_close", C.c_void_p(p))
        self._imported.clear()


_GROUPS: dict = {}


def _dist_all_gather(obj) -> list:
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def aggregate_local(grads, assignment, rank: int | None = None, world: int | None = None,
                    device=None, all_gather=None, fresh: bool = True, check: bool = False) -> dict:
    """Per-rank form of engine.aggregate (engine.py:60-79) for torchrun jobs
    (SURVEY.md §8b): every rank passes the gradients of ITS local workers
    (contiguous placement, rank_layout) and receives, for each of them, the
    owner-subset mean on that worker's owned elements.

    grads: {worker: fp32 [d] tensor on this rank's GPU} (a bare tensor when
    the rank holds one worker); gradients must be zero off the worker's mask,
    as the reference's masked backward leaves them (models.py:369-382).
    Returns {worker: [d] fp32}: gbar on the worker's owned elements, 0
    elsewhere -- exactly `aggregate(...).gbar * param_masks[w]`, bit for bit
    with the co-resident kernel.  All ranks must call it together (it is a
    collective over the peer-mapped replicas; the first call per assignment
    exchanges CUDA-IPC handles through torch.distributed).  fresh=False
    returns the peer group's replicas themselves (overwritten by the next
    call) instead of copies.  check=True waits for the kernel and raises on a
    cross-rank barrier timeout."""
    import torch.distributed as dist
    if rank is None or world is None:
        if not dist.is_initialized():
            raise ProtocolError("aggregate_local needs rank/world or an initialised torch.distributed")
        rank = dist.get_rank() if rank is None else rank
        world = dist.get_world_size() if world is None else world
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (id(assignment), rank, world, dev)
    g = _GROUPS.get(key)
    if g is None or g.assignment is not assignment:
        g = PeerGroup(assignment, rank, world, dev, all_gather or _dist_all_gather, shadows=False)
        _GROUPS[key] = g
    local = g.layout.local_workers
    if torch.is_tensor(grads):
        if len(local) != 1:
            raise ProtocolError(f"rank {rank} holds workers {local}: pass a {{worker: gradient}} dict")
        grads = {local[0]: grads}
    if sorted(grads) != local:
        raise ProtocolError(f"aggregate_local on rank {rank} received gradients for workers "
                            f"{sorted(grads)}, expected its local workers {local}")
    d = assignment.topology.total
    for w, t in grads.items():
        if not torch.is_tensor(t) or t.shape != (d,) or t.dtype != torch.float32 or t.device != dev:
            raise ProtocolError(f"worker {w}: expected a float32 [{d}] tensor on {dev}")
        if t.data_ptr() != g.replicas[w].data_ptr():
            g.replicas[w].copy_(t)
    g.launch()
    if check:
        torch.cuda.current_stream(dev).synchronize()
        g.check()
    return {w: g.replicas[w].clone() if fresh else g.replicas[w] for w in local}


def close_local_groups() -> None:
    """Unmap every peer group aggregate_local opened (call before
    destroy_process_group)."""
    for g in _GROUPS.values():
        g.close()
    _GROUPS.clear()


def bench_setup(assignment, rank: int, world: int, device):
    """bench.py --gpus G: peer group with seeded replicas (randn, zero off-mask)."""
    import torch.distributed as dist

    def all_gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    for peer in range(world):
        if peer != rank:
            try:
                N.call("sdp_enable_peer", peer)
            except Exception:
                pass  # IPC mappings enable peer access lazily
    p2p = p2p_copy_probe(rank, world, device, all_gather)
    g = PeerGroup(assignment, rank, world, device, all_gather)
    pm = assignment.param_masks
    gen = torch.Generator(device=device)
    for w, t in g.replicas.items():
        gen.manual_seed(1000 + w)
        t.copy_(torch.randn(t.numel(), generator=gen, device=device) * pm[w])
    torch.cuda.synchronize(device)
    dist.barrier()
    own = g.plan.owned_elems
    lb = link_bytes(g.plan, g.layout, shadows=True)
    meta = {"tiles": g.plan.n_tiles, "grid": g.grid, "tiles_per_cta": g.plan.tiles_per_cta,
            "roofline": {"nvlink_tx_bytes_per_launch": lb["tx"], "nvlink_rx_bytes_per_launch": lb["rx"],
                         "busbw_bytes_per_launch": busbw_bytes(g.plan, g.layout),
                         "p2p_copy_GBps_measured": p2p}}
    return g.launch, own * 4, own * 10, meta


def p2p_copy_probe(rank: int, world: int, device, all_gather, mib: int = 512, reps: int = 5) -> float:
    """Measured peer-copy bandwidth per direction: every rank
    copies `mib` MiB into its ring neighbour's CUDA-IPC-mapped buffer at the
    same time (copy engine, cudaMemcpyDefault); GB/s of this rank, CUDA events."""
    import torch.distributed as dist
    n = mib << 18  # float32 elements
    dst = torch.empty(n, dtype=torch.float32, device=device)
    src = torch.ones(n, dtype=torch.float32, device=device)
    tables = exchange_handles({"probe": ipc_export(dst)}, all_gather)
    peer = (rank + 1) % world
    h, off = tables[peer]["probe"]
    ptr_ = dst.data_ptr() if peer == rank else ipc_import(h, off)
    s = torch.cuda.current_stream(device)
    N.call("sdp_copy_async", C.c_void_p(ptr_), C.c_void_p(src.data_ptr()), C.c_size_t(n * 4),
           C.c_void_p(s.cuda_stream))
    torch.cuda.synchronize(device)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        N.call("sdp_copy_async", C.c_void_p(ptr_), C.c_void_p(src.data_ptr()), C.c_size_t(n * 4),
               C.c_void_p(s.cuda_stream))
    e1.record(s)
    torch.cuda.synchronize(device)
    gbps = n * 4 * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    dist.barrier()
    if peer != rank:
        N.call("sdp_ipc_close", C.c_void_p(ptr_))
    del dst, src
    return gbps


def link_bytes(plan: SyncPlan, layout: RankLayout, shadows: bool) -> dict:
    """Bytes this rank's NVLink ports carry per launch, per direction.  The
    leader of a tile reads 4 B per element from every remote owner (their TX,
    its RX) and writes 4 B (+ 2 B bf16 shadow) to every remote owner (its TX,
    their RX); summed over every rank's led tiles (plan.leaders)."""
    tiles = plan.all_tiles
    lens = (tiles["len_flags"] & N.TILE_LEN_MASK).astype(np.int64)
    bits = tiles["owner_bits"].astype(np.uint64)
    me = layout.rank
    wb = 4 + (2 if shadows else 0)
    mine_remote = np.zeros(len(tiles), dtype=np.int64)   # my workers among the tile's owners
    remote = np.zeros(len(tiles), dtype=np.int64)        # owners not on the leader's GPU
    leader = plan.leaders
    for w in range(layout.n_workers):
        on = ((bits >> np.uint64(w)) & np.uint64(1)).astype(bool)
        g = int(layout.gpu_of[w])
        remote += (on & (leader != g)).astype(np.int64)
        if g == me:
            mine_remote += (on & (leader != me)).astype(np.int64)
    led = leader == me
    rx = int((lens * remote)[led].sum() * 4 + (lens * mine_remote)[~led].sum() * wb)
    tx = int((lens * remote)[led].sum() * wb + (lens * mine_remote)[~led].sum() * 4)
    return {"tx": tx, "rx": rx}


def busbw_bytes(plan: SyncPlan, layout: RankLayout) -> int:
    """SURVEY §8(d) bus bytes of this rank per sync (the nccl-tests busbw
    convention): sum over the elements j this rank's GPU owns of
    2(k_j - 1)/k_j * 4 B, k_j = number of distinct GPUs owning j.  Tiles are
    counted with their owner union (uniform tiles exactly; the few mixed
    tiles of a block assignment approximately)."""
    tiles = plan.all_tiles
    lens = (tiles["len_flags"] & N.TILE_LEN_MASK).astype(np.float64)
    bits = tiles["owner_bits"].astype(np.uint64)
    gmask = np.zeros(len(tiles), dtype=np.int64)
    for w in range(layout.n_workers):
        on = ((bits >> np.uint64(w)) & np.uint64(1)).astype(bool)
        gmask[on] |= 1 << int(layout.gpu_of[w])
    k = np.bitwise_count(gmask.astype(np.uint64)).astype(np.float64)
    mine = ((gmask >> layout.rank) & 1).astype(bool) & (k > 0)
    return int((2 * (k[mine] - 1) / k[mine] * lens[mine] * 4).sum())
