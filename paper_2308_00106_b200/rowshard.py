"""Row-sharded multi-GPU SpMV with an x all-gather between iterations (K8).

The reference's only parallelism is the even row split of spmv_csr_parallel
(kernels.py:38-49, 102-128): disjoint output row ranges, no reduction.  Here
each rank (one process per GPU, torch.distributed over NCCL) owns the rows
[r_k, r_{k+1}) of make_row_partition(n_rows, world) and the same-index slice
of x (square matrices).  One step is

    all_gather(x slices -> padded full x)   (NCCL over NVLink / NVSwitch)
    y_k = A_k x                              (libsme CSR kernel on the shard)

Slices are padded to pad = ceil(n / world) entries so the gather is one
equal-chunk all_gather_into_tensor; the shard's column ids are remapped once
(sme_rowshard_remap_cols) from matrix columns to slots of the padded vector.
With the CSR-vector kernel and the parent matrix's lanes the sharded y is
bitwise equal to the 1-GPU y (no row's reduction order changes).

Pipelined exchange (kernel 'seg', the C4 path).  A shard of a randomly permuted
matrix needs ~all of x, and its SpMV is a sequence of column-panel passes that
each read ONE x slice.  The shard's panels are aligned to the ranks' padded
slots (P a multiple of world), so pass p needs only the slot of rank
p // (P / world).  The exchange is then world broadcasts (rank k's slot from
rank k, in rank order) on a communication stream, and the compute stream starts
the passes of slot k as soon as broadcast k has landed: the transfer of slot
k+1 overlaps the passes of slot k, instead of one all-gather ahead of all
passes.  The pass order (hence y, bit for bit) is that of the non-pipelined
seg SpMV of the same shard.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _cuda, _lib
from ._cuda import ptr, stream
from .kernels import default_lanes, make_row_partition, spmv_into
from .matio import CsrMatrix


class ShardPlan:
    """Host-side partition of rows (and of x) over `world` ranks."""

    def __init__(self, n_rows: int, n_cols: int, world: int):
        if world < 1:
            raise ValueError("world size must be >= 1")
        self.n_rows, self.n_cols, self.world = int(n_rows), int(n_cols), int(world)
        self.rows = make_row_partition(self.n_rows, self.world).boundaries
        self.cols = make_row_partition(self.n_cols, self.world).boundaries
        self.pad = -(-self.n_cols // self.world)

    def row_range(self, rank: int) -> tuple[int, int]:
        return int(self.rows[rank]), int(self.rows[rank + 1])

    def col_range(self, rank: int) -> tuple[int, int]:
        return int(self.cols[rank]), int(self.cols[rank + 1])

    def slot_of(self, col: np.ndarray) -> np.ndarray:
        """Host statement of the column -> padded-slot map (the kernel is the product path)."""
        col = np.asarray(col, dtype=np.int64)
        part = np.searchsorted(self.cols, col, side="right") - 1
        return part * self.pad + (col - self.cols[part])

    def pad_slice(self, x_local: torch.Tensor) -> torch.Tensor:
        """x slice of this rank padded to `pad` entries (the all-gather chunk)."""
        out = torch.zeros(self.pad, dtype=x_local.dtype, device=x_local.device)
        out[: x_local.numel()] = x_local
        return out

    def unpad(self, x_full_padded: torch.Tensor) -> torch.Tensor:
        parts = [x_full_padded[k * self.pad : k * self.pad + (self.cols[k + 1] - self.cols[k])] for k in range(self.world)]
        return torch.cat(parts)


def allgather_padded(x_full: torch.Tensor, x_chunk: torch.Tensor, group=None) -> None:
    """x_full[k*pad:(k+1)*pad] <- rank k's chunk.  NCCL: one all_gather_into_tensor;
    other backends (gloo, for CPU tests): all_gather into views."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(x_full, x_chunk, group=group)
    else:
        world = dist.get_world_size(group)
        views = list(x_full.view(world, -1).unbind(0))
        dist.all_gather(views, x_chunk, group=group)


def pipelined_exchange(x_full: torch.Tensor, x_chunk: torch.Tensor, rank: int, world: int, on_slot, group=None):
    """Assemble the padded x from every rank's chunk by `world` in-order broadcasts;
    on_slot(k) runs after slot k is in place (on the caller's side of the stream
    hand-off: with CUDA tensors the broadcasts run on a side stream and on_slot
    receives the CUDA event to wait on, see RowShardedSpMV.step)."""
    pad = x_chunk.numel()
    x_full[rank * pad : (rank + 1) * pad].copy_(x_chunk)
    for k in range(world):
        dist.broadcast(x_full[k * pad : (k + 1) * pad], src=k, group=group)
        on_slot(k)


class RowShardedSpMV:
    """One rank's shard of A plus the gathered-x buffer; step() = all-gather + SpMV."""

    def __init__(self, m: CsrMatrix, plan: ShardPlan, rank: int, kernel: str = "vector", lanes: int | None = None,
                 *, local: bool = False):
        """m: the whole matrix (this rank's rows are sliced out), or with local=True
        already this rank's row shard (rows [lo, hi) of the whole matrix, all columns):
        a sharded setup builds only its own rows (bench.py multi-GPU)."""
        self.plan, self.rank, self.kernel = plan, rank, kernel
        lo, hi = plan.row_range(rank)
        self.row_lo, self.row_hi = lo, hi
        if local:
            if m.n_rows != hi - lo or m.n_cols != plan.n_cols:
                raise ValueError(f"local shard is {m.n_rows} x {m.n_cols}, rank {rank} owns {hi - lo} x {plan.n_cols}")
            lo, hi = 0, m.n_rows
        p0, p1 = int(m.d_row_ptr[lo]), int(m.d_row_ptr[hi])
        dev = m.d_row_ptr.device
        # a shard of a wide (int64 row_ptr) matrix goes back to int32 offsets when it fits
        row_ptr = (m.d_row_ptr[lo : hi + 1] - p0).to(_cuda.row_ptr_dtype(p1 - p0)).contiguous()
        col = torch.empty(p1 - p0, dtype=torch.int32, device=dev)
        _lib.call("sme_rowshard_remap_cols", p1 - p0, m.n_cols, plan.world, plan.pad, ptr(m.d_col_idx) + 4 * p0,
                  ptr(col), stream())
        val = m.d_values[p0:p1].clone()
        self.local = CsrMatrix._from_device(hi - lo, plan.world * plan.pad, row_ptr, col, val)
        # the parent's lanes keep every row's reduction order -> bitwise equal to 1 GPU
        self.lanes = lanes or (default_lanes(m) if kernel == "vector" else None)
        self.x_full = torch.zeros(plan.world * plan.pad, dtype=m.dtype, device=dev)
        self.y = torch.empty(hi - lo, dtype=m.dtype, device=dev)
        self.seg = None
        if kernel in ("seg", "auto"):
            from .kernels import auto_kernel
            from .seg import auto_seg_panels, seg_of

            if kernel == "seg" or auto_kernel(self.local) == "seg":
                # panels aligned to the ranks' padded slots: P = world * ceil(P_auto / world)
                per = -(-auto_seg_panels(self.local) // plan.world)
                self.seg = seg_of(self.local, plan.world * per)
                self.kernel = "seg"
        self._comm = None

    @property
    def nnz(self) -> int:
        return self.local.nnz

    def spmv(self, x_full: torch.Tensor | None = None) -> torch.Tensor:
        xf = self.x_full if x_full is None else x_full
        if self.seg is not None:
            self.seg.spmv_into(xf, self.y)
        else:
            spmv_into(self.local, xf, self.y, self.kernel, lanes=self.lanes)
        return self.y

    @property
    def pipelined(self) -> bool:
        """Per-slot broadcasts pipelined with the panel passes (seg shards); the env
        SME_PIPELINED_EXCHANGE=0 falls back to one all-gather before the passes, =force
        pipelines even a world of one (a 1-GPU check of the NCCL broadcast path)."""
        import os

        mode = os.environ.get("SME_PIPELINED_EXCHANGE", "1")
        return self.seg is not None and mode != "0" and (self.plan.world > 1 or mode == "force")

    def step(self, x_chunk: torch.Tensor, group=None) -> torch.Tensor:
        """Exchange the padded x chunks of every rank, then y_local = A_local x.

        seg shards: per-slot broadcasts on a side stream, each slot's panel passes
        launched as soon as it lands (pipelined_exchange); other kernels: one
        all-gather, then the SpMV."""
        if not self.pipelined:
            allgather_padded(self.x_full, x_chunk, group)
            return self.spmv()
        world, lay = self.plan.world, self.seg
        per = lay.n_panels // world
        main = torch.cuda.current_stream()
        comm = self._comm = self._comm or torch.cuda.Stream(device=self.x_full.device)
        comm.wait_stream(main)  # the previous step's passes are done reading x_full
        events = []

        def landed(k: int) -> None:
            ev = torch.cuda.Event()
            ev.record(comm)
            events.append(ev)

        with torch.cuda.stream(comm):
            pipelined_exchange(self.x_full, x_chunk, self.rank, world, landed, group)
        for p in range(lay.n_panels):
            if p % per == 0:
                main.wait_event(events[p // per])
            lay._window(p, self.x_full)
            lay._pass(p, self.x_full, self.y)
        lay._window(None, None)
        return self.y


def virtual_ranks(m: CsrMatrix, world: int, kernel: str = "vector") -> list[RowShardedSpMV]:
    """All `world` shards on the current device (single-GPU test of the multi-GPU path)."""
    plan = ShardPlan(m.n_rows, m.n_cols, world)
    return [RowShardedSpMV(m, plan, k, kernel) for k in range(world)]


def virtual_step(shards: list[RowShardedSpMV], x: torch.Tensor) -> torch.Tensor:
    """The all-gather replaced by device copies: every shard sees the same padded x."""
    plan = shards[0].plan
    x_full = torch.zeros(plan.world * plan.pad, dtype=x.dtype, device=x.device)
    for k in range(plan.world):
        lo, hi = plan.col_range(k)
        x_full[k * plan.pad : k * plan.pad + hi - lo] = x[lo:hi]
    return torch.cat([s.spmv(x_full).clone() for s in shards])


def require_cuda_rank(local_rank: int) -> torch.device:
    _cuda.require_cuda()
    torch.cuda.set_device(local_rank)
    return torch.device("cuda", local_rank)


# ---------------------------------------------------------------------------
# Multi-GPU power iteration with the exchange fused into the SpMV epilogue
# ---------------------------------------------------------------------------
class IpcBuffer:
    """A whole cudaMalloc allocation (sme_ipc_malloc) shared with the other ranks of the
    node through a CUDA IPC handle, viewed as a torch tensor without a copy."""

    def __init__(self, n: int, device: torch.device, dtype=torch.float64):
        import ctypes

        self.n, self.dtype = int(n), dtype
        esize = torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        _lib.call("sme_ipc_malloc", max(1, self.n) * esize, ctypes.byref(p))
        self.ptr = int(p.value)
        typestr = {torch.float64: "<f8", torch.float32: "<f4"}[dtype]
        cai = {"shape": (self.n,), "typestr": typestr, "data": (self.ptr, False), "version": 3, "strides": None}
        self.tensor = torch.as_tensor(type("CAI", (), {"__cuda_array_interface__": cai})(), device=device)

    def handle(self) -> bytes:
        import ctypes

        buf = (ctypes.c_uint8 * 64)()
        _lib.call("sme_ipc_get_handle", self.ptr, buf)
        return bytes(buf)

    @staticmethod
    def open(handle: bytes) -> int:
        import ctypes

        p = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        _lib.call("sme_ipc_open", buf, ctypes.byref(p))
        return int(p.value)

    def free(self) -> None:
        if self.ptr:
            self.tensor = None
            _lib.call("sme_ipc_free", self.ptr)
            self.ptr = 0


class DistributedPowerIteration:
    """Row-sharded power iteration on the symmetric permutation C = P A P^-1 (the
    folded ROW_COLUMN operator of iterative.py), one rank per GPU.

    Every rank keeps the FULL iterate in two IPC-shared buffers (ping-pong).  One
    step is the shard's seg panel passes, the last with the epilogue of
    sme_spmv_seg_epi_peers: each finished row v = s * (C w)[r] is stored into this
    rank's next buffer and, over NVLink, into every peer's — the all-gather of the
    iterate is fused into the SpMV, row by row, instead of following it.  Then one
    8-byte all-reduce of the shards' sums of squares, which is also the step's
    barrier: no rank starts writing the other buffer before every rank has finished
    reading it.  Same eigenpair as the one-GPU PowerIteration (rows are disjoint,
    so nothing else is exchanged).
    """

    def __init__(self, A: CsrMatrix, p, x0, group=None):
        from .iterative import PermutedOperator
        from .seg import seg_of

        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        dev = A.d_row_ptr.device
        op = PermutedOperator(A, p, p)  # C = permute_csr(A, p, p)
        self.op, self.n = op, A.n_rows
        plan = ShardPlan(self.n, self.n, self.world)
        lo, hi = plan.row_range(self.rank)
        self.row_lo, self.row_hi = lo, hi
        Cm = op.B
        p0, p1 = int(Cm.d_row_ptr[lo]), int(Cm.d_row_ptr[hi])
        local = CsrMatrix._from_device(hi - lo, self.n,
                                       (Cm.d_row_ptr[lo : hi + 1] - p0).to(_cuda.row_ptr_dtype(p1 - p0)).contiguous(),
                                       Cm.d_col_idx[p0:p1].clone(), Cm.d_values[p0:p1].clone())
        self.local = local
        self.lay = seg_of(local, full_last=True, split_rows=False)  # its epilogue pass stores to peers
        self.bufs = [IpcBuffer(self.n, dev), IpcBuffer(self.n, dev)]
        handles = [b.handle() for b in self.bufs]
        everyone = [None] * self.world
        dist.all_gather_object(everyone, handles, group=group)
        self.opened: list[int] = []
        self.peers = []
        for b in range(2):
            ptrs = []
            for j in range(self.world):
                if j != self.rank:
                    q = IpcBuffer.open(everyone[j][b])
                    self.opened.append(q)
                    ptrs.append(q)
            self.peers.append(torch.tensor(ptrs or [0], dtype=torch.int64, device=dev))
        z = op.to_permuted(x0)
        z = z / torch.linalg.vector_norm(z)
        self.bufs[0].tensor.copy_(z)
        self.cur = 0
        self.res = torch.tensor([1.0, 0.0], dtype=torch.float64, device=dev)
        self.partials = torch.zeros(self.lay.n_warps, dtype=torch.float64, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        self.tmp = torch.empty(max(1, hi - lo), dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        dist.barrier(group=group)

    def step(self) -> None:
        lay, a, b = self.lay, self.bufs[self.cur].tensor, self.bufs[1 - self.cur]
        P = lay.n_panels
        for q in range(P - 1):
            lay._window(q, a)
            lay._pass(q, a, self.tmp)
        lay._window(P - 1, a)
        vb = 8
        o = int(lay.offsets[P - 1])
        _lib.call("sme_spmv_seg_epi_peers", _lib.SME_F64, lay.n_warps, ptr(lay.pk) + 4 * o, ptr(lay.val) + vb * o,
                  ptr(lay.hdr) + 4 * (o // 128), ptr(lay.plans) + 4 * (P - 1) * (lay.n_warps + 1),
                  ptr(a) + vb * int(lay.bounds_host[P - 1]), ptr(self.tmp), int(P > 1), b.ptr, self.row_lo,
                  ptr(self.peers[1 - self.cur]), self.world - 1, ptr(self.res), ptr(self.partials), ptr(self.ticket),
                  ptr(self.res), stream())
        lay._window(None, None)
        dist.all_reduce(self.res[1:2], group=self.group)  # global ||w||^2, and the step barrier
        torch.rsqrt(self.res[1:2], out=self.res[0:1])
        self.cur = 1 - self.cur

    def run(self, steps: int) -> None:
        for _ in range(steps):
            self.step()

    @property
    def eigenvalue(self) -> float:
        return float(self.res[1].sqrt().item())

    def x(self) -> torch.Tensor:
        return self.op.from_permuted(self.bufs[self.cur].tensor * self.res[0])

    def close(self) -> None:
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # no peer still stores into our buffers
        for q in self.opened:
            _lib.call("sme_ipc_close", q)
        self.opened = []
        dist.barrier(group=self.group)
        for buf in self.bufs:
            buf.free()
