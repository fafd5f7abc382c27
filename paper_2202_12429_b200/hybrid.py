"""DLRM hybrid parallelism over N GPUs.

Embeddings are model-parallel: rank r owns the tables ``shard.table_shards``
deals it (round-robin) and runs the whole BagPipe path -- planner, HBM
cache, pinned store, EmbeddingBag -- for those tables over the GLOBAL batch.
The dense MLPs are data-parallel: rank r trains examples
[r*B/N, (r+1)*B/N).  Per iteration:

1. forward all-to-all: rank r's pooled rows [B, T_r, D] (example-major, so
   the rows for rank q's examples are one contiguous block) go to their
   example owners; each rank reassembles [B/N, T, D] in global table order;
2. the dense step (bottom MLP, interaction, top MLP, backward);
3. backward all-to-all of the pooled-row gradients to the table owners,
   scaled by 1/N (the global loss is the mean over all B examples, each
   rank's loss the mean over its B/N);
4. MLP gradients all-reduced (sum / N) before the SGD step;
5. the owners' EmbeddingBag backward + optimizer on their cached rows.

``EmbeddingExchange`` is backend-agnostic (NCCL on GPUs, gloo on CPU in
tests/test_hybrid_dist.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .shard import table_shards


class EmbeddingExchange:
    """All-to-all of pooled embedding rows between table owners and example owners."""

    def __init__(self, num_tables: int, dim: int, rank: int, world: int, group=None, shards=None):
        self.num_tables, self.dim, self.rank, self.world, self.group = num_tables, dim, rank, world, group
        self.shards = shards if shards is not None else table_shards(num_tables, world)
        self.local_tables = self.shards[rank]
        order = [t for s in self.shards for t in s]        # concatenation order of the received blocks
        self.to_global = torch.tensor([order.index(t) for t in range(num_tables)], dtype=torch.long)
        self.to_blocks = torch.tensor(order, dtype=torch.long)
        self._dev = None

    def _idx(self, device):
        if self._dev != device:
            self.to_global = self.to_global.to(device)
            self.to_blocks = self.to_blocks.to(device)
            self._dev = device
        return self.to_global, self.to_blocks

    def forward(self, pooled_local: torch.Tensor) -> torch.Tensor:
        """[B, T_r, D] rows of this rank's tables -> [B/N, T, D] for this rank's examples."""
        b, t_r, d = pooled_local.shape
        n = self.world
        if b % n:
            raise ValueError(f"global batch {b} not divisible by {n} ranks")
        bl = b // n
        recv = torch.empty(sum(bl * len(s) * d for s in self.shards), dtype=pooled_local.dtype,
                           device=pooled_local.device)
        dist.all_to_all_single(recv, pooled_local.contiguous().view(-1),
                               output_split_sizes=[bl * len(s) * d for s in self.shards],
                               input_split_sizes=[bl * t_r * d] * n, group=self.group)
        blocks = torch.split(recv, [bl * len(s) * d for s in self.shards])
        cat = torch.cat([blk.view(bl, len(s), d) for blk, s in zip(blocks, self.shards)], dim=1)
        to_global, _ = self._idx(cat.device)
        return cat.index_select(1, to_global)

    def backward(self, grad: torch.Tensor, scale: float | None = None) -> torch.Tensor:
        """[B/N, T, D] gradients of this rank's examples -> [B, T_r, D] for this rank's tables."""
        bl, t, d = grad.shape
        n = self.world
        _, to_blocks = self._idx(grad.device)
        blocks = grad.index_select(1, to_blocks)            # [B/N, T, D] in block (owner) order
        send = torch.cat([c.reshape(-1) for c in torch.split(blocks, [len(s) for s in self.shards], dim=1)])
        if scale is not None:
            send.mul_(scale)
        t_r = len(self.local_tables)
        recv = torch.empty(n * bl * t_r * d, dtype=grad.dtype, device=grad.device)
        dist.all_to_all_single(recv, send, output_split_sizes=[bl * t_r * d] * n,
                               input_split_sizes=[bl * len(s) * d for s in self.shards], group=self.group)
        return recv.view(n * bl, t_r, d)


def allreduce_mean_(tensors, world: int, group=None) -> None:
    """Average gradients across ranks in one flat all-reduce."""
    if world == 1 or not tensors:
        return
    flat = torch.cat([t.reshape(-1) for t in tensors])
    dist.all_reduce(flat, group=group)
    flat.div_(world)
    off = 0
    for t in tensors:
        k = t.numel()
        t.copy_(flat[off:off + k].view_as(t))
        off += k


class PeerExchange:
    """The exchange over NVLink peer memory (csrc/peer.cu): no NCCL on the
    embedding data path.  Every rank owns two [bl, T, D] f32 buffers, shared
    with CUDA IPC handles exchanged over torch.distributed:

    * ``rows``  -- the table owners' EmbeddingBag forward stores pooled rows
      straight into the example owner's buffer, at the row's global table
      column (the dense step reads it in place);
    * ``grads`` -- the example owner writes its pooled-row gradients here and
      the table owners' reduce-by-key backward loads them over NVLink.

    Two flag barriers per iteration (rows ready, gradients ready) order the
    phases and protect buffer reuse.  Same interface fields as
    EmbeddingExchange (shards, local_tables, world, rank, num_tables)."""

    def __init__(self, num_tables: int, dim: int, rank: int, world: int, bl: int, group=None, shards=None):
        import ctypes as C

        from . import _lib as L
        from .device import _wrap_device

        self.num_tables, self.dim, self.rank, self.world, self.bl, self.group = num_tables, dim, rank, world, bl, group
        self.shards = shards if shards is not None else table_shards(num_tables, world)
        self.local_tables = self.shards[rank]
        lib = L.lib()
        self._lib, self._L = lib, L
        nbytes = bl * num_tables * dim * 4
        own, handles = {}, {}
        for name, size in (("rows", nbytes), ("grads", nbytes), ("flags", 4 * world)):
            ptr, h = C.c_void_p(), (C.c_uint8 * 64)()
            L.check(lib.bp_ipc_alloc(size, C.byref(ptr), h), "bp_ipc_alloc")
            own[name], handles[name] = ptr.value, bytes(h)
        self._own = own
        gathered = [None] * world
        dist.all_gather_object(gathered, handles, group=group)
        self._opened = []
        peers = {name: [] for name in own}
        for q in range(world):
            for name in own:
                if q == rank:
                    peers[name].append(own[name])
                    continue
                ptr = C.c_void_p()
                buf = (C.c_uint8 * 64).from_buffer_copy(gathered[q][name])
                L.check(lib.bp_ipc_open(buf, C.byref(ptr)), "bp_ipc_open")
                self._opened.append(ptr.value)
                peers[name].append(ptr.value)
        dev = torch.device("cuda", torch.cuda.current_device())
        self._d_rows = torch.tensor(peers["rows"], dtype=torch.int64, device=dev)
        self._d_grads = torch.tensor(peers["grads"], dtype=torch.int64, device=dev)
        self._d_flags = torch.tensor(peers["flags"], dtype=torch.int64, device=dev)
        self._d_cols = torch.tensor(self.local_tables, dtype=torch.int32, device=dev)
        t_r = len(self.local_tables)
        self.rows_x = L.PeerXchg(world, rank, bl, num_tables, t_r, L.ptr(self._d_cols), L.ptr(self._d_rows),
                                 L.ptr(self._d_flags), own["flags"])
        self.grads_x = L.PeerXchg(world, rank, bl, num_tables, t_r, L.ptr(self._d_cols), L.ptr(self._d_grads),
                                  L.ptr(self._d_flags), own["flags"])
        self.rows = _wrap_device(own["rows"], torch.float32, bl * num_tables * dim).view(bl, num_tables, dim)
        self.grads = _wrap_device(own["grads"], torch.float32, bl * num_tables * dim).view(bl, num_tables, dim)
        self.epoch = 0
        dist.barrier(group=group)  # every rank opened every handle

    def barrier(self, stream) -> None:
        """Device-side barrier of all ranks on `stream` (bounded spin)."""
        import ctypes as C

        self.epoch += 1
        L = self._L
        L.check(self._lib.bp_peer_barrier(L.Context.get().handle, C.byref(self.rows_x), self.epoch,
                                          L.stream_ptr(stream)), "bp_peer_barrier")

    def close(self) -> None:
        if getattr(self, "_own", None) is None:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        for p in self._opened:
            self._lib.bp_ipc_close(p)
        dist.barrier(group=self.group)
        for p in self._own.values():
            self._lib.bp_ipc_free(p)
        self._own = None
