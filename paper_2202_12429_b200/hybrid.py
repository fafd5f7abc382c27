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

    def __init__(self, num_tables: int, dim: int, rank: int, world: int, group=None):
        self.num_tables, self.dim, self.rank, self.world, self.group = num_tables, dim, rank, world, group
        self.shards = table_shards(num_tables, world)
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
