"""DLRM mode: the BagPipe embedding path feeding a real dense model.

The reference replaces the model with a gradient stub (reference SPEC.md:8,
trainer.py:1-8); the north star asks for the EmbeddingBag forward/backward
with SGD/Adagrad on cached rows in front of DLRM's dense MLPs.  The dense
part (bottom MLP, pairwise-dot interaction, top MLP) stays in PyTorch -- it
is not the hot path -- and runs on the engine's compute stream between the
two native halves of an iteration:

    bp_engine_dlrm_forward   apply plan, lookup, EmbeddingBag gather -> pooled
    (PyTorch)                dense model forward / backward, MLP SGD step
    bp_engine_dlrm_backward  EmbeddingBag backward + SGD/Adagrad in place,
                             dirty marking, eviction, counters

Everything else (planner, prefetch, gate, write-back, report) is the
pipelined engine of engine.py.  No reference counterpart exists, so parity is
against a PyTorch fp32 CPU model (tests/test_gpu_dlrm.py, rel 1e-5).
"""

from __future__ import annotations

import copy
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch
from torch import nn

from . import _lib as L
from .errors import ConfigurationError

BP_OPT_SGD = 0
BP_OPT_ADAGRAD = 1


def mlp(sizes, last_act: bool, in_pad: int = 0) -> nn.Sequential:
    """Linear+ReLU stack.  ``in_pad`` extra input features (always fed zeros)
    widen the first layer to a multiple of 8 so bf16 GEMMs hit aligned
    tensor-core kernels; their weight columns start at zero and, with zero
    inputs, get zero gradient, so the model equals the unpadded one (the
    live columns keep the unpadded layer's init)."""
    layers = []
    for i in range(len(sizes) - 1):
        fan_in = sizes[i] + (in_pad if i == 0 else 0)
        lin = nn.Linear(fan_in, sizes[i + 1])
        if fan_in != sizes[i]:
            ref = nn.Linear(sizes[i], sizes[i + 1])
            with torch.no_grad():
                lin.weight.zero_()
                lin.weight[:, :sizes[i]].copy_(ref.weight)
                lin.bias.copy_(ref.bias)
        layers.append(lin)
        if i < len(sizes) - 2 or last_act:
            layers.append(nn.ReLU())
    return nn.Sequential(*layers)


class _Interact(torch.autograd.Function):
    """Fused DLRM interaction (csrc/interact.cu): [x | tril(z z^T) | 0-pad]."""

    @staticmethod
    def forward(ctx, x, emb, out_stride: int, grad_rows=None):
        x = x.contiguous()
        emb = emb.contiguous().float()
        b, t, d = emb.shape
        bf = x.dtype == torch.bfloat16
        out = torch.empty((b, out_stride), dtype=x.dtype, device=x.device)
        L.check(L.lib().bp_dlrm_interact_forward(L.ptr(x), int(bf), L.ptr(emb), b, t, d, L.ptr(out), int(bf),
                                                 out_stride, L.stream_ptr()), "bp_dlrm_interact_forward")
        ctx.save_for_backward(x, emb)
        ctx.out_stride = out_stride
        ctx.grad_rows = grad_rows
        return out

    @staticmethod
    def backward(ctx, gout):
        x, emb = ctx.saved_tensors
        b, t, d = emb.shape
        gout = gout.contiguous()
        gx = torch.empty_like(x)
        gemb = torch.empty_like(emb)
        # grad_rows (optional): row of (b, t) in gemb -- the EmbeddingBag's
        # key-sorted order, so the embedding backward streams it
        rows = ctx.grad_rows
        L.check(L.lib().bp_dlrm_interact_backward_rows(L.ptr(x), int(x.dtype == torch.bfloat16), L.ptr(emb),
                                                       L.ptr(gout), int(gout.dtype == torch.bfloat16), b, t, d,
                                                       ctx.out_stride, L.ptr(gx), L.ptr(gemb),
                                                       L.ptr(rows) if rows is not None else None, L.stream_ptr()),
                "bp_dlrm_interact_backward_rows")
        return gx, gemb, None, None


def _pad8(n: int) -> int:
    return (-n) % 8


class _LinearAct(torch.autograd.Function):
    """y = relu?(x W^T + b) on the GPU: bias (and ReLU) in the cuBLASLt GEMM
    epilogue (torch._addmm_activation), and in backward the bias gradient as
    a GEMV against a ones vector instead of a column reduction over the
    batch (measured 23 us per layer at B = 16,384 as a reduction)."""

    _ones: dict = {}

    @staticmethod
    def forward(ctx, x, w, b, relu: bool):
        y = torch._addmm_activation(b, x, w.t(), use_gelu=False) if relu else torch.addmm(b, x, w.t())
        ctx.save_for_backward(x, w, y if relu else None)
        ctx.relu = relu
        return y

    @staticmethod
    def backward(ctx, g):
        x, w, y = ctx.saved_tensors
        if ctx.relu:
            g = torch.ops.aten.threshold_backward(g, y, 0)
        key = (g.shape[0], g.dtype, g.device)
        ones = _LinearAct._ones.get(key)
        if ones is None:
            ones = _LinearAct._ones[key] = torch.ones(g.shape[0], dtype=g.dtype, device=g.device)
        return g @ w, g.t() @ x, torch.mv(g.t(), ones), None


def _run_mlp(seq: nn.Sequential, x: torch.Tensor) -> torch.Tensor:
    """nn.Sequential of Linear (+ ReLU) through _LinearAct on CUDA tensors."""
    if not x.is_cuda:
        return seq(x)
    mods = list(seq)
    i = 0
    while i < len(mods):
        lin = mods[i]
        relu = i + 1 < len(mods) and isinstance(mods[i + 1], nn.ReLU)
        x = _LinearAct.apply(x.to(lin.weight.dtype), lin.weight, lin.bias, relu)
        i += 2 if relu else 1
    return x


class DLRMDense(nn.Module):
    """Bottom MLP -> pairwise dot interaction with the T pooled embeddings -> top MLP."""

    def __init__(self, num_dense: int, num_tables: int, dim: int, bottom=(512, 256, 64), top=(1024, 1024, 512, 256)):
        super().__init__()
        self.num_tables, self.dim, self.num_dense = num_tables, dim, num_dense
        self.dense_pad = _pad8(num_dense)
        self.bottom = mlp((num_dense,) + tuple(bottom) + (dim,), last_act=True, in_pad=self.dense_pad)
        n = num_tables + 1
        self.pairs = n * (n - 1) // 2
        self.top_pad = _pad8(self.pairs + dim)
        self.top = mlp((self.pairs + dim,) + tuple(top) + (1,), last_act=False, in_pad=self.top_pad)
        li, lj = torch.tril_indices(n, n, offset=-1)
        # strictly-lower-triangle entries of the flattened [n, n] Gram matrix;
        # index_select's backward is a plain index_add (no sort), unlike the
        # advanced-indexing form zz[:, li, lj]
        self.register_buffer("tril_flat", li * n + lj, persistent=False)

    def forward(self, dense: torch.Tensor, pooled: torch.Tensor, grad_rows: torch.Tensor | None = None) -> torch.Tensor:
        """grad_rows (CUDA only, int32 [B*T]): store the gradient of pooled row
        (b, t) at row grad_rows[b*T + t] of pooled.grad (a permutation)."""
        if dense.shape[1] == self.num_dense and self.dense_pad:
            dense = nn.functional.pad(dense, (0, self.dense_pad))
        x = _run_mlp(self.bottom, dense)                      # [B, D]
        if pooled.is_cuda:
            # fused CUDA interaction (no eager fallback on the GPU path)
            return _run_mlp(self.top, _Interact.apply(x, pooled, self.pairs + self.dim + self.top_pad,
                                                      grad_rows)).squeeze(1)
        z = torch.cat([x.unsqueeze(1).to(pooled.dtype), pooled], dim=1)  # [B, T+1, D]
        zz = torch.bmm(z, z.transpose(1, 2))                  # [B, T+1, T+1]
        inter = zz.flatten(1).index_select(1, self.tril_flat)  # [B, pairs]
        feats = [x.to(inter.dtype), inter]
        if self.top_pad:
            feats.append(inter.new_zeros((inter.shape[0], self.top_pad)))
        return self.top(torch.cat(feats, dim=1)).squeeze(1)


@dataclass
class DLRMConfig:
    """Dense model + embedding optimizer for DLRM mode."""

    emb_optimizer: str = "sgd"   # "sgd" | "adagrad"
    emb_lr: float = 0.01
    adagrad_eps: float = 1e-10
    mlp_lr: float = 0.01
    bottom: tuple = (512, 256, 64)
    top: tuple = (1024, 1024, 512, 256)
    mlp_dtype: str = "fp32"      # "fp32" | "bf16" (autocast for the dense MLPs only)
    seed: int = 0
    cuda_graph: bool = True      # replay the dense step (fwd + bwd + SGD) as one captured CUDA graph
    sorted_grad: bool = True     # interaction backward stores pooled-row gradients in key-sorted order (1 GPU)

    def __post_init__(self):
        if self.emb_optimizer not in ("sgd", "adagrad"):
            raise ConfigurationError("emb_optimizer must be 'sgd' or 'adagrad'")
        if self.mlp_dtype not in ("fp32", "bf16"):
            raise ConfigurationError("mlp_dtype must be 'fp32' or 'bf16'")

    @property
    def opt_code(self) -> int:
        return BP_OPT_ADAGRAD if self.emb_optimizer == "adagrad" else BP_OPT_SGD


class _MasterSGD:
    """SGD on fp32 master weights from the gradients of a bf16 compute copy,
    then the copy refreshed from the masters (mixed precision without
    autocast's per-layer casts)."""

    def __init__(self, master: list, lowp: list, lr: float):
        self.master, self.lowp, self.lr = master, lowp, lr

    def zero_grad(self, set_to_none: bool = True):
        for p in self.lowp:
            p.grad = None

    @torch.no_grad()
    def step(self):
        # one fused launch over every tensor (bp_dlrm_master_sgd): fp32 master
        # update from the bf16 gradient, then the bf16 copy refreshed
        if self.master[0].is_cuda and len(self.master) <= L.SGD_MAX_TENSORS:
            t = L.SgdTensors()
            t.n = len(self.master)
            for k, (m, p) in enumerate(zip(self.master, self.lowp)):
                t.master[k], t.lowp[k], t.grad[k] = m.data_ptr(), p.data_ptr(), p.grad.data_ptr()
                t.numel[k] = m.numel()
            L.check(L.lib().bp_dlrm_master_sgd(C.byref(t), float(np.float32(self.lr)), L.stream_ptr()),
                    "bp_dlrm_master_sgd")
            return
        for m, p in zip(self.master, self.lowp):
            m.add_(p.grad, alpha=-self.lr)
        torch._foreach_copy_(self.lowp, self.master)


class DLRMTrainer:
    """Runs the dense model between the two native halves of an iteration."""

    def __init__(self, dcfg: DLRMConfig, num_dense: int, num_tables: int, dim: int, model: DLRMDense | None = None,
                 exchange=None):
        """exchange: a hybrid.EmbeddingExchange for N > 1 (model-parallel tables,
        data-parallel MLPs); None on one GPU."""
        self.dcfg = dcfg
        self.dim = dim
        self.exchange = exchange
        torch.manual_seed(dcfg.seed)
        self.model = (model or DLRMDense(num_dense, num_tables, dim, dcfg.bottom, dcfg.top)).cuda()
        if dcfg.mlp_dtype == "bf16":
            # bf16 compute copy of the fp32 master model: no per-step casts
            self.compute_model = copy.deepcopy(self.model).to(torch.bfloat16)
            self.opt = _MasterSGD(list(self.model.parameters()), list(self.compute_model.parameters()), dcfg.mlp_lr)
        else:
            self.compute_model = self.model
            self.opt = torch.optim.SGD(self.model.parameters(), lr=dcfg.mlp_lr)
        self.losses: list = []
        self.async_peer = os.environ.get("BAGPIPE_B200_ASYNC_PEER", "1") == "1"
        # single GPU, dims the sorted backward supports: gradients in key-sorted order
        self._sorted = dcfg.sorted_grad and (exchange is None or exchange.world <= 1) and dim in (4, 8, 16, 32)
        self._dense_dev: dict = {}
        self._graphs: dict = {}

    def row_width(self) -> int:
        """Width of a stored row: weights (+ Adagrad accumulators)."""
        return 2 * self.dim if self.dcfg.opt_code == BP_OPT_ADAGRAD else self.dim

    def _pad_dense(self, dense: torch.Tensor) -> torch.Tensor:
        """Dense features padded to the bottom MLP's aligned input width once,
        so the per-step copy into the graph's static input is contiguous (a
        strided [B, 13] -> [B, 16] copy runs as a slow 2D memcpy)."""
        pad = self.model.dense_pad
        if pad and dense.shape[1] == self.model.num_dense:
            dense = nn.functional.pad(dense, (0, pad))
        return dense.contiguous()

    def set_device_dense(self, pos: int, dense: torch.Tensor, labels: torch.Tensor) -> None:
        self._dense_dev[pos] = (self._pad_dense(dense), labels)

    def can_split(self) -> bool:
        """Single GPU and the NVLink peer exchange: the iteration is enqueued by
        train_begin and its counters read later by the engine
        (bp_engine_train_end), so the host prepares the next iteration while
        this one runs (the peer exchange's device barriers keep the ranks'
        buffer reuse ordered across iterations)."""
        ex = self.exchange
        return ex is None or ex.world <= 1 or (hasattr(ex, "rows_x") and self.async_peer)

    def train(self, pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain, res) -> None:
        if self.exchange is not None and self.exchange.world > 1:
            if hasattr(self.exchange, "rows_x"):
                return self._train_peer(pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain, res)
            return self._train_hybrid(pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain, res)
        self.train_begin(pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain)
        L.check(pipe.lib.bp_engine_train_end(pipe.eng, C.byref(res)), "bp_engine_train_end")

    def train_begin(self, pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain) -> None:
        if self.exchange is not None and self.exchange.world > 1:
            return self._train_peer(pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain, None)
        lib = pipe.lib
        batch = pipe.batches[pos]
        n_occ = int(batch.packed_occurrences()[0].size)
        b = batch.num_examples
        t = n_occ // max(b, 1)
        stream = pipe.stream
        with torch.cuda.stream(stream):
            dense, labels = self._inputs(pos, batch, slice(None))
            g = self._graph(b, t, dense.shape[1]) if self.dcfg.cuda_graph else None
            # the native forward writes the pooled rows straight into the
            # graph's static input (or a fresh leaf in eager mode)
            pooled = g["emb"] if g is not None else torch.empty((b, t, self.dim), dtype=torch.float32, device="cuda")
            L.check(lib.bp_engine_dlrm_forward(pipe.eng, pos, plan.slot, nxt, skip_key, has_skip, self.dim,
                                               L.ptr(pooled)), "bp_engine_dlrm_forward")
            rows = None
            if self._sorted:
                rows = g["rows"] if g is not None else torch.empty(b * t, dtype=torch.int32, device="cuda")
                L.check(lib.bp_engine_dlrm_grad_rows(pipe.eng, pos, L.ptr(rows)), "bp_engine_dlrm_grad_rows")
            if g is not None:
                g["dense"][:, :dense.shape[1]].copy_(dense)
                g["labels"].copy_(labels)
                g["graph"].replay()
                if g["step"] is not None:
                    g["step"].replay()
                grad = g["grad"]
                self.losses.append(g["loss"].detach().clone())
            else:
                emb = pooled.requires_grad_(True)
                loss = self._loss(dense, emb, labels, rows)
                self.opt.zero_grad(set_to_none=True)
                loss.backward()
                self.opt.step()
                grad = emb.grad.contiguous()
                self.losses.append(loss.detach())
            L.check(lib.bp_engine_dlrm_backward_begin(pipe.eng, pos, plan.slot, L.ptr(grad), int(self._sorted),
                                                      self.dim, self.dcfg.opt_code,
                                                      float(np.float32(self.dcfg.emb_lr)),
                                                      float(np.float32(self.dcfg.adagrad_eps)), chunk, drain),
                    "bp_engine_dlrm_backward_begin")

    def _inputs(self, pos, batch, sl):
        dev = self._dense_dev.pop(pos, None)
        if dev is None:
            dense = torch.from_numpy(np.ascontiguousarray(batch.dense[sl], dtype=np.float32)).to("cuda")
            labels = torch.from_numpy(np.ascontiguousarray(batch.labels[sl], dtype=np.float32)).to("cuda")
            return self._pad_dense(dense), labels
        dense, labels = dev
        return dense[sl], labels[sl]

    def _backward(self, pipe, pos, plan, grad, chunk, drain, res) -> None:
        """Synchronous EmbeddingBag backward (hybrid NCCL path; occurrence-order gradients)."""
        L.check(pipe.lib.bp_engine_dlrm_backward(pipe.eng, pos, plan.slot, L.ptr(grad), self.dim, self.dcfg.opt_code,
                                                 float(np.float32(self.dcfg.emb_lr)),
                                                 float(np.float32(self.dcfg.adagrad_eps)), chunk, drain,
                                                 C.byref(res)), "bp_engine_dlrm_backward")

    def _train_hybrid(self, pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain, res) -> None:
        """N > 1 (hybrid.py): this rank's tables over the global batch ->
        all-to-all -> the dense step on this rank's B/N examples -> reverse
        all-to-all (x 1/N) -> mean all-reduce of MLP gradients -> SGD."""
        from .hybrid import allreduce_mean_

        ex = self.exchange
        lib = pipe.lib
        batch = pipe.batches[pos]
        b = batch.num_examples
        t_local = int(batch.packed_occurrences()[0].size) // max(b, 1)
        bl = b // ex.world
        sl = slice(ex.rank * bl, (ex.rank + 1) * bl)
        with torch.cuda.stream(pipe.stream):
            dense, labels = self._inputs(pos, batch, sl)
            pooled = torch.empty((b, t_local, self.dim), dtype=torch.float32, device="cuda")
            L.check(lib.bp_engine_dlrm_forward(pipe.eng, pos, plan.slot, nxt, skip_key, has_skip, self.dim,
                                               L.ptr(pooled)), "bp_engine_dlrm_forward")
            emb_in = ex.forward(pooled)
            g = self._graph(bl, ex.num_tables, dense.shape[1], with_step=False) if self.dcfg.cuda_graph else None
            if g is not None:
                g["emb"].detach().copy_(emb_in)
                g["dense"][:, :dense.shape[1]].copy_(dense)
                g["labels"].copy_(labels)
                g["graph"].replay()
                grad, loss = g["grad"], g["loss"]
            else:
                emb = emb_in.requires_grad_(True)
                loss = self._loss(dense, emb, labels)
                self.opt.zero_grad(set_to_none=True)
                loss.backward()
                grad = emb.grad.contiguous()
            self.losses.append(loss.detach().clone())
            allreduce_mean_([p.grad for p in self.compute_model.parameters()], ex.world)
            if g is not None and g["step"] is not None:
                g["step"].replay()
            else:
                self.opt.step()
            grad_local = ex.backward(grad, scale=1.0 / ex.world)
            self._backward(pipe, pos, plan, grad_local, chunk, drain, res)

    def _train_peer(self, pipe, pos, plan, nxt, skip_key, has_skip, chunk, drain, res) -> None:
        """N > 1 over NVLink peer memory (hybrid.PeerExchange): the forward
        stores pooled rows into the example owners' buffers, a device
        barrier, the dense step reading its buffer in place, gradients into
        the local gradient buffer, a barrier, the mean all-reduce of MLP
        gradients + SGD, and the table owners' backward loading the
        gradients over NVLink (x 1/N)."""
        import ctypes as C

        from .hybrid import allreduce_mean_

        ex = self.exchange
        lib = pipe.lib
        batch = pipe.batches[pos]
        bl = batch.num_examples // ex.world
        sl = slice(ex.rank * bl, (ex.rank + 1) * bl)
        stream = pipe.stream
        with torch.cuda.stream(stream):
            dense, labels = self._inputs(pos, batch, sl)
            L.check(lib.bp_engine_dlrm_forward_peer(pipe.eng, pos, plan.slot, nxt, skip_key, has_skip, self.dim,
                                                    C.byref(ex.rows_x)), "bp_engine_dlrm_forward_peer")
            ex.barrier(stream)
            g = self._graph(bl, ex.num_tables, dense.shape[1], with_step=False, emb=ex.rows) \
                if self.dcfg.cuda_graph else None
            if g is not None:
                g["dense"][:, :dense.shape[1]].copy_(dense)
                g["labels"].copy_(labels)
                g["graph"].replay()
                grad, loss = g["grad"], g["loss"]
            else:
                emb = ex.rows.detach().requires_grad_(True)
                loss = self._loss(dense, emb, labels)
                self.opt.zero_grad(set_to_none=True)
                loss.backward()
                grad = emb.grad
            ex.grads.copy_(grad)
            ex.barrier(stream)
            self.losses.append(loss.detach().clone())
            allreduce_mean_([p.grad for p in self.compute_model.parameters()], ex.world)
            if g is not None and g["step"] is not None:
                g["step"].replay()
            else:
                self.opt.step()
            args = (pipe.eng, pos, plan.slot, C.byref(ex.grads_x), 1.0 / ex.world, self.dim, self.dcfg.opt_code,
                    float(np.float32(self.dcfg.emb_lr)), float(np.float32(self.dcfg.adagrad_eps)), chunk, drain)
            if res is None:  # asynchronous: counters read by the engine later
                L.check(lib.bp_engine_dlrm_backward_peer_begin(*args), "bp_engine_dlrm_backward_peer_begin")
            else:
                L.check(lib.bp_engine_dlrm_backward_peer(*args, C.byref(res)), "bp_engine_dlrm_backward_peer")

    def _loss(self, dense, emb, labels, grad_rows=None):
        logits = self.compute_model(dense, emb, grad_rows).float()
        return nn.functional.binary_cross_entropy_with_logits(logits, labels)

    def _graph(self, b: int, t: int, n_dense: int, with_step: bool = True, emb=None) -> dict:
        """The dense step for a (B, T) batch shape, captured once as a CUDA
        graph over static input buffers (the pooled embeddings, dense
        features, labels).  Replaying it costs one launch instead of ~100
        eager kernel launches from Python.  Warm-up passes before capture run
        forward+backward only, so the model's parameters are untouched."""
        key = (b, t, n_dense, with_step, None if emb is None else emb.data_ptr())
        g = self._graphs.get(key)
        if g is not None:
            return g
        dev = "cuda"
        own_emb = emb is None
        # static input: a fresh buffer, or caller memory read in place (the
        # peer exchange's row buffer)
        emb = torch.zeros((b, t, self.dim), dtype=torch.float32, device=dev, requires_grad=True) if emb is None \
            else emb.detach().requires_grad_(True)
        dense = torch.zeros((b, self.model.num_dense + self.model.dense_pad), dtype=torch.float32, device=dev)
        labels = torch.zeros((b,), dtype=torch.float32, device=dev)
        # sorted-gradient row map (filled per batch by bp_engine_dlrm_grad_rows
        # before each replay; identity for the warm-up passes)
        rows = torch.arange(b * t, dtype=torch.int32, device=dev) if (self._sorted and with_step and own_emb) \
            else None
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                self._loss(dense, emb, labels, rows).backward()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.opt.zero_grad(set_to_none=True)
        emb.grad = None
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="thread_local"):
            loss = self._loss(dense, emb, labels, rows)
            loss.backward()
            if with_step:
                self.opt.step()
            grad = emb.grad.contiguous()
        step = None
        if not with_step:
            # the SGD step as its own graph, replayed after the gradient all-reduce
            step = torch.cuda.CUDAGraph()
            with torch.cuda.graph(step, pool=graph.pool(), capture_error_mode="thread_local"):
                self.opt.step()
        g = {"graph": graph, "step": step if not with_step else None, "emb": emb, "dense": dense, "labels": labels,
             "loss": loss, "grad": grad, "rows": rows}
        self._graphs[key] = g
        return g

    def loss_history(self) -> list:
        return [float(x) for x in self.losses]
