"""DLRM mode at the Criteo-Kaggle shape (BASELINE.json configs[1]) against a
PyTorch fp32 CPU model: 26 tables / 33,762,577 rows, D=16, batch 16,384,
the bench's MLPs (13-512-256-64-16 / 367-1024-1024-512-256-1) in fp32, HBM
cache 1% of rows, lookahead 2 (evictions mid-run), 4 iterations through the pipelined
engine (plans, prefetch, eviction, write-back, EmbeddingBag fwd/bwd + SGD in
place).  No reference counterpart exists for the model (the
reference trainer is a stub), so the oracle is dense PyTorch fp32 training;
tolerance rel 1e-5 (north star) on the loss, on every iteration's pooled
outputs and on every touched table row afterwards.

The CPU model holds only the rows the trace touches (plain SGD leaves an
untouched row exactly unchanged), initialised with the reference's
functional init (oracle.init_rows = store.py:29-42)."""

from __future__ import annotations

import copy

import numpy as np
import pytest
import torch

from oracle import bagpipe_oracle as O
from paper_2202_12429_b200.traces import Schema, ZipfSpec, batchify_columns, generate_columns

pytestmark = pytest.mark.gpu

CK_ROWS = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27, 14992, 5461306,
           10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)
SCHEMA = Schema(26, CK_ROWS, 13, 16)
RTOL = 1e-5


def test_ck_shape_dlrm_fp32_matches_cpu():
    from paper_2202_12429_b200.dlrm import DLRMConfig, DLRMDense
    from paper_2202_12429_b200.engine import EngineConfig, run_dlrm

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    iters, batch, seed, lr = 4, 16384, 11, 0.05
    rows, labels, dense = generate_columns(ZipfSpec(SCHEMA, 1.05, iters * batch, 1))
    batches = batchify_columns(rows, labels, dense, batch)
    torch.manual_seed(0)
    model = DLRMDense(SCHEMA.num_dense, SCHEMA.num_tables, SCHEMA.emb_dim)

    # ---- CPU fp32 reference over the touched rows only
    T, D = SCHEMA.num_tables, SCHEMA.emb_dim
    touched = [np.unique(rows[:, t]) for t in range(T)]
    tables = [torch.nn.Parameter(torch.from_numpy(O.init_rows(seed, np.full(u.size, t), u, D))) for t, u in
              enumerate(touched)]
    cpu_model = copy.deepcopy(model)
    mopt = torch.optim.SGD(cpu_model.parameters(), lr=lr)
    eopt = torch.optim.SGD(tables, lr=lr)
    want_loss, want_pooled = [], []
    torch.set_num_threads(max(1, torch.get_num_threads()))
    for b in batches:
        local = [torch.from_numpy(np.searchsorted(touched[t], b.rows[:, t])) for t in range(T)]
        emb = torch.stack([tables[t][local[t]] for t in range(T)], dim=1)
        want_pooled.append(emb.detach().numpy().copy())
        logits = cpu_model(torch.from_numpy(np.ascontiguousarray(b.dense, dtype=np.float32)), emb)
        loss = torch.nn.functional.binary_cross_entropy_with_logits(logits, torch.from_numpy(
            b.labels.astype(np.float32)))
        mopt.zero_grad()
        eopt.zero_grad()
        loss.backward()
        mopt.step()
        eopt.step()
        want_loss.append(loss.item())

    # ---- the pipelined GPU engine, eager dense step (pooled rows observable)
    cap = SCHEMA.total_rows // 100
    cfg = EngineConfig(cache_capacity=cap, batch_size=batch, lookahead=2, num_shards=1, seed=seed, lr=lr)
    dcfg = DLRMConfig(emb_optimizer="sgd", emb_lr=lr, mlp_lr=lr, mlp_dtype="fp32", cuda_graph=False)
    from paper_2202_12429_b200 import dlrm as D_

    got_pooled = []
    orig = D_.DLRMTrainer._loss

    def spy(self, dense, emb, labels, grad_rows=None):
        got_pooled.append(emb.detach().cpu().numpy().copy())
        return orig(self, dense, emb, labels, grad_rows)

    D_.DLRMTrainer._loss = spy
    try:
        report, trainer = run_dlrm(cfg, SCHEMA, batches, dcfg, model=copy.deepcopy(model))
    finally:
        D_.DLRMTrainer._loss = orig
    got_loss = trainer.loss_history()
    assert len(got_loss) == iters and len(got_pooled) == iters
    np.testing.assert_allclose(got_loss, want_loss, rtol=RTOL)
    for i in range(iters):
        np.testing.assert_allclose(got_pooled[i], want_pooled[i], rtol=RTOL, atol=1e-7, err_msg=f"pooled it {i}")
    table = report.final_store.table_view()
    base = SCHEMA.table_base()
    for t in range(T):
        got = table[base[t] + touched[t], :D]
        np.testing.assert_allclose(got, tables[t].detach().numpy(), rtol=RTOL, atol=1e-7, err_msg=f"table {t}")
    assert report.totals["dirty_evictions"] > 0
