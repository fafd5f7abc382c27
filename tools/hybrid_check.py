"""DLRM hybrid parallelism on N GPUs vs one-process PyTorch CPU training.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/hybrid_check.py \
      [sgd|adagrad] [peer|nccl]

Each rank runs the pipelined engine for its table shard (hybrid.py) with the
NCCL all-to-all exchange; rank 0 gathers the final tables and MLP weights
and compares them with tests/test_gpu_dlrm.cpu_reference.  Exit 0 = match.
"""

from __future__ import annotations

import copy
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main() -> int:
    opt_name = sys.argv[1] if len(sys.argv) > 1 else "sgd"
    kind = sys.argv[2] if len(sys.argv) > 2 else "peer"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    from test_gpu_dlrm import SCHEMA, _batches, cpu_reference

    from paper_2202_12429_b200.dlrm import DLRMConfig, DLRMDense
    from paper_2202_12429_b200.engine import EngineConfig, run_dlrm
    from paper_2202_12429_b200.hybrid import EmbeddingExchange, PeerExchange
    from paper_2202_12429_b200.shard import shard_batches

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.manual_seed(0)
    model = DLRMDense(SCHEMA.num_dense, SCHEMA.num_tables, SCHEMA.emb_dim, bottom=(64, 32), top=(64, 32))
    batches = _batches()
    lr, eps, seed = 0.05, 1e-10, 7
    if kind == "peer":
        ex = PeerExchange(SCHEMA.num_tables, SCHEMA.emb_dim, rank, world, 256 // world)
    else:
        ex = EmbeddingExchange(SCHEMA.num_tables, SCHEMA.emb_dim, rank, world)
    cfg = EngineConfig(cache_capacity=1200, batch_size=256, lookahead=3, num_shards=1, seed=seed, lr=lr)
    dcfg = DLRMConfig(emb_optimizer=opt_name, emb_lr=lr, mlp_lr=lr, adagrad_eps=eps, bottom=(64, 32), top=(64, 32))
    report, trainer = run_dlrm(cfg, SCHEMA, shard_batches(batches, ex.local_tables), dcfg, model=copy.deepcopy(model),
                               exchange=ex)
    table = report.final_store.table_view()
    base = SCHEMA.table_base()
    mine = {t: np.array(table[base[t]:base[t + 1], :SCHEMA.emb_dim]) for t in ex.local_tables}
    losses = torch.tensor(trainer.loss_history(), dtype=torch.float64, device="cuda")
    dist.all_reduce(losses)
    losses /= world
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    ok = True
    if rank == 0:
        want_losses, want_tables, want_model, want_ill = cpu_reference(batches, model, opt_name, lr, eps, seed)
        np.testing.assert_allclose(losses.cpu().numpy(), want_losses, rtol=1e-4)
        atol = 1e-4 if opt_name == "adagrad" else 1e-6
        got = {}
        for part in gathered:
            got.update(part)
        assert sorted(got) == list(range(SCHEMA.num_tables))
        for t in range(SCHEMA.num_tables):
            # Adagrad: components the reference stepped on a near-zero
            # accumulated gradient are order-sensitive (test_gpu_dlrm.py)
            well = np.ones(want_tables[t].shape, bool) if want_ill is None else ~want_ill[t]
            np.testing.assert_allclose(got[t][well], want_tables[t][well], rtol=1e-5, atol=atol, err_msg=f"table {t}")
            assert np.all(np.abs(got[t][~well] - want_tables[t][~well]) <= lr * len(batches) + 1e-6)
        for (name, p), (_, q) in zip(trainer.model.named_parameters(), want_model.named_parameters()):
            np.testing.assert_allclose(p.detach().cpu().numpy(), q.detach().numpy(), rtol=1e-4, atol=1e-6,
                                       err_msg=name)
        print(f"hybrid DLRM x{world} ({opt_name}, {kind} exchange) == single-process CPU training", flush=True)
    dist.barrier()
    if kind == "peer":
        ex.close()
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
