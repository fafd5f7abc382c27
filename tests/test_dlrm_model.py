"""DLRM dense model (CPU): the 8-aligned padding of the first bottom/top
layers and the flattened-index interaction compute exactly the unpadded
DLRM (bottom MLP -> pairwise dots -> top MLP), and padded weight columns
never move under SGD."""

from __future__ import annotations

import torch

from paper_2202_12429_b200.dlrm import DLRMDense


def _unpadded_forward(m: DLRMDense, dense, pooled):
    x = dense
    for layer in m.bottom:
        if isinstance(layer, torch.nn.Linear):
            w = layer.weight[:, :x.shape[1]]
            x = x @ w.T + layer.bias
        else:
            x = torch.relu(x)
    z = torch.cat([x.unsqueeze(1), pooled], dim=1)
    n = z.shape[1]
    li, lj = torch.tril_indices(n, n, offset=-1)
    inter = torch.bmm(z, z.transpose(1, 2))[:, li, lj]
    h = torch.cat([x, inter], dim=1)
    for layer in m.top:
        if isinstance(layer, torch.nn.Linear):
            h = h @ layer.weight[:, :h.shape[1]].T + layer.bias
        else:
            h = torch.relu(h)
    return h.squeeze(1)


def test_padded_dlrm_equals_unpadded():
    torch.manual_seed(0)
    m = DLRMDense(13, 26, 16, bottom=(32, 16), top=(32, 8)).double()
    assert m.dense_pad == 3 and (m.pairs + 16 + m.top_pad) % 8 == 0
    dense = torch.randn(64, 13, dtype=torch.float64)
    pooled = torch.randn(64, 26, 16, dtype=torch.float64)
    torch.testing.assert_close(m(dense, pooled), _unpadded_forward(m, dense, pooled), rtol=1e-12, atol=1e-12)
    first_bottom = m.bottom[0].weight
    first_top = m.top[0].weight
    assert torch.all(first_bottom[:, 13:] == 0) and torch.all(first_top[:, m.pairs + 16:] == 0)
    opt = torch.optim.SGD(m.parameters(), lr=0.1)
    m(dense, pooled).sum().backward()
    opt.step()
    assert torch.all(first_bottom[:, 13:] == 0) and torch.all(first_top[:, m.pairs + 16:] == 0)


def test_interaction_gradient_matches_advanced_indexing():
    torch.manual_seed(1)
    m = DLRMDense(13, 5, 8, bottom=(16,), top=(16,)).double()
    dense = torch.randn(16, 13, dtype=torch.float64)
    pooled = torch.randn(16, 5, 8, dtype=torch.float64, requires_grad=True)
    m(dense, pooled).sum().backward()
    g1 = pooled.grad.clone()
    pooled.grad = None
    _unpadded_forward(m, dense, pooled).sum().backward()
    torch.testing.assert_close(g1, pooled.grad, rtol=1e-12, atol=1e-12)
