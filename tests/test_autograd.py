"""Tape integration: SLA2AttentionFunction / SLA2Attention as an autograd
node (Tape::sla2_attention, tape.hpp:263-286). The device gradients are checked against
torch.autograd of an independent dense float64 restatement of the SLA2 forward with the same
(bit-exact) routing mask: out = a softmax_masked(Q K~^T / sqrt d) V + (1 - a) phi(Q) H_c / den."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dense_sla2(q, k, v, rho, mask, bq, bk, smooth=True):
    import torch
    n, d = q.shape
    kt = k - k.mean(dim=0, keepdim=True) if smooth else k
    qb = torch.arange(n, device=q.device) // bq
    kb = torch.arange(n, device=q.device) // bk
    keep = mask[qb][:, kb].bool()
    s = (q @ kt.T) / np.sqrt(d)
    p = torch.softmax(s.masked_fill(~keep, float("-inf")), dim=1)
    o_s = p @ v
    lin = (torch.softmax(q, dim=1) @ torch.softmax(kt, dim=1).T).masked_fill(keep, 0.0)
    o_l = (lin @ v) / lin.sum(dim=1, keepdim=True)
    full = mask.bool().all(dim=1)[qb]
    a = torch.sigmoid(rho[qb]).clamp(torch.finfo(torch.float64).tiny, 1 - torch.finfo(torch.float64).eps / 2)
    a = torch.where(full, torch.ones_like(a), a)[:, None]
    o_l = torch.where(full[:, None], torch.zeros_like(o_l), o_l)
    return a * o_s + (1 - a) * o_l


@pytest.mark.parametrize("N,d,bq,bk,kp,smooth", [(512, 64, 64, 64, 25.0, True), (256, 32, 32, 64, 40.0, False)])
def test_autograd_node_matches_dense_autograd(cuda, N, d, bq, bk, kp, smooth):
    import torch
    import paper_2602_12675_b200 as sla2
    from paper_2602_12675_b200.autograd import SLA2Attention
    B, H = 2, 2
    torch.manual_seed(0)
    layer = SLA2Attention(H, N, d, bq=bq, bk=bk, k_percent=kp, smooth=smooth, device=cuda)
    q, k, v = (torch.randn((B, H, N, d), device=cuda, requires_grad=True) for _ in range(3))
    w = torch.randn((B, H, N, d), device=cuda)
    out = layer(q, k, v)
    (out * w).sum().backward()
    mask = layer.last_mask
    drho_ref = torch.zeros_like(layer.rho, dtype=torch.float64)
    for b in range(B):
        for h in range(H):
            q64, k64, v64 = (x.detach()[b, h].double().requires_grad_() for x in (q, k, v))
            rho64 = layer.rho.detach()[h].double().requires_grad_()
            ref = _dense_sla2(q64, k64, v64, rho64, mask[b, h], bq, bk, smooth)
            assert float((ref.detach() - out.detach()[b, h].double()).abs().max()) <= 1e-4 * float(ref.detach().abs().max())
            (ref * w[b, h].double()).sum().backward()
            for got, want, name in ((q.grad[b, h], q64.grad, "dq"), (k.grad[b, h], k64.grad, "dk"),
                                    (v.grad[b, h], v64.grad, "dv")):
                err = float((got.double() - want).abs().max() / want.abs().max())
                assert err <= 1e-4, (name, b, h, err)
            drho_ref[h] += rho64.grad
    err = float((layer.rho.grad.double() - drho_ref).abs().max() / max(float(drho_ref.abs().max()), 1e-30))
    assert err <= 1e-4, ("drho", err)
    assert isinstance(sla2.CapturedForward, type)


def test_autograd_rejects_bf16(cuda):
    import torch
    import paper_2602_12675_b200 as sla2
    from paper_2602_12675_b200.autograd import sla2_attention
    x = torch.zeros((1, 1, 256, 64), device=cuda, dtype=torch.bfloat16)
    with pytest.raises(sla2.ContractError):
        sla2_attention(x, x, x, torch.zeros((1, 4), device=cuda), torch.eye(64, device=cuda)[None],
                       torch.eye(64, device=cuda)[None])
