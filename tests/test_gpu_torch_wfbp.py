"""Autograd-driven WFBP (torch_wfbp.Wfbp) on one GPU: a training step through the scheduler equals a
plain PyTorch SGD step (fp32 reference of the same op) for every parameter — FC layers via SFB
factors from the backward hooks, conv/BN layers via flat dense buckets; WFBP == sequential."""
import numpy as np
import pytest

from tests._util import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

if have_gpu():
    import torch
    import torch.nn as nn
    import paper_1706_03292_b200 as pos
    from paper_1706_03292_b200.torch_wfbp import Wfbp


def make_model(seed):
    torch.manual_seed(seed)
    return nn.Sequential(
        nn.Conv2d(3, 8, 3, padding=1), nn.BatchNorm2d(8), nn.ReLU(),
        nn.Conv2d(8, 8, 3, padding=1, bias=False), nn.ReLU(), nn.Flatten(),
        nn.Linear(8 * 8 * 8, 200), nn.ReLU(), nn.Linear(200, 10)).cuda()


@pytest.mark.parametrize("sequential", [False, True])
@pytest.mark.parametrize("bucket_mb", [0.0, 16.0])
def test_wfbp_step_equals_torch_sgd(sequential, bucket_mb):
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    K, lr = 16, 0.05
    x = torch.randn(K, 3, 8, 8, device="cuda")
    y = torch.randint(0, 10, (K,), device="cuda")
    ref = make_model(0)
    loss = nn.functional.cross_entropy(ref(x), y)
    loss.backward()
    with torch.no_grad():
        expect = {n: (p - lr * p.grad).detach().clone() for n, p in ref.named_parameters()}

    model = make_model(0)
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    wf = Wfbp(model, ctx, K, bucket_mb=bucket_mb, dtype="f32", factor_dtype=torch.float32,
              sequential=sequential)
    loss2 = nn.functional.cross_entropy(model(x), y)
    assert torch.allclose(loss, loss2)
    wf.step(loss2, lr=lr)
    torch.cuda.synchronize()
    for n, p in model.named_parameters():
        got, exp = p.detach().double().cpu().numpy(), expect[n].double().cpu().numpy()
        scale = np.max(np.abs(exp))
        assert np.max(np.abs(got - exp)) <= 1e-5 * scale, n
    # a second step keeps working (triggers re-armed, factors released)
    loss3 = nn.functional.cross_entropy(model(x), y)
    wf.step(loss3, lr=lr)
    torch.cuda.synchronize()
    assert float(loss3) < float(loss2) + 1e-3
    wf.close()
    ctx.close()
