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


@pytest.mark.parametrize("per_layer_gate", [False, True])
def test_wfbp_fc_forced_to_ps_and_per_layer_gate(per_layer_gate):
    """One FC layer synchronised by PS (flat [W|b] buffer; Algorithm 1 would pick SFB here — the
    GoogLeNet-at-16-nodes case of PAPER:517 forced), and the per-layer forward gate of PAPER:158
    instead of the global end: three steps equal three plain PyTorch SGD steps."""
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    K, lr = 16, 0.05
    xs = [torch.randn(K, 3, 8, 8, device="cuda") for _ in range(3)]
    ys = [torch.randint(0, 10, (K,), device="cuda") for _ in range(3)]
    ref = make_model(1)
    for x, y in zip(xs, ys):
        ref.zero_grad()
        nn.functional.cross_entropy(ref(x), y).backward()
        with torch.no_grad():
            for p in ref.parameters():
                p -= lr * p.grad
    model = make_model(1)
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    wf = Wfbp(model, ctx, K, dtype="f32", factor_dtype=torch.float32, force_ps=("6",),
              per_layer_gate=per_layer_gate)
    assert wf.schemes == {"6": pos.POS_SCHEME_PS, "8": pos.POS_SCHEME_SFB}
    for x, y in zip(xs, ys):
        wf.step(nn.functional.cross_entropy(model(x), y), lr=lr)
    torch.cuda.synchronize()
    for (n, p), (_, q) in zip(model.named_parameters(), ref.named_parameters()):
        got, exp = p.detach().double().cpu().numpy(), q.detach().double().cpu().numpy()
        assert np.max(np.abs(got - exp)) <= 1e-5 * np.max(np.abs(exp)), n
    wf.close()
    ctx.close()


def test_wfbp_short_last_batch_is_padded_and_long_batch_raises():
    """A short last batch (K' < K rows) is padded with zero factor rows (they add nothing to U^T V):
    the step equals torch SGD on the K' samples; more rows than K is refused."""
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    K, Ks, lr = 16, 11, 0.05
    x = torch.randn(Ks, 3, 8, 8, device="cuda")
    y = torch.randint(0, 10, (Ks,), device="cuda")
    ref = make_model(2)
    nn.functional.cross_entropy(ref(x), y).backward()
    with torch.no_grad():
        expect = {n: (p - lr * p.grad).detach().clone() for n, p in ref.named_parameters()}
    model = make_model(2)
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    wf = Wfbp(model, ctx, K, dtype="f32", factor_dtype=torch.float32)
    wf.step(nn.functional.cross_entropy(model(x), y), lr=lr)
    torch.cuda.synchronize()
    for n, p in model.named_parameters():
        got, exp = p.detach().double().cpu().numpy(), expect[n].double().cpu().numpy()
        assert np.max(np.abs(got - exp)) <= 1e-5 * np.max(np.abs(exp)), n
    xl = torch.randn(K + 1, 3, 8, 8, device="cuda")
    with pytest.raises(ValueError):
        wf.step(nn.functional.cross_entropy(model(xl), torch.zeros(K + 1, dtype=torch.long, device="cuda")), lr=lr)
    wf.close()
    ctx.close()
