"""PyTorch integration of the WFBP scheduler: wait-free backpropagation driven by autograd.

PAPER:311 §4.2 — "figure out where the backpropagation proceeds (L6), and insert Poseidon's syncer
APIs in between gradient generation and application (L7)". Here:

* every nn.Linear becomes a PosLinear whose backward computes only grad_input = grad_output · W and
  hands the sufficient factors u = grad_output (K x M), v = input (K x N) to the scheduler
  (pos_sched_factors_ready, on the backward's CUDA stream, right after the grad_input GEMM has read W
  — the WAR point of PAPER:152). No dW is formed by autograd for SFB layers; the library rebuilds and
  applies it (A4).
* every other parameterised module (Conv2d, BatchNorm) is a DENSE layer: its parameters become
  views into flat bucket buffers (library-symmetric when P > 1), .grad views into matching gradient
  buckets; a post-accumulate-grad hook fires pos_sched_grad_ready once all of the bucket's
  parameters have their gradient.
* Wfbp.step(loss) = Algorithm 2: begin (C := 0), loss.backward() (triggers in L..1 order as autograd
  reaches each layer), end (the current stream waits until every layer is applied).

The update is W += alpha * (sum of all workers' gradients) with alpha = -lr / P for a loss that is a
mean over each worker's K samples (readings S5, S6): the library performs the SGD step itself, so no
torch optimizer is used for these parameters.
"""
from __future__ import annotations

import math

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import Context, Scheduler, POS_IN_BF16, POS_IN_F32, POS_SCHEME_SFB, pos_padded_size


class _PosLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, layer):
        w = weight.to(x.dtype) if x.dtype != weight.dtype else weight
        b = None if bias is None else (bias.to(x.dtype) if x.dtype != bias.dtype else bias)
        ctx.save_for_backward(x, w)
        ctx.layer = layer
        return F.linear(x, w, b)

    @staticmethod
    def backward(ctx, grad_out):
        x, w = ctx.saved_tensors
        layer = ctx.layer
        grad_in = grad_out @ w if ctx.needs_input_grad[0] else None   # b^l reads W here ...
        u = grad_out.reshape(-1, grad_out.shape[-1]).contiguous()
        v = x.reshape(-1, x.shape[-1]).contiguous()
        layer._wfbp.factors_ready(layer._wfbp_index, u, v)         # ... then the sync may write W
        return grad_in, None, None, None


class PosLinear(nn.Linear):
    """nn.Linear whose weight gradient is synchronised by SFB (or PS) through the scheduler."""

    _wfbp = None
    _wfbp_index = -1

    def forward(self, x):
        if self._wfbp is None or not torch.is_grad_enabled():
            return F.linear(x, self.weight.to(x.dtype), None if self.bias is None else self.bias.to(x.dtype))
        return _PosLinearFn.apply(x, self.weight, self.bias, self)


def convert_linear(module: nn.Module) -> nn.Module:
    """Replace every nn.Linear (recursively) with a PosLinear sharing the same parameters."""
    for name, child in list(module.named_children()):
        if type(child) is nn.Linear:
            pl = PosLinear(child.in_features, child.out_features, bias=child.bias is not None,
                           device=child.weight.device, dtype=child.weight.dtype)
            pl.weight = child.weight
            if child.bias is not None:
                pl.bias = child.bias
            setattr(module, name, pl)
        else:
            convert_linear(child)
    return module


class Wfbp:
    """Attach Poseidon's per-layer synchronisation to a model (layers in module registration order,
    which is the forward order of sequential CNNs; backward triggers arrive in reverse)."""

    def __init__(self, model: nn.Module, ctx: Context, batch_per_gpu: int, bucket_mb: float = 16.0,
                 dtype: str = "bf16", factor_dtype=torch.bfloat16, sequential: bool = False,
                 timing=False):
        self.model = convert_linear(model)
        self.ctx = ctx
        self.P = ctx.world
        self.K = batch_per_gpu
        self.factor_dtype = factor_dtype
        dev = next(model.parameters()).device
        layers = []
        for mod in model.modules():
            params = [p for p in mod.parameters(recurse=False) if p.requires_grad]
            if not params:
                continue
            layers.append(mod)
        self.layers = layers
        # Scheduler layers: one per FC layer, one per bucket of consecutive dense modules (a bucket
        # is triggered once, by the last of its parameters' post-accumulate-grad hooks, so the host
        # pays one library call per bucket, not per module).
        units = []
        bucket_elems = int(bucket_mb * 2 ** 20 / 4)
        i = 0
        while i < len(layers):
            if isinstance(layers[i], PosLinear):
                units.append(("fc", layers[i]))
                i += 1
                continue
            group, n_tot = [], 0
            while i < len(layers) and not isinstance(layers[i], PosLinear):
                m = layers[i]
                n_m = sum(p.numel() for p in m.parameters(recurse=False) if p.requires_grad)
                group.append(m)
                n_tot += n_m
                i += 1
                if n_tot >= bucket_elems:
                    break
            units.append(("dense", group, n_tot))
        self.sched = Scheduler(ctx, len(units), timing=timing, sequential=sequential)
        self._keep = []              # factors alive until the iteration ends
        self._buffers = []
        self._pending = [0] * len(units)   # parameters of each bucket still without a gradient
        self._nparams = [0] * len(units)
        in_dt = POS_IN_BF16 if factor_dtype == torch.bfloat16 else POS_IN_F32
        for ui, un in enumerate(units):
            if un[0] == "fc":
                mod = un[1]
                M, N = mod.out_features, mod.in_features
                scheme = self.sched.add_fc(ui, M, N, self.K, mod.weight.data, None if mod.bias is None else mod.bias.data,
                                           None, dtype=dtype, in_dtype=in_dt)
                if scheme != POS_SCHEME_SFB:
                    raise NotImplementedError("FC layer on the PS path needs a flat [W|b] buffer")
                mod._wfbp, mod._wfbp_index = self, ui
                mod.weight.requires_grad_(False)   # dW is never formed by autograd
                if mod.bias is not None:
                    mod.bias.requires_grad_(False)
                # the forward must still see the layer as trainable for grad_input: x requires grad
                continue
            _, group, n_tot = un
            Pn = pos_padded_size(n_tot, self.P)
            if self.P > 1:
                Wf, Gf = ctx.sym_empty(Pn), ctx.sym_empty(Pn)
            else:
                Wf, Gf = torch.zeros(Pn, device=dev), torch.zeros(Pn, device=dev)
            off = 0
            hook = self._make_hook(ui)
            for m in group:
                for p in m.parameters(recurse=False):
                    if not p.requires_grad:
                        continue
                    k = p.numel()
                    # same strides as the original parameter (e.g. channels_last conv weights), so
                    # autograd accumulates straight into the bucket
                    wv = torch.as_strided(Wf, p.shape, p.stride(), off)
                    wv.copy_(p.data)
                    p.data = wv
                    p.grad = torch.as_strided(Gf, p.shape, p.stride(), off)
                    p.register_post_accumulate_grad_hook(hook)
                    self._nparams[ui] += 1
                    off += k
            self.sched.add_dense_bucket(ui, [n_tot], Wf, Gf)
            self._buffers.append((Wf, Gf))

    def _make_hook(self, ui):
        pending, sched = self._pending, self.sched

        def hook(p):
            pending[ui] -= 1
            if pending[ui] == 0:
                sched.grad_ready(ui, torch.cuda.current_stream())
        return hook

    def factors_ready(self, li, u, v):
        u = u.to(self.factor_dtype) if u.dtype != self.factor_dtype else u
        v = v.to(self.factor_dtype) if v.dtype != self.factor_dtype else v
        self._keep += [u, v]
        self.sched.factors_ready(li, u, v, torch.cuda.current_stream())

    def zero_grad(self):
        for _, Gf in self._buffers:
            Gf.zero_()

    def step(self, loss, lr: float):
        """One Algorithm-2 iteration: C := 0, backward (per-layer triggers), wait until all applied."""
        self._pending[:] = self._nparams
        self.zero_grad()
        self.sched.begin(-lr / self.P)
        loss.backward()
        self.sched.end(torch.cuda.current_stream())
        self._keep.clear()

    def close(self):
        self.sched.close()
