"""PyTorch integration of the WFBP scheduler: wait-free backpropagation driven by autograd.

PAPER:311 §4.2 — "figure out where the backpropagation proceeds (L6), and insert Poseidon's syncer
APIs in between gradient generation and application (L7)". Here:

* every nn.Linear becomes a PosLinear whose backward computes only grad_input = grad_output · W and
  hands the sufficient factors u = grad_output (K x M), v = input (K x N) to the scheduler
  (pos_sched_factors_ready) with TWO events: `factors_ready`, recorded before the grad_input GEMM
  (the pack and gather may start at once), and `weights_free`, recorded after it (the WAR point of
  PAPER:152: the reconstruction writes W only once b^l has read it). No dW is formed by autograd;
  the library rebuilds and applies it (A4). An FC layer that Algorithm 1 sends to PS (e.g.
  GoogLeNet's FC at 16 nodes), or that is forced there, keeps the same hook: the library
  forms its local dense gradient from the factors and synchronises a flat [W | b] buffer.
* every other parameterised module (Conv2d, BatchNorm) is a DENSE layer: its parameters become
  views into flat bucket buffers (library-symmetric when P > 1), .grad views into matching gradient
  buckets; a post-accumulate-grad hook fires pos_sched_grad_ready once all of the bucket's
  parameters have their gradient.
* Wfbp.step(loss) = Algorithm 2: begin (C := 0), loss.backward() (triggers in L..1 order as autograd
  reaches each layer), end. With per_layer_gate=True the end does not block the stream: a forward
  pre-hook makes f^l of the next iteration wait for layer l's own sync only (pos_sched_wait_layer) —
  the cross-iteration overlap the paper notes TensorFlow misses.

The update is W += alpha * (sum of all workers' gradients) with alpha = -lr / P for a loss that is a
mean over each worker's K samples (readings S5, S6): the library performs the SGD step itself, so no
torch optimizer is used for these parameters.
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import (POS_IN_BF16, POS_IN_F32, POS_SCHEME_PS, POS_SCHEME_SFB, Context, Scheduler,
               pos_choose_scheme, pos_padded_size)


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
        wf = layer._wfbp
        u, v = wf.factors(grad_out.reshape(-1, grad_out.shape[-1]), x.reshape(-1, x.shape[-1]))
        ev_f, ev_w = wf.events(layer._wfbp_index)
        ev_f.record()                                              # u, v complete
        grad_in = grad_out @ w if ctx.needs_input_grad[0] else None   # b^l reads W here ...
        ev_w.record()                                              # ... and no longer after this
        wf.sched.factors_ready(layer._wfbp_index, u, v, factors_ev=ev_f, weights_free=ev_w)
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
    which is the forward order of sequential CNNs; backward triggers arrive in reverse).

    force_ps: names (as in model.named_modules()) of nn.Linear layers to synchronise by PS instead
    of Algorithm 1's choice. per_layer_gate: gate each layer's next forward on its own sync.

    Construct it on the stream that will run the training steps (for CUDA-graph capture: the
    capture stream): the post-accumulate-grad hooks keep every dense parameter's AccumulateGrad node
    alive, and autograd synchronises each backward with the stream that node was created on."""

    def __init__(self, model: nn.Module, ctx: Context, batch_per_gpu: int, bucket_mb: float = 16.0,
                 dtype: str = "bf16", factor_dtype=torch.bfloat16, sequential: bool = False,
                 timing=False, force_ps=(), per_layer_gate: bool = False):
        self.model = convert_linear(model)
        self.ctx = ctx
        self.P = ctx.world
        self.K = batch_per_gpu
        self.factor_dtype = factor_dtype
        self.per_layer_gate = per_layer_gate
        dev = next(model.parameters()).device
        names = {m: n for n, m in model.named_modules()}
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
        self._events = {}
        self._pending = [0] * len(units)   # parameters of each bucket still without a gradient
        self._nparams = [0] * len(units)
        self.schemes = {}
        in_dt = POS_IN_BF16 if factor_dtype == torch.bfloat16 else POS_IN_F32
        alloc = (lambda k: ctx.sym_empty(k)) if self.P > 1 else (lambda k: torch.zeros(k, device=dev))
        for ui, un in enumerate(units):
            if un[0] == "fc":
                mod = un[1]
                M, N = mod.out_features, mod.in_features
                forced = names.get(mod) in set(force_ps)
                scheme = POS_SCHEME_PS if forced else pos_choose_scheme(M, N, self.K, self.P)
                b = None if mod.bias is None else mod.bias
                if scheme == POS_SCHEME_SFB:
                    self.sched.add_fc(ui, M, N, self.K, mod.weight.data, None if b is None else b.data,
                                      None, dtype=dtype, in_dtype=in_dt)
                else:
                    # PS for an FC layer: W and b live in one flat [W | b] buffer (and the local dense
                    # gradient in a matching one), padded to the shard table
                    n = M * N + (M if b is not None else 0)
                    Pn = pos_padded_size(n, self.P)
                    Wf, Gf = alloc(Pn), alloc(Pn)
                    Wf[:M * N].copy_(mod.weight.data.reshape(-1))
                    mod.weight.data = Wf[:M * N].view(M, N)
                    if b is not None:
                        Wf[M * N:n].copy_(b.data)
                        b.data = Wf[M * N:n]
                    s = self.sched.add_fc(ui, M, N, self.K, mod.weight.data,
                                          None if b is None else b.data, Gf, dtype=dtype, in_dtype=in_dt,
                                          force_scheme=POS_SCHEME_PS)
                    assert s == POS_SCHEME_PS
                    self._buffers.append((Wf, Gf, False))
                self.schemes[names.get(mod)] = scheme
                mod._wfbp, mod._wfbp_index = self, ui
                mod.weight.requires_grad_(False)   # dW is never formed by autograd
                if mod.bias is not None:
                    mod.bias.requires_grad_(False)
                # the forward must still see the layer as trainable for grad_input: x requires grad
                if per_layer_gate:
                    mod.register_forward_pre_hook(self._make_gate(ui))
                continue
            _, group, n_tot = un
            Pn = pos_padded_size(n_tot, self.P)
            Wf, Gf = alloc(Pn), alloc(Pn)
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
                if per_layer_gate:
                    m.register_forward_pre_hook(self._make_gate(ui))
            self.sched.add_dense_bucket(ui, [n_tot], Wf, Gf)
            self._buffers.append((Wf, Gf, True))
        self._synced_once = False

    def _make_hook(self, ui):
        pending, sched = self._pending, self.sched

        def hook(p):
            pending[ui] -= 1
            if pending[ui] == 0:
                sched.grad_ready(ui, torch.cuda.current_stream())
        return hook

    def _make_gate(self, ui):
        def gate(module, args):
            if self._synced_once and torch.is_grad_enabled():
                self.sched.wait_layer(ui, torch.cuda.current_stream())   # f^l waits for s^l only
        return gate

    def events(self, ui):
        ev = self._events.get(ui)
        if ev is None:
            ev = self._events[ui] = (torch.cuda.Event(), torch.cuda.Event())
        return ev

    def factors(self, u, v):
        """The K factor rows in the factor dtype. A short last batch is padded with zero rows (zero
        factors add nothing to U^T V); more rows than the registered K is an error."""
        rows = u.shape[0]
        if rows > self.K:
            raise ValueError(f"{rows} sample rows but the layers were registered with K = {self.K}")
        u = u.to(self.factor_dtype).contiguous()
        v = v.to(self.factor_dtype).contiguous()
        if rows < self.K:
            u = torch.cat([u, u.new_zeros(self.K - rows, u.shape[1])])
            v = torch.cat([v, v.new_zeros(self.K - rows, v.shape[1])])
        self._keep += [u, v]
        return u, v

    def zero_grad(self):
        for _, Gf, dense in self._buffers:
            if dense:
                Gf.zero_()

    def step(self, loss, lr: float):
        """One Algorithm-2 iteration: C := 0, backward (per-layer triggers), then wait until all
        applied (or, with per_layer_gate, close the iteration and let each f^l gate itself)."""
        # the previous iteration's factors: every consumer of them is complete in stream order by
        # now (global end, or each layer's forward gate), so their memory may be reused
        self._keep = []
        self._pending[:] = self._nparams
        self.zero_grad()
        self.sched.begin(-lr / self.P)
        loss.backward()
        if self.per_layer_gate:
            self.sched.end_layers(torch.cuda.current_stream())
        else:
            self.sched.end(torch.cuda.current_stream())
        self._synced_once = True

    def close(self):
        self.sched.close()
