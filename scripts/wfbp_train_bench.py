"""Exposed synchronisation time of a real training step (SURVEY §8(d) "Exposed sync"; the north
star's third target): VGG19-22K (or another config) forward + backward at batch K per GPU, bf16
autocast, channels_last, synthetic images and labels, with Poseidon's per-layer synchronisation
driven by autograd hooks (WFBP), versus
  local:   the plain single-GPU PyTorch step doing the same update (autograd dW + SGD, no sync) —
           the baseline the exposed fraction is quoted against ("exposed_frac_wfbp_vs_local");
  nosync:  the same forward/backward without dW or any update (a lower bound, not a real step);
and versus the sequential schedule (sync after the whole backward, the Caffe+PS analogue of
PAPER:407).

    python scripts/wfbp_train_bench.py [--config c3] [--steps 20]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/wfbp_train_bench.py

Prints one JSON line on rank 0.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.nn as nn

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos  # noqa: E402
from paper_1706_03292_b200.torch_wfbp import Wfbp, convert_linear  # noqa: E402
import synth_inputs as si  # noqa: E402


def build_model(name, dev):
    import torchvision.models as tvm
    torch.manual_seed(0)
    if name == "vgg19_22k":
        m = tvm.vgg19(num_classes=21841)
        res = 224
    elif name == "vgg19":
        m = tvm.vgg19()
        res = 224
    elif name == "alexnet":
        m = tvm.alexnet()
        res = 224
    elif name == "inception_v3":
        m = tvm.inception_v3(aux_logits=False, init_weights=False)
        res = 299
    else:
        raise ValueError(name)
    return m.to(dev).to(memory_format=torch.channels_last), res, (21841 if name == "vgg19_22k" else 1000)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--bucket-mb", type=float, default=16.0)
    ap.add_argument("--max-ctas", type=int, default=-1, help="cap of the reconstruction grid (0 = all SMs)")
    ap.add_argument("--graph", action="store_true",
                    help="capture the whole training step (forward, backward, synchronisation) as one CUDA "
                         "graph: no host launch overhead in either arm, so the difference is the sync itself")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        ctx = pos.Context.from_torch_distributed()
    else:
        ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    if a.max_ctas >= 0:
        ctx.set_max_ctas(a.max_ctas)
    model_name, K = si.CONFIGS[a.config]
    torch.backends.cudnn.benchmark = True
    g = torch.Generator(device=dev)
    g.manual_seed(rank)

    # every arm is built, warmed up and captured on ONE side stream: the post-accumulate-grad hooks
    # keep each parameter's AccumulateGrad node alive, and torch syncs a backward with the stream the
    # node was created on — the legacy default stream would break graph capture
    side = torch.cuda.Stream()

    def run(mode):
        with torch.cuda.stream(side):
            return _run(mode)

    def _run(mode):
        model, res, ncls = build_model(model_name, dev)
        wf = opt = None
        if mode == "local":
            # plain single-GPU PyTorch training step with the same update: autograd dW for every
            # layer + SGD (foreach) — the work a step does without any synchronisation
            opt = torch.optim.SGD(model.parameters(), lr=1e-3, momentum=0.0, foreach=True)
        elif mode == "nosync":
            convert_linear(model)
            for mod in model.modules():                 # same compute: no dW for FC layers
                if isinstance(mod, nn.Linear):
                    mod.weight.requires_grad_(False)
                    if mod.bias is not None:
                        mod.bias.requires_grad_(False)
        else:
            wf = Wfbp(model, ctx, K, bucket_mb=a.bucket_mb, sequential=(mode == "sequential"))
        x = torch.randn(K, 3, res, res, device=dev, generator=g).to(memory_format=torch.channels_last)
        y = torch.randint(0, ncls, (K,), device=dev, generator=g)
        lossf = nn.CrossEntropyLoss()

        def step():
            with torch.autocast("cuda", dtype=torch.bfloat16):
                out = model(x)
                loss = lossf(out.float(), y)
            if opt is not None:
                opt.zero_grad(set_to_none=True)
                loss.backward()
                opt.step()
            elif wf is None:
                for p in model.parameters():
                    p.grad = None
                loss.backward()
            else:
                wf.step(loss, lr=1e-3)
            return loss

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        run_step = step
        if a.graph:
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            gph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gph, stream=side):
                g_loss = step()
            torch.cuda.synchronize()

            def run_step():
                gph.replay()
                return g_loss
            for _ in range(3):
                run_step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.steps):
            loss = run_step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        lv = float(loss.item())
        run_step = gph = None            # the graph references the scheduler's events
        torch.cuda.synchronize()
        if wf is not None:
            wf.close()
        del model, wf
        torch.cuda.empty_cache()
        return ms, lv

    t_local, _ = run("local")
    t_nosync, _ = run("nosync")
    t_wfbp, loss_w = run("wfbp")
    t_seq, loss_s = run("sequential") if not os.environ.get("WFBP_ONLY") else (float("nan"), 0.0)
    out = {"metric": "exposed_sync_fraction", "config": a.config, "model": model_name, "per_gpu_batch": K,
           "n_gpus": world, "ms_step_local_sgd": t_local,
           "exposed_ms_wfbp_vs_local": t_wfbp - t_local, "exposed_frac_wfbp_vs_local": (t_wfbp - t_local) / t_wfbp,
           "ms_step_nosync": t_nosync, "ms_step_wfbp": t_wfbp, "ms_step_sequential": t_seq,
           "exposed_ms_wfbp": t_wfbp - t_nosync, "exposed_frac_wfbp": (t_wfbp - t_nosync) / t_wfbp,
           "exposed_ms_sequential": t_seq - t_nosync, "exposed_frac_sequential": (t_seq - t_nosync) / t_seq,
           "loss_finite": all(map(lambda v: v == v and abs(v) < 1e4, [loss_w, loss_s])),
           "bucket_mb": a.bucket_mb, "max_ctas": a.max_ctas,
           "launch": "whole step captured as one CUDA graph" if a.graph else "eager", "dtype": "bf16 autocast, fp32 master weights"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
