"""Dump the synthetic workload layer shapes from torchvision
architectures instantiated on the `meta` device (no weights, no data).

Writes synth_inputs/shapes.json. Layers are listed in FORWARD order (l = 1..L);
backward / WFBP order is the reverse (§3, C_t = [f^1..f^L, b^L..b^1]).
Each entry: {"name", "kind": "fc"|"dense", "M", "N", "bias"} for fc (M = out_features,
N = in_features, SURVEY §8 notation) and {"name", "kind": "dense", "n"} for conv/BN
modules (weights + bias flattened).
"""
import json, torch, torchvision.models as tvm

def layers_of(model):
    out = []
    for name, mod in model.named_modules():
        if isinstance(mod, torch.nn.Linear):
            out.append({"name": name, "kind": "fc", "M": mod.out_features, "N": mod.in_features,
                        "bias": mod.bias is not None})
        elif isinstance(mod, (torch.nn.Conv2d, torch.nn.BatchNorm2d)):
            n = sum(p.numel() for p in mod.parameters(recurse=False))
            if n:
                out.append({"name": name, "kind": "dense", "n": n})
    return out

def main():
    with torch.device("meta"):
        models = {
            "alexnet": tvm.alexnet(),
            "vgg19": tvm.vgg19(),
            "vgg19_22k": tvm.vgg19(num_classes=21841),
            "inception_v3": tvm.inception_v3(aux_logits=True, init_weights=False),
        }
    res = {}
    for k, m in models.items():
        ls = layers_of(m)
        total = sum(p.numel() for p in m.parameters())
        covered = sum(l["n"] if l["kind"] == "dense" else l["M"] * l["N"] + (l["M"] if l["bias"] else 0) for l in ls)
        assert covered == total, (k, covered, total)
        res[k] = {"total_params": total, "layers": ls}
        print(k, total, len(ls), sum(1 for l in ls if l["kind"] == "fc"))
    json.dump(res, open("synth_inputs/shapes.json", "w"), indent=1)

if __name__ == "__main__":
    main()
