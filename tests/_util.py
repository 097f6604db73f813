"""Shared test helpers: uploads of host-generated inputs with identical bits, error norms."""
import numpy as np

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

import synth_inputs as si


def have_gpu() -> bool:
    return torch is not None and torch.cuda.is_available()


def to_dev(x: np.ndarray, dtype: str = "f32"):
    """Upload host values. dtype 'bf16' uploads the bf16 bit patterns (values must already be
    bf16-representable, or they are rounded RNE on the host)."""
    if dtype == "bf16":
        bits = si.bf16_round(np.ascontiguousarray(x, dtype=np.float32)).reshape(x.shape)
        return torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def to_host(t) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def err(x, ref) -> float:
    """Normwise infinity relative error (reading S15): max|x - ref| / max|ref|."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    d = np.max(np.abs(x - ref)) if x.size else 0.0
    s = np.max(np.abs(ref)) if ref.size else 0.0
    if s == 0.0:
        return float(d)
    return float(d / s)


def padded(n: int, P: int) -> int:
    from oracle.shard import padded_size
    return padded_size(n, P)
