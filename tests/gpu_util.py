"""Helpers for the -m gpu parity tests: upload bf16-exact arrays, read back as fp64."""
import numpy as np
import torch

from synth import bf16_bits, round_bf16


def dev_bf16(a):
    bits = bf16_bits(np.ascontiguousarray(a))
    return torch.from_numpy(bits.view(np.int16)).cuda().view(torch.bfloat16)


def dev_f32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def stream():
    return torch.cuda.current_stream().cuda_stream


__all__ = ["dev_bf16", "dev_f32", "host", "rel", "stream", "round_bf16"]
