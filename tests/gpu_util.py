"""Shared helpers for the -m gpu parity tests (no method arithmetic)."""
import numpy as np
import torch

import synth
from oracle import numerics as nx


def bf16_tensor(a_f32, device="cuda"):
    """fp32 numpy -> bf16 torch on device, RNE (same rounding as the oracle)."""
    bits = nx.bf16_bits(np.asarray(a_f32, np.float32))
    return torch.from_numpy(bits.view(np.int16).copy()).to(device).view(torch.bfloat16)


def to_np(t):
    """torch (any float dtype, any device) -> float64 numpy."""
    return t.detach().float().cpu().numpy().astype(np.float64)


def seeded(seed, tid, n, std=1.0):
    return synth.values(seed, tid, 0, n, synth.std_to_k(std))


def rel_norm(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
