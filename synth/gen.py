"""Counter-based generator: value(seed, tensor_id, idx).

    h = splitmix64(seed XOR (tensor_id << 40) XOR idx)        (all mod 2^64)
    u = float32(h >> 40) * 2^-24                               (exact: 24-bit int)
    x = float32(u - 0.5f) * k,  k = float32(sqrt(12) * std)    (u - 0.5f is exact;
                                                                one rounding in *)

Uniform on [-k/2, k/2) with standard deviation std.  Any slice of any tensor can
be regenerated independently (no sequential state), so the CUDA path can
initialise a 70B-parameter stack on the device while the oracle regenerates
exactly the elements it samples.  Random init with a fixed seed is what the
paper's own correctness run used (§5.6).
"""
import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

SEED_WEIGHTS = 0


def seed_inputs(rank: int, micro: int = 0) -> int:
    """Inputs of rank r's micro-batch `micro` (gradient accumulation)."""
    return 1000 + rank + 4096 * micro


def seed_targets(rank: int, micro: int = 0) -> int:
    return 2000 + rank + 4096 * micro


def splitmix64(x):
    """Vectorised splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _G
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_u24(seed: int, tensor_id: int, idx):
    """The 24 high bits of the hash as an integer array (exact)."""
    key = np.uint64((seed ^ (tensor_id << 40)) & 0xFFFFFFFFFFFFFFFF)
    h = splitmix64(np.asarray(idx, dtype=np.uint64) ^ key)
    return (h >> np.uint64(40)).astype(np.uint32)


def std_to_k(std: float) -> np.float32:
    """k = fp32(sqrt(12) * std), one rounding from a double."""
    return np.float32(np.sqrt(12.0) * std)


K_MLP = np.float32(0.125)      # U(+-1/16) = PyTorch default Linear(256,256) init
K_UNIT = std_to_k(1.0)         # inputs / targets, std 1


def values(seed: int, tensor_id: int, start: int, count: int, k) -> np.ndarray:
    """float32 values for elements [start, start+count) of tensor `tensor_id`."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    u = uniform_u24(seed, tensor_id, idx).astype(np.float32) * np.float32(2.0 ** -24)
    return (u - np.float32(0.5)) * np.float32(k)
