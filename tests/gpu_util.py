"""Helpers for the -m gpu parity tests: move seeded bf16 bit patterns between
numpy (oracle side) and torch CUDA tensors (libds side) without any arithmetic."""
import numpy as np
import torch


def to_dev(bits: np.ndarray) -> torch.Tensor:
    """uint16 bf16 bits -> CUDA bf16 tensor with the identical bit patterns."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def to_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def to_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def i32(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).cuda()


def valid_slots(lens, table, block_size=16):
    """(row, block, slot) for every valid token position of each sequence."""
    out = []
    for r, l in enumerate(lens):
        for t in range(int(l)):
            out.append((r, int(table[r, t // block_size]), t % block_size, t))
    return out


def pages_match(cache_bits: np.ndarray, opool, layer: int, lens, table, heads=None) -> bool:
    """Compare the valid slots of every page of `layer` between the GPU pool
    (numpy uint16 [L][2][NB][n][16][D]) and the oracle pool."""
    n = cache_bits.shape[3]
    heads = range(n) if heads is None else heads
    cache_pages = {}
    for (r, blk, slot, _t) in valid_slots(lens, table):
        for kv in (0, 1):
            for h in heads:
                key = (kv, blk, h)
                if key not in cache_pages:
                    cache_pages[key] = opool.page(layer, kv, blk, h)
                if not np.array_equal(cache_bits[layer, kv, blk, h, slot], cache_pages[key][slot]):
                    return False
    return True
