"""ORACLE — TEST INFRASTRUCTURE ONLY.

Brute-force dense causal attention in numpy fp64 for tiny inputs: a second,
independent code path (library matmul + explicit mask) that pins the C oracle.

  S = scale * Q K^T  + M   (M_ij = -inf for j > i; "attention only
                            operates among the tokens in the same request")
  P = rowsoftmax(S) ;  O = P V           (§2.1; classic MHA P:454)
"""
from __future__ import annotations

import numpy as np


def bits_to_f64(b) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def dense_causal_attention(q_bits, k_bits, v_bits, cu_seqlens, scale: float) -> np.ndarray:
    q, k, v = bits_to_f64(q_bits), bits_to_f64(k_bits), bits_to_f64(v_bits)
    T, n, d = q.shape
    out = np.zeros((T, n, d))
    for r in range(len(cu_seqlens) - 1):
        s0, s1 = int(cu_seqlens[r]), int(cu_seqlens[r + 1])
        l = s1 - s0
        if l == 0:
            continue
        mask = np.triu(np.full((l, l), -np.inf), k=1)
        for h in range(n):
            S = scale * (q[s0:s1, h, :] @ k[s0:s1, h, :].T) + mask
            S = S - S.max(axis=1, keepdims=True)
            P = np.exp(S)
            P = P / P.sum(axis=1, keepdims=True)
            out[s0:s1, h, :] = P @ v[s0:s1, h, :]
    return out
