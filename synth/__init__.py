"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no quantization, no
scales, no GEMM): it only draws random numbers with the shapes and value
distributions of the paper's workloads (DESIGN.md §4 "input recipe").
Both `oracle/` and the product receive exactly these arrays.

Recipe:
  * activations x ~ N(0, 1) fp32 (LayerNorm outputs are ~unit variance per
    row); 1% of entries x10 to exercise clamping; 0.1% replaced by exact
    ties (n + 1/2) * 2^-2 to exercise the half-even rule (R2).
  * weights W ~ N(0, 0.02^2) (BERT initializer convention), biases
    U(-0.1, 0.1), LayerNorm gamma = 1 + N(0, 0.02^2), beta ~ N(0, 0.02^2).
  * seeds: weights 1000*layer + {0: QKV, 1: O, 2: FFN1, 3: FFN2, 4: LN};
    activations seed 0 (+ rank for row shards); calibration seed 1000000+.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# BASELINE.json configs (BJ.configs[0..4]); heads for BERT-large is the
# standard 16 (not stated in BJ).
CONFIGS = {
    "c1_linear": dict(M=128, K=768, N=768),
    "c2_bert_base_b1s128": dict(batch=1, seq=128, hidden=768, heads=12, ffn=3072, layers=1),
    "c3_bert_base_12l_b32s128": dict(batch=32, seq=128, hidden=768, heads=12, ffn=3072, layers=12),
    "c4_bert_large_b256s512": dict(batch=256, seq=512, hidden=1024, heads=16, ffn=4096, layers=1),
}


def activations(rows: int, cols: int, seed: int = 0, outliers: bool = True,
                ties_step: float = 0.25) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, cols), dtype=np.float32)
    if outliers and rows * cols > 0:
        m = rng.random((rows, cols)) < 0.01
        x[m] *= np.float32(10.0)
        t = rng.random((rows, cols)) < 0.001
        n = rng.integers(-40, 40, size=(rows, cols)).astype(np.float32)
        x[t] = ((n + np.float32(0.5)) * np.float32(ties_step))[t]
    return x


def weight(rows: int, cols: int, seed: int, std: float = 0.02) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(std))


def bias(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed + 500)
    return rng.uniform(-0.1, 0.1, size=n).astype(np.float32)


def ln_params(n: int, seed: int):
    rng = np.random.default_rng(seed)
    g = (np.float32(1.0) + rng.standard_normal(n, dtype=np.float32) * np.float32(0.02))
    b = rng.standard_normal(n, dtype=np.float32) * np.float32(0.02)
    return g.astype(np.float32), b.astype(np.float32)


@dataclass
class LayerFloat:
    """fp32 parameters of one BERT layer (before any quantization)."""
    hidden: int
    heads: int
    ffn: int
    w_qkv: np.ndarray
    b_qkv: np.ndarray
    w_o: np.ndarray
    b_o: np.ndarray
    w_1: np.ndarray
    b_1: np.ndarray
    w_2: np.ndarray
    b_2: np.ndarray
    ln1_g: np.ndarray
    ln1_b: np.ndarray
    ln2_g: np.ndarray
    ln2_b: np.ndarray


def layer_params(hidden: int, heads: int, ffn: int, layer: int = 0) -> LayerFloat:
    s = 1000 * layer
    g1, b1 = ln_params(hidden, s + 4)
    g2, b2 = ln_params(hidden, s + 5)
    return LayerFloat(
        hidden, heads, ffn,
        weight(3 * hidden, hidden, s + 0), bias(3 * hidden, s + 0),
        weight(hidden, hidden, s + 1), bias(hidden, s + 1),
        weight(ffn, hidden, s + 2), bias(ffn, s + 2),
        weight(hidden, ffn, s + 3), bias(hidden, s + 3),
        g1, b1, g2, b2)


def hidden_states(batch: int, seq: int, hidden: int, seed: int = 0) -> np.ndarray:
    """Layer input h^{l-1}: [batch*seq, hidden], ~unit variance rows."""
    return activations(batch * seq, hidden, seed=seed, outliers=True)


def varlen_seqlens(batch: int, valid_tokens: int, max_seq: int = 128, seed: int = 7):
    """Lengths of `batch` sequences summing to `valid_tokens` (Table 2, P:256:
    'valid tokens' = non-padding tokens), each in [1, max_seq]."""
    rng = np.random.default_rng(seed)
    assert batch <= valid_tokens <= batch * max_seq
    w = rng.random(batch) + 0.2
    L = np.maximum(1, np.floor(w / w.sum() * valid_tokens)).astype(int)
    L = np.minimum(L, max_seq)
    i = 0
    while L.sum() < valid_tokens:
        if L[i % batch] < max_seq:
            L[i % batch] += 1
        i += 1
    while L.sum() > valid_tokens:
        if L[i % batch] > 1:
            L[i % batch] -= 1
        i += 1
    return [int(v) for v in L]
