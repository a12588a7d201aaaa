"""Low-rank Gaussian-mixture generator.

Recipe G(struct_seed, row_seed; n, d, C, r, s_sub, s_n):
  * centres      mu_c = normalise(N(0, I_d))                 c = 0..C-1
  * bases        B_c  = QR(N(0, 1)^{d x r}).Q                orthonormal, d x r
    (mu and B come from one generator seeded by struct_seed alone)
  * row i        z_i ~ U[0, C),  u_i ~ N(0, I_r)/sqrt(r),  e_i ~ N(0, I_d)/sqrt(d)
                 x_i = normalise(mu_{z_i} + s_sub * B_{z_i} u_i + s_n * e_i)
    row draws come from a generator seeded by (row_seed, chunk index) for
    chunks of CHUNK rows, so any row range (a shard) is reproducible on its
    own and the same rows come out whatever the shard split.

Queries are fresh draws from the same mixture with a different row_seed
(agent-step queries are not corpus members, Alg. 1 line
"ExtractSearchQuery").

Everything is computed in float32 with torch on the requested device.  The
CPU and CUDA generators give different streams, so a test always hands the
SAME tensor (moved between devices) to both the oracle and the library.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

CHUNK = 1 << 16

# The five BASELINE.json configs.  n=21,015,324 is the
# DPR 100-word Wikipedia split size.
CONFIGS = {
    "c1": dict(n=10_000, d=128, nq=100, k=10, C=16, r=16, s_sub=1.0, s_n=0.7,
               corpus_dtype="f32"),
    "c2": dict(n=1_000_000, d=768, nq=256, k=10, C=128, r=32, s_sub=1.0, s_n=0.7,
               corpus_dtype="bf16"),
    "c3": dict(n=21_015_324, d=768, nq=512, k=10, C=128, r=32, s_sub=1.0, s_n=0.7,
               corpus_dtype="bf16"),
    "c4": dict(n=21_015_324, d=768, nq=512, k=10, C=128, r=32, s_sub=1.0, s_n=0.7,
               corpus_dtype="bf16", nlist=16384),
    "c5": dict(n=21_015_324, d=768, nq=64, k=5, C=128, r=32, s_sub=1.0, s_n=0.7,
               corpus_dtype="bf16"),
    # paper-shaped: the paper's encoder all-MiniLM-L6-v2 gives 384-d
    # embeddings (App. B.3) and the agent reads top-1..5 documents
    "p384": dict(n=21_015_324, d=384, nq=512, k=5, C=128, r=32, s_sub=1.0, s_n=0.7,
                 corpus_dtype="bf16"),
}
CORPUS_SEED = 1234
QUERY_SEED = 5678


@dataclasses.dataclass
class Mixture:
    d: int
    C: int
    r: int
    s_sub: float
    s_n: float
    mu: torch.Tensor      # [C, d] f32
    B: torch.Tensor       # [C, d, r] f32


def make_mixture(d, C, r, s_sub=1.0, s_n=0.7, struct_seed=CORPUS_SEED, device="cpu"):
    g = torch.Generator(device="cpu").manual_seed(int(struct_seed))
    mu = torch.randn(C, d, generator=g, dtype=torch.float64)
    mu = mu / mu.norm(dim=1, keepdim=True)
    G = torch.randn(C, d, r, generator=g, dtype=torch.float64)
    Q, _ = torch.linalg.qr(G)
    return Mixture(d, C, r, float(s_sub), float(s_n),
                   mu.to(torch.float32).to(device), Q.to(torch.float32).to(device))


def _chunk_seed(row_seed: int, chunk: int) -> int:
    # splitmix64 of (row_seed, chunk): a seed per chunk, independent of n.
    z = (int(row_seed) * 0x9E3779B97F4A7C15 + int(chunk) + 1) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return (z ^ (z >> 31)) & 0x7FFFFFFFFFFFFFFF


def _draw_chunk(mix: Mixture, row_seed: int, chunk: int, device) -> torch.Tensor:
    dev = torch.device(device)
    g = torch.Generator(device=dev).manual_seed(_chunk_seed(row_seed, chunk))
    R, d, r = CHUNK, mix.d, mix.r
    z = torch.randint(0, mix.C, (R,), generator=g, device=dev)
    u = torch.randn(R, r, generator=g, device=dev) / math.sqrt(r)
    x = torch.randn(R, d, generator=g, device=dev) * (mix.s_n / math.sqrt(d))
    mu, B = mix.mu.to(dev), mix.B.to(dev)
    x += mu[z]
    order = torch.argsort(z, stable=True)
    counts = torch.bincount(z, minlength=mix.C).tolist()
    start = 0
    for c, cnt in enumerate(counts):
        if cnt:
            idx = order[start:start + cnt]
            x[idx] += mix.s_sub * (u[idx] @ B[c].T)
            start += cnt
    x /= x.norm(dim=1, keepdim=True)
    return x


def draw_rows(mix: Mixture, n: int, row_seed: int, start: int = 0, device="cpu") -> torch.Tensor:
    """Rows [start, start+n) of the stream `row_seed`, float32 [n, d], unit norm."""
    out = torch.empty(n, mix.d, dtype=torch.float32, device=device)
    draw_rows_into(mix, out, row_seed, start)
    return out


def draw_rows_into(mix: Mixture, out: torch.Tensor, row_seed: int, start: int = 0) -> torch.Tensor:
    """Fill `out` ([n, d], float32 or bfloat16, any device) with rows [start, start+n).

    bfloat16 outputs are rounded to nearest-even by torch's cast (DESIGN.md
    reading R3), chunk by chunk, so the 21M x 768 corpus never exists in f32.
    """
    n = out.shape[0]
    dev = out.device
    row = start
    end = start + n
    while row < end:
        ci = row // CHUNK
        c0 = ci * CHUNK
        lo = row - c0
        hi = min(end - c0, CHUNK)
        x = _draw_chunk(mix, row_seed, ci, dev)
        out[row - start: row - start + (hi - lo)] = x[lo:hi].to(out.dtype)
        row = c0 + hi
    return out


def to_bf16_bits(x: torch.Tensor) -> np.ndarray:
    """RNE-round (torch cast) to bf16 and return the raw uint16 bits as numpy."""
    b = x.detach().to("cpu").to(torch.bfloat16).contiguous()
    return b.view(torch.int16).numpy().view(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def planted_corpus(n, d, winners, seed=7, device="cpu"):
    """Corpus of small random rows with 'planted' clear winners for tile-edge tests.

    Returns (corpus f32 [n,d], queries f32 [len(winners), d]); query j equals
    row winners[j] exactly, and every other row is scaled to norm 0.5 so the
    planted row wins by a wide margin (SURVEY.md §8(c) pin P7).
    """
    g = torch.Generator(device="cpu").manual_seed(seed)
    X = torch.randn(n, d, generator=g)
    X = 0.5 * X / X.norm(dim=1, keepdim=True)
    Q = torch.randn(len(winners), d, generator=g)
    Q = Q / Q.norm(dim=1, keepdim=True)
    for j, w in enumerate(winners):
        X[w] = Q[j]
    return X.to(device), Q.to(device)
