"""Seeded synthetic inputs shared by tests, bench.py and smoke().

This module holds NONE of the method's arithmetic (no inner products, no
top-k, no k-means).  It only draws numbers: a low-rank Gaussian mixture of
unit-norm embeddings shaped like the paper's passage corpus (PAPER.md
App. B.3, "approximately 21 million text chunks ... embedded into a
... vector") with the recipe of SURVEY.md §8(d) / DESIGN.md §3.
"""
from .synth import (  # noqa: F401
    CONFIGS,
    CORPUS_SEED,
    QUERY_SEED,
    Mixture,
    make_mixture,
    draw_rows,
    draw_rows_into,
    to_bf16_bits,
    bf16_bits_to_f32,
    planted_corpus,
)
