"""Seeded synthetic inputs shared by the oracle side and the product side.

Holds no SOM arithmetic (DESIGN.md §4 "input recipe")."""
from .corpus import CONFIGS, Corpus, bank_corpus, init_rows, uniform_matrix

__all__ = ["CONFIGS", "Corpus", "bank_corpus", "init_rows", "uniform_matrix"]
