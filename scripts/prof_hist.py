#!/usr/bin/env python
"""Histogram-mode lexer alone on the bench corpus (for ncu: `-k regex:lex_fast -s 2 -c 1`)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2601_13345_b200 import corpus, native

rt = native.get_runtime(0)
corp = corpus.bench_corpus(seed=4, target_bytes=0, n_kernels=38_400, rt=rt)
res = corpus.lex_histogram(corp, rt=rt)
for _ in range(4):
    corpus.lex_histogram(corp, out=res, rt=rt)
torch.cuda.synchronize()
print("segments fast/exact:", res.path_counts.cpu().tolist()[:2] if res.path_counts is not None else None)
