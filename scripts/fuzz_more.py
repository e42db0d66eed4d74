"""Extra seeds of the differential lexer fuzz (tests/test_lexer_fuzz.py) on the GPU.  usage: fuzz_more.py [first] [count]"""
import sys
sys.path[:0] = [".", "tests", "oracle"]
import torch
from paper_2601_13345_b200 import native
import test_lexer_fuzz as F

first = int(sys.argv[1]) if len(sys.argv) > 1 else 100
count = int(sys.argv[2]) if len(sys.argv) > 2 else 20
native.get_runtime(0)
bad = 0
for seed in range(first, first + count):
    try:
        F.test_fast_path_and_exact_walk_agree_on_mutated_kernels("gpu", seed)
    except AssertionError as ex:
        bad += 1
        print("seed", seed, "FAIL", str(ex)[:400])
print(f"fuzz: {count} seeds x 400 mutated kernels, failures: {bad}")
