"""Microbenchmark sweep on the GPU (paper_2601_06765_b200.bench.microbench):
one JSON line per (kind, size, duplicate rate)."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06765_b200.bench import microbench  # noqa: E402

sizes = [int(x) for x in (sys.argv[1:] or [1 << 20, 1 << 22, 1 << 24])]
for n in sizes:
    for dup in (0.5, 0.9, 0.99):
        print(json.dumps(microbench("dict_build", n, dup, seed=0)), flush=True)
    print(json.dumps(microbench("row_assemble", n, seed=0)), flush=True)
    print(json.dumps(microbench("mod_fma", 4 * n, seed=0)), flush=True)
