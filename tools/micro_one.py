"""One microbenchmark call (for ncu captures): micro_one.py KIND SIZE [DUP]."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_06765_b200.bench import microbench  # noqa: E402

kind, size = sys.argv[1], int(sys.argv[2])
dup = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
print(json.dumps(microbench(kind, size, dup, seed=0, reps=1)))
