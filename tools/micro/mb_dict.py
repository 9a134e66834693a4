"""dict_build microbench at 2^24 keys (50 % / 99 % duplicates); argv[1] = reps."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2601_06765_b200.bench import microbench  # noqa: E402

for dup in (0.5, 0.99):
    d = microbench("dict_build", 1 << 24, duplicate_rate=dup, seed=1, reps=int(sys.argv[1]))
    print(json.dumps({k: d[k] for k in ("duplicate_rate", "unique_out", "elapsed_ns", "hbm_frac", "dict_path")}))
