"""The sharded compile_batch of SURVEY §8e on the CUDA engine (csrc/shard.cu,
dist.ShardedCompiler): `world` processes share cuda:0 and exchange over gloo.
The rank-order concatenation of the slices must equal the single-GPU plan
byte for byte on every batch of whole runs and on north-star replays
(cyclic-8 steps 10 and 19, Katsura-11 step 4); world 3 leaves some ranks
without rows or frontier slices on the small batches (empty exchanges)."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, name, tmp_path):
    port = _free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "_shard_worker.py"), str(r), str(world), str(port),
                               name, str(tmp_path)]) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=900) == 0
    reports = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    for rep in reports:
        assert rep, "no batches"
        for b in rep:
            assert all(b["ok"].values()), b
    return reports


@pytest.mark.parametrize("world,name", [(2, "cyclic6"), (3, "cyclic5"), (2, "katsura6"),
                                        (2, "snap:cyclic8_p32003:10,19"), (3, "snap:katsura11_p32003:4")])
def test_sharded_plan_equals_single_gpu(cuda, tmp_path, world, name):
    reports = _run(world, name, tmp_path)
    # the ranks' row ranges tile the final rows in order
    for b in range(len(reports[0])):
        ranges = [rep[b]["rows"] for rep in reports]
        assert ranges[0][0] == 0 and ranges[-1][1] == reports[0][b]["r"]
        assert all(a[1] == c[0] for a, c in zip(ranges, ranges[1:]))
