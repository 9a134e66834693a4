"""Binary F4 state snapshots (snapshot.py): a restored state is
the saved one (basis text, pair queue, counters) and a corrupted blob is
rejected.  CPU suite: states rebuilt from the reference's own snapshots."""

import pytest

from conftest import load_snapshots, state_from_snapshot
from paper_2601_06765_b200.snapshot import dumps_state, loads_state
from paper_2601_06765_b200.systems import format_system


@pytest.mark.parametrize("name", ["cyclic6_p32003", "katsura11_p32003"])
def test_snapshot_round_trip(name):
    for k, snap in sorted(load_snapshots(name).items())[:2]:
        ring, st = state_from_snapshot(snap)
        st.zero_reductions = 7
        blob = dumps_state(st)
        st2 = loads_state(blob)
        assert format_system(st2.ring, st2.basis) == format_system(ring, st.basis) == snap["basis"]
        assert [(q.i, q.j, q.lcm, q.degree, q.key) for q in st2.pairs] == \
            [(q.i, q.j, q.lcm, q.degree, q.key) for q in st.pairs]
        assert st2.zero_reductions == 7 and st2.ring.modulus.p == ring.modulus.p
        bad = bytearray(blob)
        bad[len(bad) // 2] ^= 1
        with pytest.raises(ValueError):
            loads_state(bytes(bad))
