"""CPU: the numpy Philox4x32-10 restatement (tests/philox_ref.py) against the
published known-answer vectors; it then pins the device generator (GPU tests)."""
import numpy as np

from philox_ref import KAT, philox4x32_10


def test_philox_known_answers():
    for ctr, key, want in KAT:
        got = philox4x32_10(np.array(ctr, np.uint32), np.array(key, np.uint32))
        assert [int(v) for v in got] == list(want)
