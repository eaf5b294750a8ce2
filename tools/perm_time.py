"""Device time of the permutation null model (stk_simulate, method 2): the
parallel Fisher-Yates vs the sequential kernel (STK_SEQ_PERMUTATION=1).
    python tools/perm_time.py [n] [realisations]"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04753_b200 import _lib  # noqa: E402
from paper_1912_04753_b200.stripley import device, est, geom  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
d = device.get(0)
region = geom.StudyRegion([[0, 0], [50000, 0], [50000, 50000], [0, 50000]], 0, 63072000)
grid = est.DistanceGrid.regular(80.0, 2000.0, 207360, 5184000)
d.configure(region, grid)
rng = np.random.default_rng(1)
x = rng.uniform(0, 50000, n); y = rng.uniform(0, 50000, n); t = rng.integers(0, 63072001, n)
shape = (grid.cells_s(), grid.cells_t())
up, lo = np.zeros(shape), np.zeros(shape)
for rep in range(2):
    tel = _lib.StkTelemetry()
    t0 = time.perf_counter()
    d.check(d.lib.stk_simulate(d.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t, C.c_int64), n, 2, 7, 0,
                               m, None, _lib.ptr(up), _lib.ptr(lo), C.byref(tel)))
    wall = time.perf_counter() - t0
print(json.dumps({"n": n, "realisations": m, "seq": bool(os.environ.get("STK_SEQ_PERMUTATION")),
                  "gen_ms": tel.gen_ms, "total_ms": tel.total_ms, "wall_s": wall}))
