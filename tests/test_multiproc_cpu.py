"""CPU, world_size 2 over gloo: the multi-GPU exchange steps of rt.run_job.

Each rank owns a slice of the work exactly as on GPUs (contiguous block of
realisations; a 1/W slice of the observed pattern's pair work by input index);
the per-rank partial results are produced by the oracle here (no GPU), and
the two all-reduces (exact integer SUM of 128-bit fixed-point limbs, MAX/MIN
of envelopes) must reproduce the single-process answer bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, golden


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import port as orc
    from paper_1912_04753_b200.stripley import rt

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden("sample_result.npz")
    x, y, t, ring = g["x"], g["y"], g["t"], g["ring"]
    s, tv = g["s"], g["tv"]
    n = len(x)
    # observed pattern: this rank's centers (input index % world == rank)
    sel = np.arange(n) % world == rank
    idx = np.nonzero(sel)[0]
    parts = [orc.pair_histogram(x, y, t, ring, 0, 365, s, tv, centers=(int(i), int(i) + 1), threads=1)
             for i in idx]
    counts = sum(p["counts"].astype(object) for p in parts)
    tot = sum(p["sum_hi"].astype(object) * (1 << 64) + p["sum_lo"].astype(object) for p in parts)
    hi = np.array([[int(v) >> 64 for v in row] for row in tot], dtype=np.uint64)
    lo = np.array([[int(v) & ((1 << 64) - 1) for v in row] for row in tot], dtype=np.uint64)
    counts = counts.astype(np.uint64)
    c_all, hi_all, lo_all = rt.allreduce_exact(counts, hi, lo)
    # realisations: contiguous block
    sims = int(g["sims"])
    r0, r1 = rt.shard_range(sims, rank, world)
    ls = []
    for r in range(r0, r1):
        sx, sy, st = orc.generate_cstr(n, ring, 0, 365, int(g["seed"]) + r)
        ls.append(orc.estimate(sx, sy, st, ring, 0, 365, s, tv, threads=1)["l"])
    if ls:
        up, lw = orc.envelopes(np.stack(ls))
    else:
        up, lw = np.full(s.shape + tv.shape, -np.inf), np.full(s.shape + tv.shape, np.inf)
    up, lw = rt.allreduce_envelopes(up, lw)
    if rank == 0:
        np.savez(os.path.join(out_dir, "combined.npz"), counts=c_all, hi=hi_all, lo=lo_all,
                 upper=up, lower=lw)
    dist.destroy_process_group()


def test_two_rank_exchange_matches_single_process(tmp_path):
    from oracle import port as orc

    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    res = np.load(tmp_path / "combined.npz")
    g = golden("sample_result.npz")
    x, y, t, ring = g["x"], g["y"], g["t"], g["ring"]
    s, tv = g["s"], g["tv"]
    full = orc.pair_histogram(x, y, t, ring, 0, 365, s, tv)
    assert np.array_equal(res["counts"], full["counts"])
    assert np.array_equal(res["hi"], full["sum_hi"]) and np.array_equal(res["lo"], full["sum_lo"])
    # finalize of the combined exact sums reproduces the golden K
    hist = np.array([[orc_fixed(h, l) for h, l in zip(rh, rl)] for rh, rl in zip(res["hi"], res["lo"])])
    k = orc.finalize(hist, len(x), orc.area(ring), 365)
    assert np.array_equal(k, orc.finalize(full["hist"], len(x), orc.area(ring), 365))
    assert np.max(np.abs(k - g["k"]) / np.maximum(np.abs(g["k"]), 1e-300)) <= 1e-12
    assert np.max(np.abs(res["upper"] - g["upper"])) <= 1e-9 * np.max(np.abs(g["upper"]))
    assert np.max(np.abs(res["lower"] - g["lower"])) <= 1e-9 * np.max(np.abs(g["lower"]))


def orc_fixed(hi, lo):
    import oracle

    return oracle._load_port().orc_fixed_to_double(int(hi), int(lo))
