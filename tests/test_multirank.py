"""CPU multi-process tests of the N>1 path (gloo, world size 2 and 3).

The multi-GPU sweep deals the 64-plan chunks of its work list (every row's
plan-index space, rows in list order) round-robin over the ranks
(cg_shard_row_plans restates the device filter's mapping, shard_global_chunk),
each rank reduces its chunks to per-budget bests (cg_merge_budget_bests: the
rule of the device atomicMin + tie resolve), one all-gather exchanges them and
every rank merges with the reference's tie-break (merge_take, shared by the
device merge kernel and cg_merge_row_shards).  Here the engine library decides
which plans each rank owns and performs both merges; the per-chunk bests come
from the C oracle (no GPU here); the exchange is a real torch.distributed
all-gather over gloo, and the merged rows must equal the unsharded rows bit
for bit.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cpy
from parity_util import diff_json
from paper_2506_04203_b200 import engine as eng
from paper_2506_04203_b200 import workloads as W

pytestmark = pytest.mark.skipif(not cpy.available(), reason="oracle not built")

HW = dict(W.hardware(8), gpus_per_node=4)
PARAMS = dict(W.DEFAULT_COST_MODEL, queueing_sim_requests=300)
CASES = [
    ("small-7b", {"arrival_rate": 0.8, "mean_input_tokens": 200.0, "mean_output_tokens": 80.0,
                  "p95_input_tokens": 600.0, "p95_output_tokens": 240.0}, 8),
    ("small-7b", {"arrival_rate": 0.05, "mean_input_tokens": 300.0, "mean_output_tokens": 10.0,
                  "p95_input_tokens": 900.0, "p95_output_tokens": 30.0}, 7),   # light load: many ties
    ("mid-70b", {"arrival_rate": 0.3, "mean_input_tokens": 400.0, "mean_output_tokens": 100.0,
                 "p95_input_tokens": 1200.0, "p95_output_tokens": 300.0}, 8),
]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # one work list holding the three rows, in order (chunk offsets matter)
        totals = [cpy.row_shard(HW, PARAMS, W.model_spec(m, 1), wl, N, 0, 0)[2] for m, wl, N in CASES]
        for ci, (mname, wl, N) in enumerate(CASES):
            model = W.model_spec(mname, 1)
            parts = [cpy.row_shard(HW, PARAMS, model, wl, N, lo, hi)
                     for lo, hi in eng.shard_row_plans(totals, ci, rank, world)]
            none = np.full(N + 1, np.iinfo(np.uint64).max, dtype=np.uint64)
            lat = np.stack([p[0] for p in parts]) if parts else none[None]
            pid = np.stack([p[1] for p in parts]) if parts else none[None]
            bits, idx = eng.merge_budget_bests(HW, PARAMS, model, N, lat, pid)
            mine = torch.from_numpy(np.stack([bits.view(np.int64), idx.view(np.int64)]))
            gathered = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(gathered, mine)
            lat = np.stack([g[0].numpy().view(np.uint64) for g in gathered])
            pid = np.stack([g[1].numpy().view(np.uint64) for g in gathered])
            merged = eng.merge_row_shards(HW, PARAMS, model, N, lat, pid)
            results[(rank, ci)] = merged
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_rows_merge_to_the_unsharded_row(world):
    mgr = mp.Manager()
    results = mgr.dict()
    port = free_port()
    mp.spawn(worker, args=(world, port, results), nprocs=world, join=True)
    for ci, (mname, wl, N) in enumerate(CASES):
        full = cpy.row(HW, PARAMS, W.model_spec(mname, 1), wl, N)
        for rank in range(world):
            got = results[(rank, ci)]
            assert not diff_json(got, full), (world, rank, ci, diff_json(got, full)[:3])


def test_shard_row_plans_partition_every_row():
    lists = [[0], [1], [7], [1000], [490772], [64, 0, 65, 129, 3], [5000, 7, 0, 64 * 13]]
    for num_plans in lists:
        nchunks = sum((p + 63) // 64 for p in num_plans)
        for world in (1, 2, 3, 8):
            owned = [0] * world
            for row, P in enumerate(num_plans):
                cover = np.zeros(P, dtype=np.int32)
                for rank in range(world):
                    rs = eng.shard_row_plans(num_plans, row, rank, world)
                    assert rs == sorted(rs)
                    for lo, hi in rs:
                        assert 0 <= lo < hi <= P and (hi - lo == 64 or hi == P) and lo % 64 == 0
                        cover[lo:hi] += 1
                        owned[rank] += 1
                assert (cover == 1).all(), (num_plans, row, world)
            # chunks are dealt round-robin: shares differ by at most one chunk
            assert sum(owned) == nchunks and max(owned) - min(owned) <= 1
