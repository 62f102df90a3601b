"""CPU multi-process tests of the N>1 path (gloo, world size 2 and 3).

The multi-GPU sweep shards every row's plan-index space with a static
contiguous split (cg_shard_range), each rank reduces its shard to per-budget
bests, one all-gather exchanges them and every rank merges with the
reference's tie-break (merge_take, shared by the device merge kernel and
cg_merge_row_shards).  Here the shards are evaluated by the C oracle, the
exchange is a real torch.distributed all-gather over gloo, and the merged
row must equal the unsharded row bit for bit.
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
        for ci, (mname, wl, N) in enumerate(CASES):
            model = W.model_spec(mname, 1)
            _, _, total = cpy.row_shard(HW, PARAMS, model, wl, N, 0, 0)
            lo, hi = eng.shard_range(total, rank, world)
            bits, idx, _ = cpy.row_shard(HW, PARAMS, model, wl, N, lo, hi)
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


def test_shard_ranges_partition_the_items():
    for total in (0, 1, 7, 1000, 490772):
        for world in (1, 2, 3, 8):
            spans = [eng.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
