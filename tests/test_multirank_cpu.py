"""N>1 path on CPU (gloo, world_size 2): batch sharding, per-rank work on each shard, gather to
rank 0 and max-over-ranks timing — the same host logic bench.py runs under torchrun on GPUs.
Each rank runs the (CPU) oracle on its shard; rank 0 checks the gathered result equals one
oracle run over the whole batch (sequences are independent: no exchange step)."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import os, sys, time
sys.path.insert(0, {root!r}); sys.path.insert(0, {oracle!r})
import numpy as np, torch, torch.distributed as dist
import oracle
from paper_2505_03780_b200 import parallel, workload as W
dist.init_process_group("gloo")
world, rank = dist.get_world_size(), dist.get_rank()
shape = dict(W.C4, batch_size=6, seq_len=200, num_q_heads=16, num_kv_heads=2)
d = W.make_decode(shape, device="cpu", lens=[200, 17, 1, 130, 64, 199], extra_blocks=2)
counts = [parallel.shard_range(6, world, r).count for r in range(world)]
sh = parallel.shard_range(6, world, rank)
sl = slice(sh.start, sh.start + sh.count)
t0 = time.perf_counter()
out = torch.from_numpy(oracle.decode(d.q[sl], d.k_cache, d.v_cache, d.block_table[sl], d.seq_lens[sl]))
ms = (time.perf_counter() - t0) * 1e3
ms_max = parallel.max_over_ranks(ms)
assert ms_max >= ms
full = parallel.gather_to_rank0(out, counts)
# prefill sharding by kv-head group
groups = list(parallel.kv_head_groups(8, world, rank))
assert len(groups) == 4 and groups[0] == 4 * rank
if rank == 0:
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    assert full.shape == ref.shape
    assert np.abs(full.numpy() - ref).max() == 0.0
    v = parallel.weak_scaling_value(1e9, 10, ms_max, world, 1e9)
    assert v > 0
    print("RANK0_OK", counts, round(ms_max, 3))
dist.barrier()
dist.destroy_process_group()
'''


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_shard_gather_max():
    script = WORKER.format(root=str(ROOT), oracle=str(ROOT / "oracle"))
    port = free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE="2", RANK=str(r),
                   LOCAL_RANK=str(r), OMP_NUM_THREADS="1")
        procs.append(subprocess.Popen([sys.executable, "-c", script], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    assert "RANK0_OK" in outs[0][0]


@pytest.mark.parametrize("total,world", [(256, 8), (64, 3), (5, 8), (1, 1)])
def test_shard_range_partitions(total, world):
    from paper_2505_03780_b200.parallel import shard_range
    shards = [shard_range(total, world, r) for r in range(world)]
    assert sum(s.count for s in shards) == total
    pos = 0
    for s in shards:
        assert s.start == pos
        pos += s.count
    assert max(s.count for s in shards) - min(s.count for s in shards) <= 1
