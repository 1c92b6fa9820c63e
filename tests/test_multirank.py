"""World-size-2 gloo tests of the N>1 path (CPU): frame sharding (weak
scaling, disjoint Philox substreams), tally reduction and max-over-ranks
timing.  The decoder stand-in on CPU is the oracle (test infrastructure);
on GPUs bench.py runs the same plumbing with NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.cpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle
    from paper_2102_11089_b200 import dist as D
    from paper_2102_11089_b200.channel import llr_batch
    from tests.util import load_code
    spec, g = load_code("C0")
    start, count = D.shard(per_rank)
    llr = llr_batch(spec, 2.0, 0, start, count).astype(np.float64)
    r = pyoracle.decode_batch(g, llr, "cirbp", i_max=5, k_info=spec.k_info, threads=1)
    t = D.Tally(5).add(r).reduce()
    tmax = D.all_max([float(rank + 1)])
    if rank == 0:
        out.put((start, t.frames, t.frame_errors, t.bit_errors, t.propagations,
                 t.counters.tolist(), t.frame_errors_at.tolist(), float(tmax[0])))
    else:
        out.put(("rank1", start))
    dist.destroy_process_group()


def test_two_rank_sharding_matches_single_process():
    per_rank = 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, per_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = [x for x in got if x[0] != "rank1"][0]
    r1 = [x for x in got if x[0] == "rank1"][0]
    assert r0[0] == 0 and r1[1] == per_rank          # disjoint, consecutive shards
    # single process over both shards
    from oracle import pyoracle
    from paper_2102_11089_b200 import dist as D
    from paper_2102_11089_b200.channel import llr_batch
    from tests.util import load_code
    spec, g = load_code("C0")
    llr = llr_batch(spec, 2.0, 0, 0, 2 * per_rank).astype(np.float64)
    ref = D.Tally(5).add(pyoracle.decode_batch(g, llr, "cirbp", i_max=5, k_info=spec.k_info))
    assert r0[1] == ref.frames == 2 * per_rank
    assert r0[2] == ref.frame_errors
    assert r0[3] == ref.bit_errors
    assert r0[4] == ref.propagations
    assert r0[5] == ref.counters.tolist()
    assert r0[6] == ref.frame_errors_at.tolist()
    assert r0[7] == 2.0                                # max over ranks


def test_single_rank_defaults():
    from paper_2102_11089_b200 import dist as D
    assert D.world() == (0, 1)
    assert D.shard(10) == (0, 10)
    assert D.all_sum([1, 2]).tolist() == [1, 2]
