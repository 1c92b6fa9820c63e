"""World-size-2 run of the N>1 path with the PRODUCT decoder: two ranks
(gloo for the tally all-reduce; both ranks on cuda:0 -- only one GPU is
available here, and the ranks never wait on each other inside a kernel: the
data path has no collective) decode disjoint frame shards through
decode_batch, reduce their tallies, and must equal one process decoding both
shards."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, kind, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2102_11089_b200 import dist as D
    from paper_2102_11089_b200.channel import llr_batch
    from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, results_to_numpy
    from tests.util import load_code
    spec, g = load_code("C1")
    start, count = D.shard(per_rank)
    llr = torch.from_numpy(llr_batch(spec, 2.0, 0, start, count)).cuda()
    cfg = ScheduleConfig(kind=kind, i_max=3, n_p=4)
    r = results_to_numpy(decode_batch(spec, llr, cfg), kind, 3)
    t = D.Tally(3).add(r).reduce()
    if rank == 0:
        out.put((t.frames, t.frame_errors, t.bit_errors, t.propagations, t.counters.tolist(),
                 t.frame_errors_at.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["cirbp", "me_cirbp", "layered"])
def test_two_rank_product_decoder_matches_single_process(kind):
    per_rank = 3000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, per_rank, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_2102_11089_b200 import dist as D
    from paper_2102_11089_b200.channel import llr_batch
    from paper_2102_11089_b200.schedules import ScheduleConfig, decode_batch, results_to_numpy
    from tests.util import load_code
    spec, g = load_code("C1")
    llr = torch.from_numpy(llr_batch(spec, 2.0, 0, 0, 2 * per_rank)).cuda()
    ref = D.Tally(3).add(results_to_numpy(decode_batch(spec, llr, ScheduleConfig(kind=kind, i_max=3, n_p=4)),
                                          kind, 3))
    assert got[0] == ref.frames == 2 * per_rank
    assert got[1:4] == (ref.frame_errors, ref.bit_errors, ref.propagations)
    assert got[4] == ref.counters.tolist()
    assert got[5] == ref.frame_errors_at.tolist()
