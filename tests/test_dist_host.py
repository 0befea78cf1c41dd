"""world_size-2 gloo tests (CPU) of the host logic of the multi-process path: unique-id
distribution, max-over-ranks timing, and the replicated control step being bitwise identical on
every rank."""
import os
import pickle
import socket
import tempfile

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import numpy as np
    import torch.distributed as dist

    import paper_2402_05302_b200 as ck
    from paper_2402_05302_b200 import dist_utils as du

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = du.broadcast_unique_id(lambda: ck.get_unique_id())
        t = du.max_over_ranks(1.5 + rank)
        # the same statistics reach every rank (in the device path they are bitwise identical)
        rng = np.random.default_rng(5)
        b = [int(x) for x in rng.integers(1, 100, size=4)]
        lsq = [float(x) for x in rng.uniform(1.0, 3.0, size=4)]
        models = [(0.001 * (i + 1), 0.01, 0.002, 0.02) for i in range(4)]
        est, split = du.control_step(lsq, 1.2, b, models, (0.2, 0.05, 0.01), 321)
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump({"uid": uid, "t": t, "est": est, "split": split}, f)
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        res = [pickle.load(open(os.path.join(d, f"r{r}.pkl"), "rb")) for r in range(world)]
    assert res[0]["uid"] == res[1]["uid"] and len(res[0]["uid"]) == 128
    assert res[0]["t"] == res[1]["t"] == 2.5
    assert res[0]["est"] == res[1]["est"]          # bitwise identical dicts of floats
    assert res[0]["split"] == res[1]["split"]
    assert sum(res[0]["split"]["b"]) == 321
