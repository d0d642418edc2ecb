"""The N>1 host path on CPU: world_size-2 gloo over 127.0.0.1.

Each rank computes its contiguous EST block's forward/backward (with the oracle
standing in for the device kernel -- this test checks the sharding and the
exchange, not the arithmetic), all-gathers the gradient slots through
paper_2208_14228_b200.dist.SlotExchange, applies the reference allreduce + SGD
(oracle) to the gathered slots, and must end with exactly the weights of the
single-process reference run -- the layout-invariance property of the step.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2208_14228_b200.dist import est_block


def test_est_block_matches_assign_ranks():
    from paper_2208_14228_b200.engine import ExecutorSpec, assign_ranks

    for E in (1, 4, 7, 8, 16, 33):
        for G in range(1, min(E, 8) + 1):
            ref = assign_ranks([ExecutorSpec("x")] * G, E)
            assert [est_block(g, G, E) for g in range(G)] == [(r[0], len(r)) for _, r in ref]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, E, B, steps, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import oracle as orc

    from paper_2208_14228_b200.dist import SlotExchange, est_block

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seed, n = 42, 256
        base, count = est_block(rank, world, E)
        xchg = SlotExchange(E, 161)
        data = orc.make_dataset(seed, n)
        params = orc.init_random(seed)
        vel = np.zeros(161)
        rng = [orc.derive_stream(0xD80F0D7A6B15EA5E, seed, base + k) for k in range(count)]
        stat = [(0.0, 0)] * count
        spe = n // (E * B)
        buckets = orc.buckets_initial(161, 64)
        for step in range(steps):
            epoch, local = divmod(step, spe)
            lists = orc.epoch_indices(seed, epoch, n, E, B)
            local_grads = np.zeros((count, 161))
            for k in range(count):
                est = base + k
                idx = lists[est][local * B:(local + 1) * B]
                w = orc.worker_rng(seed, epoch, local, est)
                xs, ys = [], []
                s = w
                for i in idx:
                    s, raw = (s + 0x9E3779B97F4A7C15) & (2**64 - 1), None
                    u = (orc.mix64(s) >> 11) * 2.0**-53
                    xs.append([v + (u - 0.5) * 0.1 for v in data[i][:8]])
                    ys.append(data[i][8])
                _, g, rng[k], m, c = orc.forward_backward(params, xs, ys, est, rng[k], stat[k][0], stat[k][1],
                                                          "tree2", 0.5)
                stat[k] = (m, c)
                local_grads[k] = g
            all_grads = xchg.allgather(torch.from_numpy(local_grads)).numpy()
            synced = orc.allreduce(all_grads, buckets, "tree2")
            params, vel = orc.sgd_step(params, vel, synced, 0.02, 0.9)
        q.put((rank, params.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("E,B,world", [(4, 2, 2), (5, 2, 2), (8, 4, 2)])
def test_two_rank_gloo_matches_single_process(oracle, E, B, world):
    steps = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, E, B, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.Run(seed=42, max_workers=E, micro_batch=B, dataset_size=256, mode="d1", layout=("gpu_fast",))
    for _ in range(steps):
        ref.step()
    want = ref.state()["params"].tobytes()
    assert results[0] == want and results[1] == want
