"""C4 across processes: the per-EST BERT step sharded by EST block over 2 processes (the 2-GPU
mapping; both share this run's one B200 -- CUDA IPC works across processes on one device), with the
exchange done by the peer-memory reducer (paper_2208_14228_b200.peer: Tree(2) hierarchical partials /
Sequential owner-computes, NVLink peer loads and stores on a multi-GPU box).  Weights on both ranks and
every EST's loss must equal the single-process run bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CFG = dict(ests=4, seqs=1, layers=2, d_model=256, heads=4, d_ff=512, seed=9, lr=0.01)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fanin, q, optimizer="sgd"):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch.distributed as dist

    from paper_2208_14228_b200.bert import BertJob

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n = CFG["ests"] // world
        job = BertJob(fanin=fanin, est_base=rank * n, est_count=n, optimizer=optimizer, **CFG)
        job.attach_peer()
        losses = [job.step().cpu().numpy().tobytes() for _ in range(3)]
        torch.cuda.synchronize()
        dist.barrier()
        q.put((rank, job.params.cpu().numpy().tobytes(), losses))
        dist.barrier()
        job.peer.close()
    except Exception:
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fanin,optimizer", [(2, "sgd"), (0, "sgd"), (2, "adam")])
def test_two_process_bert_matches_one_process(fanin, optimizer):
    import torch.multiprocessing as mp

    from paper_2208_14228_b200.bert import BertJob

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fanin, q, optimizer)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in procs:
            r, pb, losses = q.get(timeout=240)
            assert pb != "error", losses
            res[r] = (pb, losses)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    ref = BertJob(fanin=fanin, optimizer=optimizer, **CFG)
    ref_losses = [ref.step().cpu().numpy() for _ in range(3)]
    want = ref.params.cpu().numpy().tobytes()
    for r in (0, 1):
        assert res[r][0] == want, r
        for step in range(3):
            got = np.frombuffer(res[r][1][step], dtype=np.float32)
            assert got.tobytes() == ref_losses[step][2 * r:2 * r + 2].tobytes(), (r, step)


def _bench_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        out = bench.bench_bert_dist(rank, world, dist, ests=4, steps=2, warmup=1, seqs=1, layers=2, d_model=256,
                                    heads=4, d_ff=512)
        out2 = bench.bench_resnet_dist(rank, world, dist, ests=4, batch=2, steps=2, warmup=1)
        q.put((rank, {"bert": out, "resnet": out2}))
    except Exception:
        import traceback

        q.put((rank, {"error": traceback.format_exc()}))
    finally:
        dist.destroy_process_group()


def test_bench_multi_gpu_model_stack_legs():
    """bench.py's N>1 C4 and C3 legs (what the driver's scaling run executes), on 2 processes here."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        outs = [q.get(timeout=240) for _ in procs]
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, outd in outs:
        assert "error" not in outd, outd
        for out in outd.values():
            assert out["replicas_bit_identical"] and out["ests_per_gpu"] == 2 and out["samples_per_s"] > 0
