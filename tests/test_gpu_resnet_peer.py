"""C3 across processes: the per-EST ResNet-18 step sharded by EST block over 2 processes (the 2-GPU
mapping; both share this run's one B200 through CUDA IPC), exchanging through the peer-memory reducer.
Weights, per-EST losses and every EST's BatchNorm running statistics must equal the single-process run
bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CFG = dict(ests=8, batch=4, seed=5, lr=0.05, gpus=1)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fanin, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch.distributed as dist

    from paper_2208_14228_b200.resnet import ResNetJob

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        n = CFG["ests"] // world
        job = ResNetJob(fanin=fanin, est_base=rank * n, est_count=n, **CFG)
        job.attach_peer()
        losses = [job.step().cpu().numpy().tobytes() for _ in range(2)]
        torch.cuda.synchronize()
        dist.barrier()
        st = job.est_state()
        q.put((rank, job.params.cpu().numpy().tobytes(), losses, st["run_mean"].cpu().numpy().tobytes(),
               st["run_var"].cpu().numpy().tobytes()))
        dist.barrier()
        job.peer.close()
    except Exception:
        import traceback

        q.put((rank, "error", traceback.format_exc(), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fanin", [2, 0])
def test_two_process_resnet_matches_one_process(fanin):
    import torch.multiprocessing as mp

    from paper_2208_14228_b200.resnet import ResNetJob

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, fanin, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in procs:
            r, pb, losses, rm, rv = q.get(timeout=300)
            assert pb != "error", losses
            res[r] = (pb, losses, rm, rv)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    ref = ResNetJob(fanin=fanin, **CFG)
    ref_losses = [ref.step().cpu().numpy() for _ in range(2)]
    st = ref.est_state()
    rm, rv = st["run_mean"].cpu().numpy(), st["run_var"].cpu().numpy()
    want = ref.params.cpu().numpy().tobytes()
    for r in (0, 1):
        assert res[r][0] == want, r
        for step in range(2):
            assert np.frombuffer(res[r][1][step], np.float32).tobytes() == ref_losses[step][4 * r:4 * r + 4].tobytes()
        assert res[r][2] == rm[4 * r:4 * r + 4].tobytes() and res[r][3] == rv[4 * r:4 * r + 4].tobytes()
