"""Multi-process G-rank reducer over CUDA IPC + stream memory ops (paper_2208_14228_b200.peer).

Two processes share the one B200 of this run (IPC works across processes on
the same device); each maps the other's slots, partial, replica and signal
words, and the reduce-scatter / update / all-gather move data through those
peer pointers with device-side ordering only.  Both replicas must equal the
single-GPU reducer bit for bit, over several steps.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, variant, q, nonfinite=False):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    from paper_2208_14228_b200.hier import RankBuffers
    from paper_2208_14228_b200.peer import PeerGroupReducer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(rank, world, variant, q, dist, RankBuffers, PeerGroupReducer, nonfinite)
    except Exception:  # report instead of leaving the parent waiting on the queue
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(rank, world, variant, q, dist, RankBuffers, PeerGroupReducer, nonfinite=False):
    if True:
        E, n = 8, 20_003
        rng = np.random.default_rng(11)
        grads = (rng.uniform(-1, 1, (E, n)) * 10.0 ** rng.integers(-12, 13, (E, n))).astype(np.float32)
        if nonfinite:  # rank 1's slot, an element of rank 0's parameter shard
            grads[6, 100] = np.nan
        p0 = rng.uniform(-1, 1, n).astype(np.float32)
        E_loc = E // world
        torch.cuda.set_device(0)
        loc = RankBuffers(torch.from_numpy(grads[rank * E_loc:(rank + 1) * E_loc].copy()).cuda(),
                          torch.from_numpy(p0.copy()).cuda(), torch.zeros(n, dtype=torch.float32, device="cuda"),
                          torch.cuda.Stream())
        red = PeerGroupReducer(loc, E, variant, None, 0.05, 0.9)
        for _ in range(1 if nonfinite else 3):
            red.step()
        torch.cuda.synchronize()
        if nonfinite:
            from paper_2208_14228_b200.errors import NumericError

            try:
                red.check()
                raise AssertionError("no NumericError")
            except NumericError:
                pass
        else:
            red.check()
        dist.barrier()
        q.put((rank, loc.param.cpu().numpy().tobytes(), loc.vel.cpu().numpy().tobytes()))
        dist.barrier()
        red.close()


@pytest.mark.parametrize("variant", ["rank_tree2", "sequential"])
def test_two_process_ipc_reducer(oracle, variant):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in procs:
            r, pb, vb = q.get(timeout=120)
            assert pb != "error", vb
            res[r] = (pb, vb)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    E, n = 8, 20_003
    rng = np.random.default_rng(11)
    grads = (rng.uniform(-1, 1, (E, n)) * 10.0 ** rng.integers(-12, 13, (E, n))).astype(np.float32)
    p = rng.uniform(-1, 1, n).astype(np.float32)
    v = np.zeros(n, np.float32)
    for _ in range(3):
        p, v = oracle.reduce_update(grads, None, "tree2" if variant == "rank_tree2" else "seq", p, v, 0.05, 0.9)
    for r in (0, 1):
        assert res[r][0] == p.tobytes() and res[r][1] == v.tobytes()


def _trainer_worker(rank, world, port, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    from paper_2208_14228_b200.dist import DistributedTrainer
    from paper_2208_14228_b200.runlog import param_fingerprint

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        tr = DistributedTrainer(seed=42, max_workers=8, micro_batch=4, dataset_size=1024, exchange="ipc")
        hashes, losses = [], []
        for _ in range(40):
            losses.append(tr.step().cpu().numpy().tobytes())
            hashes.append(param_fingerprint(tr.params[0].cpu().numpy().tobytes()))
        tr.check()
        dist.barrier()
        q.put((rank, hashes, losses))
        dist.barrier()
        tr.peer.close()
    except Exception:
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_distributed_trainer_over_ipc_matches_reference():
    """C2 with 4 ESTs per process, 2 processes, EST slots and replicas shared through CUDA IPC:
    the reference's own per-step param fingerprints and losses, on both ranks."""
    import struct

    import torch.multiprocessing as mp

    from golden_util import load

    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_trainer_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in procs:
            k, hashes, losses = q.get(timeout=180)
            assert hashes != "error", losses
            res[k] = (hashes, losses)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for k in (0, 1):
        assert res[k][0] == r["param_hash"][:40]
        for step, blob in enumerate(res[k][1]):
            got = [struct.pack("<d", v).hex() for v in struct.unpack(f"<{len(blob) // 8}d", blob)]
            assert got == r["losses"][step][4 * k: 4 * k + 4], (k, step)


@pytest.mark.parametrize("variant", ["rank_tree2", "sequential"])
def test_two_process_ipc_reducer_non_finite_changes_nothing(variant):
    """NaN in rank 1's EST slot, inside rank 0's parameter shard: rank 0's check fails, its status is
    published to rank 1 before either commits, and both replicas keep their bytes; both raise."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, variant, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in procs:
            r, pb, vb = q.get(timeout=120)
            assert pb != "error", vb
            res[r] = (pb, vb)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    rng = np.random.default_rng(11)
    E, n = 8, 20_003
    rng.uniform(-1, 1, (E, n)), rng.integers(-12, 13, (E, n))
    p = rng.uniform(-1, 1, n).astype(np.float32)
    for r in (0, 1):
        assert res[r][0] == p.tobytes() and res[r][1] == np.zeros(n, np.float32).tobytes()
