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


def _xdev_worker(rank, world, port, q):
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
        tr = DistributedTrainer(seed=42, max_workers=8, micro_batch=4, dataset_size=1024)
        assert tr.exchange == "xdev"
        losses, hashes = [], []
        for K in (1, 7, 32, 60):  # 100 mini-batches in lock-step launches of varying length
            out = tr.run(K).cpu().numpy()
            losses += [row[tr.base:tr.base + tr.count].tobytes() for row in out]
            hashes.append(param_fingerprint(tr.params[0].cpu().numpy().tobytes()))
        tr.check()
        dist.barrier()
        q.put((rank, hashes, losses))
        dist.barrier()
        tr.close()
    except Exception:
        import traceback

        q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_lockstep_multi_process_matches_reference(world):
    """The persistent lock-step kernel across processes (CUDA IPC inboxes + counters; the processes
    share this box's GPU): C2's 100 mini-batches in 4 launches per rank reproduce the reference's
    per-step losses and the fingerprints at every launch boundary, on every rank."""
    import struct

    import torch.multiprocessing as mp

    from golden_util import load

    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_xdev_worker, args=(k, world, port, q)) for k in range(world)]
    for p in procs:
        p.start()
    try:
        res = {}
        for _ in procs:
            k, hashes, losses = q.get(timeout=240)
            assert hashes != "error", losses
            res[k] = (hashes, losses)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    n = 8 // world
    for k in range(world):
        assert res[k][0] == [r["param_hash"][i] for i in (0, 7, 39, 99)]
        for step, blob in enumerate(res[k][1]):
            got = [struct.pack("<d", v).hex() for v in struct.unpack(f"<{len(blob) // 8}d", blob)]
            assert got == r["losses"][step][n * k: n * k + n], (k, step)


def test_bench_runs_n_ranks_when_asked():
    """`python bench.py --gpus 2` without a launcher spawns 2 ranks itself: the line reports
    n_gpus 2 and the same final-weight fingerprint as the 1-GPU run of the same steps."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    args = ["--steps", "20", "--warmup", "5", "--no-bert", "--no-reducer", "--cpu-seconds", "0"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    lines = {}
    for n in (1, 2):
        out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", str(n), *args], cwd=root, env=env,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-3000:]
        lines[n] = json.loads(out.stdout.strip().splitlines()[-1])
    assert lines[1]["n_gpus"] == 1 and lines[2]["n_gpus"] == 2
    assert lines[2]["config"]["exchange"] == "xdev"
    assert lines[2]["weights_fnv"] == lines[1]["weights_fnv"]
    assert lines[2]["value"] > 0 and lines[2]["e2e"]["value"] > 0
