"""The reference API driving several GPUs from one process.

`placement.set_devices([0] * n)` gives the engine n logical devices on the one B200 of a test box:
every executor block gets its own replicas, EST slots, stream and exchange buffers, and the
lock-step multi-device kernel (bt_mlp.cu, n_dev > 1) stores EST slots into the other devices'
inboxes and signals their counters exactly as it does across NVLink; the seam path gathers slots
with peer copies.  Everything must reproduce the reference's own runs bit for bit, and an elastic
rescale across devices must equal the uninterrupted run.  (On a box with >= 2 GPUs the same tests
run with distinct GPUs via BT_TEST_DEVICES, e.g. "0,1,2,3".)
"""

import os

import numpy as np
import pytest
import torch

from golden_util import fhl, load

pytestmark = pytest.mark.gpu


def _devices(n):
    env = os.environ.get("BT_TEST_DEVICES")
    if env:
        devs = [int(x) for x in env.split(",")]
        return [devs[i % len(devs)] for i in range(n)]
    return [0] * n


@pytest.fixture(scope="module")
def bt():
    import paper_2208_14228_b200 as pkg
    from paper_2208_14228_b200 import _native

    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    _native.lib()
    return pkg


@pytest.fixture
def place():
    from paper_2208_14228_b200 import placement

    yield placement
    placement.set_devices(None)


def _cfg(bt, r):
    from test_gpu_parity import _cfg_from_doc

    return _cfg_from_doc(bt, r)


@pytest.mark.parametrize("ndev,nexec", [(2, 2), (4, 4), (8, 8), (2, 8), (4, 8)])
def test_c2_on_several_devices_matches_reference(bt, place, ndev, nexec):
    """C2 (8 ESTs): executors spread over 2/4/8 devices -> the reference's per-step losses and
    parameter fingerprints (the lock-step exchange kernel, one launch per device per run)."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    place.set_devices(_devices(ndev))
    spec = bt.RunSpec(tuple(bt.ExecutorSpec("gpu_fast") for _ in range(nexec)))
    log, ts = bt.run_training(_cfg(bt, r), spec, 100)
    assert len(ts.dev.shards) == ndev
    from paper_2208_14228_b200 import engine

    assert engine._xdev(ts) is not None  # the lock-step kernel, not the seam path
    assert [fhl(rec.losses) for rec in log.records] == r["losses"]
    assert [rec.param_hash for rec in log.records] == r["param_hash"]
    assert log.records[-1].param_hash == "cb363c5f8ef799aa"
    for ex in ts.executors:
        assert fhl(ex.model.values) == r["final_params"]
    assert [f"{c.dropout_rng:016x}" for c in ts.contexts] == r["final_dropout_rng"]
    assert f"{bt.fnv1a64(bt.checkpoint_save(ts)):016x}" == r["final_ckpt_fnv"]


@pytest.mark.parametrize("name", ["mixed_d1", "mixed_d1d2", "d0_restart", "train_d1_yaml", "small_e16"])
def test_reference_runs_on_two_devices(bt, place, name):
    """Mixed device kinds, d0 bucket rebuilds, restarts onto 3 executors, 16 ESTs over 3
    executors: the seam path across devices (and the lock-step one where it applies)."""
    from test_gpu_parity import _spec

    r = next(x for x in load("runs.json")["runs"] if x["name"] == name)
    place.set_devices(_devices(2))
    log, ts = bt.run_training(_cfg(bt, r), _spec(bt, r["layout"]), r["steps"])
    assert [fhl(rec.losses) for rec in log.records] == r["losses"]
    assert [rec.param_hash for rec in log.records] == r["param_hash"]
    assert fhl(ts.executors[0].model.values) == r["final_params"]
    assert [[fhl([c.stat.running_mean])[0], c.stat.update_count] for c in ts.contexts] == r["final_stats"]
    assert f"{bt.fnv1a64(bt.checkpoint_save(ts)):016x}" == r["final_ckpt_fnv"]


def test_run_minibatch_per_call_on_devices(bt, place):
    """The per-step API call over 4 devices (one lock-step launch per call) == the reference."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    place.set_devices(_devices(4))
    ts = bt.init_training(_cfg(bt, r), [bt.ExecutorSpec("gpu_fast")] * 4)
    for step in range(40):
        assert fhl(bt.run_minibatch(ts)) == r["losses"][step]
        assert bt.param_fingerprint(ts.executors[3].model.values) == r["param_hash"][step]


def test_rescale_8_4_2_across_devices_equals_uninterrupted(bt, place):
    """apply_layout moves EST slots and replicas between devices (slot-copy kernel over peer
    memory): 8 executors on 8 devices -> 4 on 4 -> 2 on 2 mid-run equals 1 device throughout."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    cfg = _cfg(bt, r)
    place.set_devices(_devices(8))
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * 8)
    got = list(bt.run_steps(ts, 30)[0])
    for n in (4, 2):
        place.set_devices(_devices(n))
        ts = bt.apply_layout(ts, [bt.ExecutorSpec("gpu_fast")] * n)
        assert len(ts.dev.shards) == n
        got += list(bt.run_steps(ts, 35)[0])
    assert [fhl(x) for x in got] == r["losses"]
    assert bt.param_fingerprint(ts.executors[1].model.values) == r["param_hash"][-1]
    # and back onto one device
    place.set_devices(_devices(1))
    one = bt.apply_layout(ts, [bt.ExecutorSpec("gpu_fast")])
    assert fhl(one.executors[0].model.values) == r["final_params"]


def test_spied_allreduce_sees_rank_ordered_slots_across_devices(bt, place, monkeypatch):
    """engine.allreduce is still the call site (reference test_engine.py:175-199): over 2 devices
    the spy receives every EST's gradient in rank order, and the result equals the fused path."""
    from paper_2208_14228_b200 import engine

    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    place.set_devices(_devices(2))
    ts = bt.init_training(_cfg(bt, r), [bt.ExecutorSpec("gpu_fast")] * 2)
    seen = []
    real = engine.allreduce

    def spy(replicas, bm, variant):
        seen.append(len(replicas))
        assert ts.contexts[0].pending_grads is not None and ts.contexts[3].pending_grads is None
        return real(replicas, bm, variant)

    monkeypatch.setattr(engine, "allreduce", spy)
    for step in range(5):
        assert fhl(bt.run_minibatch(ts)) == r["losses"][step]
    assert seen == [8] * 5
    assert bt.param_fingerprint(ts.executors[1].model.values) == r["param_hash"][4]


def test_tampered_replica_on_other_device_raises(bt, place):
    """A replica one ULP off on the second device: every device's launch-start check sees it and
    the step raises CorruptionError (reference test_engine.py:162-172)."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    place.set_devices(_devices(2))
    ts = bt.init_training(_cfg(bt, r), [bt.ExecutorSpec("gpu_fast")] * 2)
    bt.run_minibatch(ts)
    vals = ts.executors[1].model.values
    vals[7] = float(np.nextafter(vals[7], 2.0))
    with pytest.raises(bt.CorruptionError):
        bt.run_minibatch(ts)


def test_shard_placement_follows_assign_ranks(bt, place):
    cfg = bt.TrainRunConfig(seed=1, max_workers=16, micro_batch=4, dataset_size=1024,
                            determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_fast": 2})
    place.set_devices(_devices(4))
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * 8)
    assert [(sh.base, sh.count, sh.execs) for sh in ts.dev.shards] == [
        (0, 4, [0, 1]), (4, 4, [2, 3]), (8, 4, [4, 5]), (12, 4, [6, 7])]
    assert [str(ex.device) for ex in ts.executors] == [f"cuda:{d}" for d in _devices(4) for _ in range(2)]
