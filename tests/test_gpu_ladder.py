"""The S1-S5 reproducibility ladder on the device engine (needs a B200).

Mirrors the reference's scenario tests (test_scenarios.py:63-159) and pins
them to tests/golden/ladder.json, which the reference itself produced
(gen_golden.py:gen_ladder): for every mode and level, both runs' per-step
parameter hashes, the second run's per-step losses, and the bitdiff verdict
(first divergent step, field and worker) must be identical.  Each restart
segment is one persistent launch; restarts are in-memory apply_layout.
"""

import pytest
import torch

from golden_util import fhl, hf, load

pytestmark = pytest.mark.gpu

DOC = load("ladder.json")


@pytest.fixture(scope="module")
def bt():
    import paper_2208_14228_b200 as pkg
    from paper_2208_14228_b200 import _native

    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    _native.lib()
    return pkg


def _cfg(bt, mode):
    c = DOC["config"]
    return bt.TrainRunConfig(seed=c["seed"], max_workers=c["max_workers"], micro_batch=c["micro_batch"],
                             dataset_size=c["dataset_size"], lr=hf(c["lr"]), momentum=hf(c["momentum"]),
                             dropout_rate=hf(c["dropout_rate"]), jitter=hf(c["jitter"]),
                             bucket_capacity=c["bucket_capacity"], determinism=bt.DeterminismMode.from_label(mode),
                             device_fanins=DOC["kinds"])


def _spec(bt, d):
    lay = tuple(bt.ExecutorSpec(k) for k in d["layout"])
    return bt.RunSpec(lay, tuple(bt.RestartEvent(s, tuple(bt.ExecutorSpec(k) for k in ks)) for s, ks in d["restarts"]))


def _check_pair(bt, cfg, want):
    from paper_2208_14228_b200.runlog import bitdiff

    steps = DOC["steps"]
    la, ta = bt.run_training(cfg, _spec(bt, want["run_a"]), steps)
    lb, tb = bt.run_training(cfg, _spec(bt, want["run_b"]), steps)
    assert [r.param_hash for r in la.records] == want["hash_a"]
    assert [r.param_hash for r in lb.records] == want["hash_b"]
    assert [fhl(r.losses) for r in lb.records] == want["losses_b"]
    d = bitdiff(la, lb)
    got = None if d is None else {"step": d.step, "field": d.field, "worker": d.worker}
    assert got == want["divergence"]
    assert (ta.executors[0].model.values == tb.executors[0].model.values) == want["final_equal"]


@pytest.mark.parametrize("mode", ["d0", "d1", "d1d2"])
def test_ladder_levels_match_reference(bt, mode):
    cfg = _cfg(bt, mode)
    for lv in DOC["matrix"][mode]["levels"]:
        _check_pair(bt, cfg, lv)


@pytest.mark.parametrize("mode", ["d0", "d1", "d1d2"])
def test_run_matrix_guarantees(bt, mode):
    from paper_2208_14228_b200.scenarios import default_matrix, guaranteed_levels, run_matrix

    want = DOC["matrix"][mode]
    assert sorted(guaranteed_levels(mode)) == want["guaranteed"]
    rep = run_matrix(_cfg(bt, mode), default_matrix("gpu_a", "gpu_b", DOC["steps"]), DOC["steps"])
    assert rep.failed_guarantees() == want["failed_guarantees"] == []
    assert [r.bitwise_equal for r in rep.results] == [lv["divergence"] is None and lv["final_equal"]
                                                      for lv in want["levels"]]


@pytest.mark.parametrize("mode", ["d1", "d1d2"])
def test_staged_kind_change(bt, mode):
    """d1 diverges exactly at the first mixed-kind step (12); d1d2 never does."""
    _check_pair(bt, _cfg(bt, mode), DOC["staged"][mode])


def test_randomized_restart_schedules(bt):
    for r in DOC["random"]:
        _check_pair(bt, _cfg(bt, r["mode"]), r)
