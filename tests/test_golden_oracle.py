"""Pin the CPU oracle against golden vectors captured from the reference itself.

Golden files: tests/golden/*.json, produced by tests/golden/gen_golden.py by
calling /root/reference/pkg/src/bittrain (the reference is pure Python).  The
oracle must reproduce every one bit-for-bit before it may check the CUDA path.
"""

import numpy as np
import pytest

from golden_util import fhl, hf, hfl, load, u64

MASK64 = 2**64 - 1


def test_splitmix64_published_and_reference_streams(oracle):
    # Published splitmix64 vectors for seed 0 (test_prng.py:29-34).
    assert oracle.splitmix64_stream(0, 2) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]
    for seed_hex, outs in load("prng.json")["splitmix64"].items():
        assert oracle.splitmix64_stream(int(seed_hex, 16), 50) == [int(o, 16) for o in outs]


def test_derive_stream_and_tags(oracle):
    doc = load("prng.json")
    for case in doc["derive_stream"]:
        assert oracle.derive_stream(*[int(w, 16) for w in case["words"]]) == u64(case["state"])
    tag_dropout = 0xD80F0D7A6B15EA5E
    assert [oracle.derive_stream(tag_dropout, 42, r) for r in range(64)] == [u64(h) for h in doc["dropout_stream_seed42"]]
    assert doc["dropout_stream_seed42"][0] == "c1df52a2d236c14c"
    for c in doc["worker_rng_seed42"]:
        assert oracle.worker_rng(42, c["epoch"], c["local"], c["worker"]) == u64(c["state"])


def test_fnv1a64_vectors(oracle):
    assert oracle.fnv1a64(b"") == 0xCBF29CE484222325
    assert oracle.fnv1a64(b"foobar") == 0x85944171F73967E8
    for c in load("prng.json")["fnv1a64"]:
        assert oracle.fnv1a64(bytes.fromhex(c["hex"])) == u64(c["hash"])


def test_shuffled_range_transcripts(oracle):
    for c in load("prng.json")["shuffled_range"]:
        assert oracle.shuffled_range(c["n"], u64(c["state"])) == c["perm"]


def test_layout_arrival_perm(oracle):
    for c in load("prng.json")["layout_arrival_perm"]:
        assert oracle.layout_arrival_perm(c["n"], [tuple(x) for x in c["layout"]]) == c["perm"]


def test_reduce_sum_all_shapes(oracle):
    for c in load("reduction.json")["cases"]:
        vals = hfl(c["values"])
        assert fhl([oracle.reduce_sum(vals, "seq")]) == [c["seq"]]
        for f in (2, 3, 4, 5, 8, 16):
            assert fhl([oracle.reduce_sum(vals, f"tree{f}")]) == [c[f"tree{f}"]], (len(vals), f)


def test_reduce_sum_preserves_negative_zero(oracle):
    assert fhl([oracle.reduce_sum([-0.0], "seq")]) == fhl([-0.0])
    assert fhl([oracle.reduce_sum([-0.0], "tree2")]) == fhl([-0.0])


def test_init_random(oracle):
    for seed, vals in load("model.json")["init_random"].items():
        assert fhl(oracle.init_random(int(seed))) == vals


def test_forward_backward_golden(oracle):
    for i, c in enumerate(load("model.json")["forward_backward"]):
        loss, grads, rng, mean, cnt = oracle.forward_backward(
            hfl(c["params"]), [hfl(r) for r in c["x"]], hfl(c["y"]), c["rank"], u64(c["rng"]),
            hf(c["stat_mean"]), c["stat_count"], c["variant"], hf(c["rate"]))
        assert fhl([loss]) == [c["out_loss"]], i
        assert fhl(grads) == c["out_grads"], i
        assert rng == u64(c["out_rng"]), i
        assert fhl([mean]) == [c["out_stat_mean"]] and cnt == c["out_stat_count"], i


def test_sgd_step_golden(oracle):
    for c in load("model.json")["sgd_step"]:
        po, vo = oracle.sgd_step(hfl(c["params"]), hfl(c["vel"]), hfl(c["grads"]), hf(c["lr"]), hf(c["mu"]))
        assert fhl(po) == c["out_params"] and fhl(vo) == c["out_vel"]


def test_sgd_rejects_non_finite(oracle):
    g = [0.0] * 161
    g[5] = float("nan")
    with pytest.raises(FloatingPointError):
        oracle.sgd_step([0.0] * 161, [0.0] * 161, g, 0.1, 0.9)


def test_buckets_initial(oracle):
    assert oracle.buckets_initial(5, 2) == ((4, 3), (2, 1), (0,))
    assert [len(b) for b in oracle.buckets_initial(161, 64)] == [64, 64, 33]


def test_allreduce_golden(oracle):
    for i, c in enumerate(load("allreduce.json")["cases"]):
        reps = [hfl(r) for r in c["replicas"]]
        out = oracle.allreduce(reps, [tuple(b) for b in c["buckets"]], c["variant"])
        assert fhl(out) == c["out"], i
        # The same result through the flat rotation-table formulation the CUDA reducer uses.
        rot = None if c["variant"] == "seq" else oracle.rotation_table(c["buckets"], len(reps), len(reps[0]))
        po, _ = oracle.reduce_update(np.array(reps), rot, c["variant"], np.zeros(len(out)),
                                     np.zeros(len(out)), -1.0, 0.0)
        assert fhl(po) == c["out"], i  # p - (-1)*(0*0+g) == g exactly


def test_dataset_and_epoch_indices(oracle):
    doc = load("sampling.json")
    ds = oracle.make_dataset(42, 1024)
    assert oracle.fnv1a64(ds.astype("<f8").tobytes()) == u64(doc["dataset_42_1024"]["fnv"])
    assert [fhl(r) for r in ds[:4]] == doc["dataset_42_1024"]["head"]
    assert [fhl(r) for r in oracle.make_dataset(42, 64)] == doc["dataset_42_64"]
    for c in doc["epoch_indices"]:
        assert oracle.epoch_indices(c["seed"], c["epoch"], c["n"], c["workers"], c["micro"], c["shuffle"]) == c["lists"]


def _run_from_doc(oracle, r):
    cfg = r["config"]
    run = oracle.Run(seed=cfg["seed"], max_workers=cfg["max_workers"], micro_batch=cfg["micro_batch"],
                     dataset_size=cfg["dataset_size"], lr=hf(cfg["lr"]), momentum=hf(cfg["momentum"]),
                     dropout_rate=hf(cfg["dropout_rate"]), jitter=hf(cfg["jitter"]),
                     bucket_capacity=cfg["bucket_capacity"], mode=cfg["determinism"], devices=cfg["devices"],
                     layout=tuple(r["layout"]["initial"]))
    return run


@pytest.mark.parametrize("name", ["c1_d1", "c2_d1", "c2_d1d2", "train_d1_yaml", "mixed_d1", "mixed_d1d2",
                                  "d0_restart", "d0_plain", "small_e16"])
def test_full_runs_bit_exact(oracle, name):
    r = next(x for x in load("runs.json")["runs"] if x["name"] == name)
    run = _run_from_doc(oracle, r)
    restarts = {s: lay for s, lay in r["layout"]["restarts"]}
    for step in range(r["steps"]):
        losses = run.step()
        assert fhl(losses) == r["losses"][step], (name, step)
        st = run.state()
        assert format(oracle.fnv1a64(st["params"].astype("<f8").tobytes()), "016x") == r["param_hash"][step]
        if step + 1 in restarts:
            run.relayout(tuple(restarts[step + 1]))
    st = run.state()
    assert fhl(st["params"]) == r["final_params"] and fhl(st["velocity"]) == r["final_velocity"]
    assert [[fhl([m])[0], int(c)] for m, c in zip(st["stat_mean"], st["stat_count"])] == r["final_stats"]
    assert [format(int(x), "016x") for x in st["rng"]] == r["final_dropout_rng"]


def _ladder_hashes(oracle, doc, mode, sp):
    c = doc["config"]
    run = oracle.Run(seed=c["seed"], max_workers=c["max_workers"], micro_batch=c["micro_batch"],
                     dataset_size=c["dataset_size"], lr=hf(c["lr"]), momentum=hf(c["momentum"]),
                     dropout_rate=hf(c["dropout_rate"]), jitter=hf(c["jitter"]),
                     bucket_capacity=c["bucket_capacity"], mode=mode, devices=doc["kinds"],
                     layout=tuple(sp["layout"]))
    restarts = {s: lay for s, lay in sp["restarts"]}
    hashes, losses = [], []
    for step in range(doc["steps"]):
        losses.append(fhl(run.step()))
        hashes.append(format(oracle.fnv1a64(run.state()["params"].astype("<f8").tobytes()), "016x"))
        if step + 1 in restarts:
            run.relayout(tuple(restarts[step + 1]))
    return hashes, losses


def test_ladder_runs_bit_exact(oracle):
    """Every run of the reference's S1-S5 ladder, staged and random schedules (ladder.json)."""
    doc = load("ladder.json")
    pairs = [(m, lv) for m, v in doc["matrix"].items() for lv in v["levels"]]
    pairs += list(doc["staged"].items()) + [(r["mode"], r) for r in doc["random"]]
    for mode, p in pairs:
        assert _ladder_hashes(oracle, doc, mode, p["run_a"])[0] == p["hash_a"]
        hb, lb = _ladder_hashes(oracle, doc, mode, p["run_b"])
        assert hb == p["hash_b"] and lb == p["losses_b"]


def test_oracle_threads_do_not_change_bits(oracle):
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    run = _run_from_doc(oracle, r)
    run.set_threads(4)
    for step in range(20):
        assert fhl(run.step()) == r["losses"][step]


def test_global_batch_path(oracle):
    doc = load("global_batch.json")
    c = doc["config"]
    run = oracle.Run(seed=c["seed"], max_workers=c["max_workers"], micro_batch=c["micro_batch"],
                     dataset_size=c["dataset_size"], layout=("gpu_fast",) * c["executors"])
    for s in doc["steps"]:
        losses = run.step(np.array([hfl(row) for row in s["rows"]]))
        assert fhl(losses) == s["losses"]
        assert fhl(run.state()["params"]) == s["params"]
