"""Host-side logic of the drop-in API that runs without a GPU.

Mirrors the reference's own unit tests for the pieces that are pure host
bookkeeping: determinism labels, rank assignment, bucket maps, the ESCK byte
format (against the reference's golden checkpoints), run logs and config
parsing.
"""

import struct

import pytest

from golden_util import load

import paper_2208_14228_b200 as bt
from paper_2208_14228_b200 import checkpoint as ck
from paper_2208_14228_b200.engine import assign_ranks, split_by_rank
from paper_2208_14228_b200.runlog import Divergence, RunLog, RunRecord, float_to_hex, hex_to_float, param_fingerprint


def test_determinism_labels():
    assert bt.DeterminismMode.from_label("d1d2").label == "d1d2"
    assert bt.DeterminismMode.from_label("D0").label == "d0"
    assert bt.DeterminismMode.from_label("d0d2").label == "d0d2"
    with pytest.raises(bt.ConfigError):
        bt.DeterminismMode.from_label("d3")
    with pytest.raises(bt.ConfigError):
        bt.DeterminismMode(d0=False, d1=True)


def test_assign_ranks():
    ex = bt.ExecutorSpec
    assert [r for _, r in assign_ranks([ex("a")] * 3, 4)] == [[0, 1], [2], [3]]
    assert [r for _, r in assign_ranks([ex("a", 3), ex("a", 1)], 4)] == [[0, 1, 2], [3]]
    assert [r for _, r in assign_ranks([ex("a")] * 8, 16)] == [[2 * i, 2 * i + 1] for i in range(8)]
    for bad in ([ex("a", 3), ex("a", 2)], [ex("a", 3), ex("a")], [ex("a", 0), ex("a", 4)], [], [ex("a")] * 5):
        with pytest.raises(bt.ConfigError):
            assign_ranks(bad, 4)


def test_split_by_rank():
    rows = [((float(i),) * 8, float(i)) for i in range(8)]
    micro = split_by_rank(rows, 4)
    assert micro[0] == [rows[0], rows[4]] and micro[3] == [rows[3], rows[7]]
    with pytest.raises(bt.ConfigError):
        split_by_rank(rows, 3)


def test_bucket_maps():
    assert bt.build_buckets_initial(5, 2).buckets == ((4, 3), (2, 1), (0,))
    assert [len(b) for b in bt.build_buckets_initial(161, 64).buckets] == [64, 64, 33]
    assert bt.rebuild_buckets_first_minibatch(list(range(6)), 3).buckets == ((0, 1, 2), (3, 4, 5))
    with pytest.raises(bt.InputError):
        bt.rebuild_buckets_first_minibatch([0, 1, 1, 3], 2)
    with pytest.raises(bt.InputError):
        bt.build_buckets_initial(5, 0)
    p1 = bt.layout_arrival_perm(161, [("gpu_a", 1)] * 4)
    assert p1 == bt.layout_arrival_perm(161, [("gpu_a", 1)] * 4) != bt.layout_arrival_perm(161, [("gpu_a", 2)] * 2)


def test_variants():
    assert bt.Sequential() == bt.Sequential()
    with pytest.raises(ValueError):
        bt.Tree(0)
    from paper_2208_14228_b200.reduction import fanin_code

    assert fanin_code(bt.Sequential()) == 0 and fanin_code(bt.Tree(3)) == 3
    with pytest.raises(bt.ConfigError):
        fanin_code(bt.Tree(1))
    assert bt.KernelProfile.device_agnostic("x").reduce_variant == bt.Sequential()


def test_esck_decode_encode_roundtrip_on_reference_blobs():
    for b in load("checkpoint.json")["blobs"]:
        blob = bytes.fromhex(b["blob"])
        doc = ck.decode_esck(blob)
        assert ck.encode_esck(doc) == blob
        assert len(doc["contexts"]) == b["workers"]
        assert doc["global_step"] == b["steps"]
        assert (doc["bucket_map"] is not None) == (b["mode"] != "d0")


def test_esck_context_wire_size_and_slope():
    assert ck.CONTEXT_WIRE_SIZE == 36
    d4 = ck.decode_esck(bytes.fromhex(load("checkpoint.json")["blobs"][0]["blob"]))
    more = d4 | {"contexts": d4["contexts"] + [(k, 0, 0.0, 0, 0) for k in range(4, 8)]}
    assert len(ck.encode_esck(more)) - len(ck.encode_esck(d4)) == 4 * ck.CONTEXT_WIRE_SIZE


def test_esck_errors_carry_offsets():
    blob = bytes.fromhex(load("checkpoint.json")["blobs"][0]["blob"])
    with pytest.raises(bt.FormatError) as e:
        ck.decode_esck(b"XXXX" + blob[4:])
    assert e.value.offset == 0
    with pytest.raises(bt.FormatError) as e:
        ck.decode_esck(blob[:-3])
    assert e.value.offset > 0
    with pytest.raises(bt.FormatError):
        ck.decode_esck(blob + b"\x00")
    bad = bytearray(blob)
    struct.pack_into("<I", bad, 4, 99)
    with pytest.raises(bt.VersionError):
        ck.decode_esck(bytes(bad))
    bad = bytearray(blob)
    struct.pack_into("<I", bad, 8, 160)
    with pytest.raises(bt.FormatError):
        ck.decode_esck(bytes(bad))


def test_esck_config_errors_fire_where_the_reference_reads_them():
    """checkpoint.py:152-177: a flag mismatch or a context-count mismatch is a ConfigError even when
    the bytes after it are malformed (the reference raises before parsing further)."""
    b = next(x for x in load("checkpoint.json")["blobs"] if x["mode"] != "d0")
    blob = bytes.fromhex(b["blob"])
    doc = ck.decode_esck(blob)
    cfg = bt.TrainRunConfig(seed=42, max_workers=b["workers"], determinism=bt.DeterminismMode.from_label(b["mode"]))
    other = bt.DeterminismMode.from_label("d0" if b["mode"] != "d0" else "d1")
    cfg_flags = bt.TrainRunConfig(seed=42, max_workers=b["workers"], determinism=other)
    cfg_count = bt.TrainRunConfig(seed=42, max_workers=b["workers"] + 1, determinism=cfg.determinism)
    assert ck.decode_esck(blob, cfg)["global_step"] == doc["global_step"]
    truncated = blob[: len(blob) - 40]  # a defect after the context count
    with pytest.raises(bt.FormatError):
        ck.decode_esck(truncated, cfg)
    with pytest.raises(bt.ConfigError):
        ck.decode_esck(truncated, cfg_flags)
    with pytest.raises(bt.ConfigError):
        ck.decode_esck(truncated, cfg_count)


def test_runlog_roundtrip_and_bitdiff(tmp_path):
    import math

    for v in (0.0, -0.0, 1.5, 2.0**-1074, math.pi, float("inf")):
        assert float_to_hex(hex_to_float(float_to_hex(v))) == float_to_hex(v)
    assert float_to_hex(0.0) != float_to_hex(-0.0)
    a = [0.1] * 161
    b = list(a)
    b[80] = math.nextafter(b[80], 1.0)
    assert param_fingerprint(a) != param_fingerprint(b)

    def mk(tweak=None, field="loss"):
        log = RunLog(2, "d1", 42)
        for s in range(1, 6):
            losses = [0.5 + s, 0.5 - s]
            ph = param_fingerprint([float(s)] * 4)
            if s == tweak and field == "loss":
                losses[1] = math.nextafter(losses[1], 100.0)
            if s == tweak and field == "param":
                ph = param_fingerprint([float(s) + 1] * 4)
            log.add(RunRecord(s, losses, ph, [float(s)] * 4 if s % 2 == 0 else None))
        return log

    base = mk()
    path = tmp_path / "run.log"
    base.dump(path)
    assert RunLog.load(path).to_lines() == base.to_lines()
    assert bt.bitdiff(base, mk()) is None
    assert bt.bitdiff(base, mk(3, "loss")) == Divergence(3, "loss", 1)
    assert bt.bitdiff(base, mk(4, "param")) == Divergence(4, "param_hash")


TRAIN_YAML = """
seed: 42
max_workers: 4
micro_batch: 4
dataset_size: 1024
minibatches: 200
lr: 0.02
momentum: 0.9
dropout_rate: 0.5
jitter: 0.1
bucket_capacity: 64
determinism: d1
devices: {gpu_fast: 2, gpu_mid: 3}
layout:
  - {device: gpu_fast}
  - {device: gpu_fast}
restarts:
  - after_step: 100
    layout: [{device: gpu_fast}, {device: gpu_fast}, {device: gpu_fast}]
"""


def test_configio_train_fixture(tmp_path):
    from paper_2208_14228_b200.configio import load_train_config

    p = tmp_path / "train_d1.yaml"
    p.write_text(TRAIN_YAML)
    cfg, spec, steps, dump_every = load_train_config(p)
    assert (cfg.seed, cfg.max_workers, cfg.micro_batch, cfg.dataset_size, steps) == (42, 4, 4, 1024, 200)
    assert cfg.determinism.label == "d1" and cfg.device_fanins == {"gpu_fast": 2, "gpu_mid": 3}
    assert len(spec.layout) == 2 and spec.restarts[0].after_step == 100 and len(spec.restarts[0].layout) == 3
    with pytest.raises(bt.ConfigError):
        from paper_2208_14228_b200.configio import parse_train_config

        parse_train_config({"seed": 1})


def test_guaranteed_levels_and_matrix_shape():
    from paper_2208_14228_b200.scenarios import default_matrix, guaranteed_levels

    assert guaranteed_levels("d0") == {"S1", "S2"}
    assert guaranteed_levels("d1") == {"S1", "S2", "S4"}
    assert guaranteed_levels("d1d2") == {"S1", "S2", "S3", "S4", "S5"}
    m = default_matrix("a", "b", 16)
    assert [s.level for s in m] == ["S1", "S2", "S3", "S4", "S5"]
    assert m[3].run_b.restarts[0].after_step == 8


def test_memory_model():
    from paper_2208_14228_b200.engine import executor_peak_mu, packing_peak_mu

    assert len({executor_peak_mu(t, 1.0) for t in range(1, 17)}) == 1
    assert packing_peak_mu(16, 1.0) > 16 > executor_peak_mu(16, 1.0)


def test_model_stack_est_blocks_follow_assign_ranks():
    """C3/C4 drivers place ESTs on GPUs with the reference's mapper (engine.py:169-199)."""
    import pytest

    from paper_2208_14228_b200.errors import ConfigError
    from paper_2208_14228_b200.resnet import est_blocks

    assert est_blocks(16, 8) == [(2 * g, 2) for g in range(8)]
    assert est_blocks(16, 4) == [(0, 4), (4, 4), (8, 4), (12, 4)]
    assert est_blocks(16, 3) == [(0, 6), (6, 5), (11, 5)]
    assert est_blocks(32, 1) == [(0, 32)]
    with pytest.raises(ConfigError):
        est_blocks(4, 5)
