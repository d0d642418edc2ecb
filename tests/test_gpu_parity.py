"""CUDA path vs the oracle and the reference's golden vectors (needs a B200).

Bar: bit-exact.  The reference is binary64 with a pinned evaluation order; the
sm_100a kernels use explicit round-to-nearest ops and restate the reference
libm's tanh, so every loss, gradient, parameter and statistic must match to
the last bit (tolerance 0 ulp) -- stronger than north_star's 1e-5 relative.
Every call goes through the C-ABI (include/bittrain_b200.h) via the package.
"""

import math

import numpy as np
import pytest
import torch

from golden_util import fhl, hf, hfl, load, u64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bt():
    import paper_2208_14228_b200 as pkg
    from paper_2208_14228_b200 import _native

    assert torch.cuda.is_available(), "GPU test on a box without CUDA"
    _native.lib()
    return pkg


def test_library_is_the_in_tree_build(bt):
    from paper_2208_14228_b200 import _native

    assert _native.LIB_PATH.exists()
    maps = open("/proc/self/maps").read()
    assert str(_native.LIB_PATH) in maps


def test_device_tanh_bitexact_vs_libm(bt, oracle):
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    rng = np.random.default_rng(7)
    x = np.concatenate([rng.uniform(-4, 4, 400_000), rng.uniform(-30, 30, 200_000), rng.uniform(-1e-3, 1e-3, 100_000),
                        rng.standard_normal(100_000) * 1e-9, np.array([0.0, -0.0, 22.0, -22.0, 1e-300, np.inf,
                                                                       -np.inf, 0.5 * math.log(2), 1.0, -1.0])])
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    _native.check(_native.lib().bt_tanh_f64(xd.data_ptr(), xd.numel(), out.data_ptr(), stream()))
    got = out.cpu().numpy()
    want = np.array([math.tanh(float(v)) for v in x])  # libm, as the reference's math.tanh (np.tanh is not libm)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_device_tanh_bitexact_vs_libm_wide(bt, oracle):
    """2e7 inputs over the ranges the step's pre-activations and tanh's internal
    divisions see, plus random bit patterns: the step kernels' branch-free tanh
    (with the unchecked fast division) equals host libm bit for bit."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    rng = np.random.default_rng(11)
    x = np.concatenate([rng.uniform(-3, 3, 8_000_000), rng.uniform(-25, 25, 4_000_000),
                        rng.uniform(-1.2, 1.2, 4_000_000), rng.uniform(-1e-6, 1e-6, 1_000_000),
                        (rng.standard_normal(1_000_000) * 2.0 ** rng.integers(-60, 6, 1_000_000)),
                        rng.integers(0, 2**63, 2_000_000, dtype=np.int64).view(np.float64)])
    x = x[~np.isnan(x)]
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    _native.check(_native.lib().bt_tanh_f64(xd.data_ptr(), xd.numel(), out.data_ptr(), stream()))
    got = out.cpu().numpy()
    want = oracle.libm_tanh(x)
    bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
    assert bad.size == 0, [(float(x[i]), float(got[i]), float(want[i])) for i in bad[:5]]


def test_splitmix64_counter_form_matches_stream(bt):
    from paper_2208_14228_b200.prng import draws

    for seed_hex, outs in load("prng.json")["splitmix64"].items():
        raw, uni = draws(int(seed_hex, 16), 0, 50)
        assert [v & (2**64 - 1) for v in raw.tolist()] == [int(o, 16) for o in outs]
    raw, uni = draws(42, 0, 20)
    assert fhl(uni.tolist()) == load("prng.json")["uniform01_seed42"]


def test_dataset_and_init_on_device(bt):
    doc = load("sampling.json")
    from paper_2208_14228_b200.sampling import make_dataset_device

    ds = make_dataset_device(42, 1024).cpu().numpy()
    assert f"{bt.fnv1a64(ds.astype('<f8').tobytes()):016x}" == doc["dataset_42_1024"]["fnv"]
    assert [fhl(r) for r in make_dataset_device(42, 64).tolist()] == doc["dataset_42_64"]
    for seed, vals in load("model.json")["init_random"].items():
        assert fhl(bt.ToyModel.init_random(int(seed)).values) == vals


def test_reduce_sum_shapes(bt):
    for c in load("reduction.json")["cases"]:
        vals = hfl(c["values"])
        assert fhl([bt.reduce_sum(vals, bt.Sequential())]) == [c["seq"]]
        for f in (2, 3, 4, 5, 8, 16):
            assert fhl([bt.reduce_sum(vals, bt.Tree(f))]) == [c[f"tree{f}"]]


def _variant(bt, tag):
    return bt.Sequential() if tag == "seq" else bt.Tree(int(tag[4:]))


def test_forward_backward_golden(bt):
    for i, c in enumerate(load("model.json")["forward_backward"]):
        m = bt.ToyModel(hfl(c["params"]))
        batch = [(tuple(hfl(x)), hf(y)) for x, y in zip(c["x"], c["y"])]
        loss, grads, rng, stat = bt.forward_backward(m, batch, c["rank"], u64(c["rng"]),
                                                     bt.TrackedStat(hf(c["stat_mean"]), c["stat_count"]),
                                                     _variant(bt, c["variant"]), hf(c["rate"]))
        assert fhl([loss]) == [c["out_loss"]], i
        assert fhl(grads) == c["out_grads"], i
        assert rng == u64(c["out_rng"]), i
        assert fhl([stat.running_mean]) == [c["out_stat_mean"]] and stat.update_count == c["out_stat_count"], i


def test_allreduce_golden(bt):
    for i, c in enumerate(load("allreduce.json")["cases"]):
        bm = bt.BucketMap(c["capacity"], tuple(tuple(b) for b in c["buckets"]))
        out = bt.allreduce([hfl(r) for r in c["replicas"]], bm, _variant(bt, c["variant"]))
        assert fhl(out) == c["out"], i


def test_sgd_step_golden(bt):
    for c in load("model.json")["sgd_step"]:
        m2, o2 = bt.sgd_step(bt.ToyModel(hfl(c["params"])), bt.OptState(hf(c["lr"]), hf(c["mu"]), hfl(c["vel"])),
                             hfl(c["grads"]))
        assert fhl(m2.values) == c["out_params"] and fhl(o2.velocity) == c["out_vel"]


def test_sgd_rejects_non_finite(bt):
    g = [0.0] * 161
    g[5] = math.inf
    m = bt.ToyModel.init_random(1)
    with pytest.raises(bt.NumericError):
        bt.sgd_step(m, bt.OptState.fresh(0.1, 0.9), g)


def test_pipeline_batches_golden(bt):
    docs = load("sampling.json")["pipeline_batches"]
    for nw in (4, 8):
        pipe = bt.DataPipeline(42, 1024, nw, 4, jitter=0.1, worker_slots=2, prefetch_depth=2)
        want = {(d["step"], d["est"]): d["rows"] for d in docs if d["workers"] == nw}
        for step in range(pipe.steps_per_epoch + 2):
            for est in range(nw):
                rows = pipe.batch(est, step)
                if (step, est) in want:
                    assert [fhl(list(x) + [y]) for x, y in rows] == want[(step, est)], (nw, step, est)


def _cfg_from_doc(bt, r):
    c = r["config"]
    return bt.TrainRunConfig(seed=c["seed"], max_workers=c["max_workers"], micro_batch=c["micro_batch"],
                             dataset_size=c["dataset_size"], lr=hf(c["lr"]), momentum=hf(c["momentum"]),
                             dropout_rate=hf(c["dropout_rate"]), jitter=hf(c["jitter"]),
                             bucket_capacity=c["bucket_capacity"],
                             determinism=bt.DeterminismMode.from_label(c["determinism"]), device_fanins=c["devices"])


def _spec(bt, layout_doc):
    lay = tuple(bt.ExecutorSpec(k) for k in layout_doc["initial"])
    rs = tuple(bt.RestartEvent(s, tuple(bt.ExecutorSpec(k) for k in ks)) for s, ks in layout_doc["restarts"])
    return bt.RunSpec(lay, rs)


RUNS = ["c1_d1", "c2_d1", "c2_d1d2", "train_d1_yaml", "mixed_d1", "mixed_d1d2", "d0_restart", "d0_plain", "small_e16"]


@pytest.mark.parametrize("name", RUNS)
def test_full_run_bit_exact_vs_reference(bt, name):
    """Whole training runs (persistent fused kernel) vs the reference's own logs."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == name)
    log, ts = bt.run_training(_cfg_from_doc(bt, r), _spec(bt, r["layout"]), r["steps"])
    assert [fhl(rec.losses) for rec in log.records] == r["losses"]
    assert [rec.param_hash for rec in log.records] == r["param_hash"]
    assert fhl(ts.executors[0].model.values) == r["final_params"]
    assert fhl(ts.executors[0].opt.velocity) == r["final_velocity"]
    assert [[fhl([c.stat.running_mean])[0], c.stat.update_count] for c in ts.contexts] == r["final_stats"]
    assert [f"{c.dropout_rng:016x}" for c in ts.contexts] == r["final_dropout_rng"]
    assert f"{bt.fnv1a64(bt.checkpoint_save(ts)):016x}" == r["final_ckpt_fnv"]


@pytest.mark.parametrize("g", [1, 2, 4, 8])
def test_c2_layout_invariance_on_device(bt, g):
    """C2: 8 ESTs on 1/2/4/8 executors -> the same bits (cb363c5f8ef799aa)."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    spec = bt.RunSpec(tuple(bt.ExecutorSpec("gpu_fast") for _ in range(g)))
    log, ts = bt.run_training(_cfg_from_doc(bt, r), spec, 100)
    assert log.records[-1].param_hash == "cb363c5f8ef799aa"
    assert [rec.param_hash for rec in log.records] == r["param_hash"]


SHAPES = [  # (E, B, mode, layout kinds, dataset) -> exercises 1 CTA, multi-CTA grid barrier, generic-B path
    (16, 8, "d1", ("gpu_fast", "gpu_mid"), 1024),
    (64, 4, "d1", ("gpu_fast",) * 4, 2048),
    (12, 3, "d1d2", ("gpu_mid", "gpu_fast", "gpu_fast"), 600),
    (5, 7, "d0", ("gpu_mid",), 400),
    (32, 16, "d1", ("gpu_mid",) * 2, 4096),
    (2, 33, "d1", ("gpu_fast",), 700),
    (96, 2, "d1d2", ("gpu_mid", "gpu_fast"), 1000),  # slots too big for a cluster: grid-barrier launch
    (300, 4, "d1", ("gpu_fast",) * 3, 2400),  # slots too big for chip: grads kernel + reducer + sgd
]


@pytest.mark.parametrize("E,B,mode,layout,n", SHAPES)
def test_step_shapes_match_oracle(bt, oracle, E, B, mode, layout, n):
    cfg = bt.TrainRunConfig(seed=7, max_workers=E, micro_batch=B, dataset_size=n, lr=0.05, momentum=0.8,
                            dropout_rate=0.3, jitter=0.2, bucket_capacity=40,
                            determinism=bt.DeterminismMode.from_label(mode),
                            device_fanins={"gpu_fast": 2, "gpu_mid": 3})
    ts = bt.init_training(cfg, [bt.ExecutorSpec(k) for k in layout])
    ref = oracle.Run(seed=7, max_workers=E, micro_batch=B, dataset_size=n, lr=0.05, momentum=0.8, dropout_rate=0.3,
                     jitter=0.2, bucket_capacity=40, mode=mode, layout=layout)
    losses, trace = bt.run_steps(ts, 12, trace=True)
    for s in range(12):
        want = ref.step()
        assert np.array_equal(losses[s].view(np.uint64), want.view(np.uint64)), s
        assert np.array_equal(trace[s].view(np.uint64), ref.state()["params"].view(np.uint64)), s
    for _ in range(3):  # single-step launches continue the same trajectory
        assert fhl(bt.run_minibatch(ts)) == fhl(ref.step())
    st = ref.state()
    assert fhl(ts.executors[-1].model.values) == fhl(st["params"])
    assert [c.dropout_rng for c in ts.contexts] == [int(x) for x in st["rng"]]
    assert fhl([c.stat.running_mean for c in ts.contexts]) == fhl(st["stat_mean"])


def test_run_minibatch_matches_persistent_kernel(bt):
    """K single-step launches == one K-step persistent launch, bit for bit."""
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    cfg = _cfg_from_doc(bt, r)
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * 2)
    for step in range(40):
        assert fhl(bt.run_minibatch(ts)) == r["losses"][step]
        assert bt.param_fingerprint(ts.executors[0].model.values) == r["param_hash"][step]


def test_global_batch_path(bt):
    doc = load("global_batch.json")
    c = doc["config"]
    cfg = bt.TrainRunConfig(seed=c["seed"], max_workers=c["max_workers"], micro_batch=c["micro_batch"],
                            dataset_size=c["dataset_size"], determinism=bt.DeterminismMode.from_label("d1"),
                            device_fanins={"gpu_fast": 2, "gpu_mid": 3})
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * c["executors"])
    for s in doc["steps"]:
        rows = [(tuple(hfl(row[:8])), hf(row[8])) for row in s["rows"]]
        assert fhl(bt.run_minibatch(ts, rows)) == s["losses"]
        assert fhl(ts.executors[0].model.values) == s["params"]


def test_checkpoint_bytes_match_reference(bt):
    for b in load("checkpoint.json")["blobs"]:
        cfg = bt.TrainRunConfig(seed=42, max_workers=b["workers"], micro_batch=2, dataset_size=64,
                                determinism=bt.DeterminismMode.from_label(b["mode"]),
                                device_fanins={"gpu_fast": 2, "gpu_mid": 3})
        ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * b["executors"])
        for _ in range(b["steps"]):
            bt.run_minibatch(ts)
        blob = bt.checkpoint_save(ts)
        assert blob.hex() == b["blob"]
        ts2 = bt.checkpoint_restore(blob, [bt.ExecutorSpec("gpu_fast")] * 3, cfg)
        assert bt.checkpoint_save(ts2) == blob


def test_apply_layout_equals_byte_restart(bt):
    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    cfg = _cfg_from_doc(bt, r)
    a = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * 4)
    for _ in range(7):
        bt.run_minibatch(a)
    b = bt.checkpoint_restore(bt.checkpoint_save(a), [bt.ExecutorSpec("gpu_fast")] * 2, cfg)
    a = bt.apply_layout(a, [bt.ExecutorSpec("gpu_fast")] * 2)
    assert bt.checkpoint_save(a) == bt.checkpoint_save(b)
    for _ in range(5):
        assert bt.run_minibatch(a) == bt.run_minibatch(b)
    assert bt.checkpoint_save(a) == bt.checkpoint_save(b)


def test_tampered_replica_raises_corruption(bt):
    cfg = bt.TrainRunConfig(seed=42, max_workers=4, micro_batch=2, dataset_size=64,
                            determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_a": 2})
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_a")] * 2)
    bt.run_minibatch(ts)
    ts.executors[1].model.values[0] = math.nextafter(ts.executors[1].model.values[0], math.inf)
    with pytest.raises(bt.CorruptionError):
        bt.run_minibatch(ts)


def test_non_finite_gradient_raises_numeric(bt):
    cfg = bt.TrainRunConfig(seed=42, max_workers=4, micro_batch=2, dataset_size=64,
                            determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_a": 2})
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_a")])
    rows = [((1e308,) * 8, 1e308)] * 8
    before = ts.executors[0].model.values.tolist()
    with pytest.raises(bt.NumericError):
        bt.run_minibatch(ts, rows)
    assert ts.executors[0].model.values.tolist() == before
    assert ts.global_step == 0


def test_pending_grads_spy(bt, monkeypatch):
    """The engine calls allreduce through its module global (reference test_engine.py:175-199)."""
    import paper_2208_14228_b200.engine as engine_mod

    cfg = bt.TrainRunConfig(seed=42, max_workers=4, micro_batch=2, dataset_size=64,
                            determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_a": 2})
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_a")] * 2)
    ref = bt.init_training(cfg, [bt.ExecutorSpec("gpu_a")] * 2)
    observed = {}
    real = engine_mod.allreduce

    def spy(replicas, bm, variant):
        observed["pending"] = [None if c.pending_grads is None else list(c.pending_grads) for c in ts.contexts]
        observed["replicas"] = [list(r) for r in replicas]
        return real(replicas, bm, variant)

    monkeypatch.setattr(engine_mod, "allreduce", spy)
    losses = bt.run_minibatch(ts)
    monkeypatch.undo()
    assert observed["pending"][0] == observed["replicas"][0]
    assert observed["pending"][2] == observed["replicas"][2]
    assert observed["pending"][1] is None and observed["pending"][3] is None
    assert all(c.pending_grads is None for c in ts.contexts)
    # the unfused (spied) path and the fused kernel agree bit for bit
    assert losses == bt.run_minibatch(ref)
    assert ts.executors[0].model.values == ref.executors[0].model.values


def test_progress_error(bt):
    pipe = bt.DataPipeline(42, 64, 4, 2, jitter=0.1)
    pipe.batch(0, 0)
    with pytest.raises(bt.ProgressError):
        pipe.batch(0, 0)
    with pytest.raises(bt.ProgressError):
        pipe.batch(1, 3)


def test_distributed_trainer_single_rank_matches_reference(bt):
    """The N>1 code path (grads-only kernel -> all-gather -> fixed-order reduce kernel) run as a
    world-size-1 NCCL group reproduces the reference's C2 trajectory bit for bit."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2208_14228_b200.dist import DistributedTrainer

    r = next(x for x in load("runs.json")["runs"] if x["name"] == "c2_d1")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        tr = DistributedTrainer(seed=42, max_workers=8, micro_batch=4, dataset_size=1024, exchange="allgather")
        for step in range(40):
            losses = tr.step()
            assert fhl(losses.tolist()) == r["losses"][step], step
            assert bt.param_fingerprint(tr.params[0].cpu().numpy().tobytes()) == r["param_hash"][step], step
        tr.check()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rate", [0.0, 0.1, 0.5, 0.9, 1.0])
def test_dropout_mask_entry_point_matches_reference_draws(bt, oracle, rate):
    """bt_dropout_mask (model.py:151-161): one draw per (row, unit), rows outer, u < rate drops,
    kept units scaled by 1/(1-rate); no draws at rate 0; everything dropped at rate >= 1."""
    import ctypes as C

    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    state = derive = oracle.derive_stream(0xD80F0D7A6B15EA5E, 42, 5)
    rows, units = 37, 16
    out = torch.empty(rows * units, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_dropout_mask(state, rows, units, rate, out.data_ptr(), stream()))
    raw = np.array(oracle.splitmix64_stream(derive, rows * units), dtype=np.uint64)
    u = (raw >> np.uint64(11)).astype(np.float64) * 2.0**-53
    keep = 0.0 if rate >= 1.0 else 1.0 / (1.0 - rate)
    want = np.ones(rows * units) if rate == 0.0 else np.where(u < rate, 0.0, keep)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("dtype,es", [(0, 8), (1, 4)])
def test_allgather_params_entry_point_copies_bits(bt, dtype, es):
    """bt_allgather_params: the parameter all-gather as bit copies into every destination
    (engine.py:313-315), including a length that is not a multiple of the 16-byte vector."""
    import ctypes as C

    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    n = 10_003
    src = torch.randint(-2**31, 2**31 - 1, (n * es // 4,), dtype=torch.int32, device="cuda")
    dsts = [torch.zeros_like(src) for _ in range(5)]
    table = (C.c_void_p * 5)(*[d.data_ptr() for d in dsts])
    _native.check(_native.lib().bt_allgather_params(dtype, src.data_ptr(), table, 5, n, stream()))
    for d in dsts:
        assert torch.equal(d, src)


def test_run_steps_sampled_launch_equals_resident_lists(bt):
    """run_steps with host-made inputs (bt_mlp_run_sampled: the epoch lists computed by the native
    Fisher-Yates inside the C-ABI call, copied, then the launch) gives the bits of the launch that reads
    lists already resident on the device -- across epoch boundaries (32 mini-batches per epoch) and
    launches of 20 / 7 / 33 mini-batches; a launch whose staged epochs do not cover it is rejected."""
    import ctypes as C

    from paper_2208_14228_b200 import _native, engine

    def cfg():
        return bt.TrainRunConfig(seed=42, max_workers=8, micro_batch=4, dataset_size=1024, lr=0.02, momentum=0.9,
                                 dropout_rate=0.5, jitter=0.1, bucket_capacity=64,
                                 determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_fast": 2})

    a = bt.init_training(cfg(), [bt.ExecutorSpec("gpu_fast")])
    b = bt.init_training(cfg(), [bt.ExecutorSpec("gpu_fast")])
    for k in (20, 7, 33, 20):
        a.pipeline.drop_lists()  # host inputs every launch: the sampled path
        la, _ = engine.run_steps(a, k)
        spe = b.pipeline.steps_per_epoch
        b.pipeline.device_lists(b.global_step // spe, (b.global_step + k - 1) // spe)  # resident: bt_mlp_run
        lb, _ = engine.run_steps(b, k)
        assert np.array_equal(la.view(np.uint64), lb.view(np.uint64))
    pa = np.array(a.executors[0].model.values.tolist())
    pb = np.array(b.executors[0].model.values.tolist())
    assert np.array_equal(pa.view(np.uint64), pb.view(np.uint64))
    fs = engine._fast(a)
    fs.a.K, fs.a.step0 = 40, a.global_step  # crosses into an epoch that is not staged
    fs.a.losses = fs.io_ptr + 8 * (fs.KMAX - 40) * fs.E
    stage, lists = a.pipeline.reserve_lists(a.global_step // 32, 1)
    st = _native.lib().bt_mlp_run_sampled(C.byref(fs.a), 42, 1024, 1, a.global_step // 32, 1, stage, lists.data_ptr(),
                                          fs.host_io_ptr + 8 * (fs.KMAX - 40) * fs.E, None, None)
    assert st == 1  # InputError, nothing launched
    a.pipeline.drop_lists()


_SIGNAL_SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_2208_14228_b200 as bt
from paper_2208_14228_b200 import engine
cfg = bt.TrainRunConfig(seed=42, max_workers=8, micro_batch=4, dataset_size=1024, lr=0.02, momentum=0.9,
                        dropout_rate=0.5, jitter=0.1, bucket_capacity=64,
                        determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_fast": 2})
ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")])
h = hashlib.sha256()
for k in (20, 7, 33, 1, 20):
    ts.pipeline.drop_lists()
    out, _ = engine.run_steps(ts, k)
    h.update(np.ascontiguousarray(out).tobytes())
for _ in range(3):
    h.update(repr(bt.run_minibatch(ts)).encode())
p = np.array(ts.executors[0].model.values.tolist())
print(json.dumps({"losses": h.hexdigest(), "params": hashlib.sha256(p.tobytes()).hexdigest(), "step": ts.global_step}))
"""


def test_host_signal_results_equal_copied_results(tmp_path):
    """bt_mlp_run / bt_mlp_run_sampled in the one-copy layout with pinned host buffers: the compact build's
    epilogue writes the losses and status words into host memory and signals a done word (no device-to-host
    copy, no stream synchronisation).  The losses of launches of 20 / 7 / 33 / 1 mini-batches and
    run_minibatch calls, and the final weights, equal the copy-back path (BT_HOST_SIGNAL=0) bit for bit."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = str(Path(__file__).resolve().parent.parent)
    script = tmp_path / "sig.py"
    script.write_text(_SIGNAL_SCRIPT)
    outs = []
    # host signal on / off; the sampled launches reading their index lists zero-copy from the pinned staging
    # buffer (the device copy queued after the launch, used by the later run_minibatch calls) / copied first
    for sig, zc in (("1", "1"), ("0", "1"), ("1", "0")):
        env = dict(os.environ, BT_HOST_SIGNAL=sig, BT_LISTS_ZC=zc)
        r = subprocess.run([sys.executable, str(script), root], capture_output=True, text=True, env=env, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1] == outs[2]


def test_tampered_replica_raises_corruption_on_the_signalled_path(bt):
    """The compact build (micro-batch 4) with pinned results signals the host on its early exit too: a replica
    mismatch raises CorruptionError (not a launch error), and the sticky status makes the next call fail the
    same way without running."""
    cfg = bt.TrainRunConfig(seed=42, max_workers=8, micro_batch=4, dataset_size=1024,
                            determinism=bt.DeterminismMode.from_label("d1"), device_fanins={"gpu_fast": 2})
    ts = bt.init_training(cfg, [bt.ExecutorSpec("gpu_fast")] * 2)
    bt.run_minibatch(ts)
    ts.executors[1].model.values[0] = math.nextafter(ts.executors[1].model.values[0], math.inf)
    with pytest.raises(bt.CorruptionError):
        bt.run_minibatch(ts)
