"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container only (it needs /root/reference; the GPU box does
not have it):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/gen_golden.py

Every value below is produced by calling the reference package
(`/root/reference/pkg/src/bittrain`) through its public API; nothing here
re-implements the algorithm.  Floats are stored as little-endian binary64 hex
(the reference's own `runlog.float_to_hex` convention, runlog.py:21-23) so the
fixtures are bit-exact.  The oracle (oracle/) and the CUDA path are pinned
against these files by tests/test_golden_oracle.py and tests/test_gpu_*.py.

libm note: `forward_backward` calls `math.tanh` (model.py:148), i.e. glibc
tanh -> expm1 (the FMA ifunc variant on x86-64 with FMA; glibc 2.39 here).
Loss/param fixtures are therefore pinned to that libm.  The CUDA tanh
(paper_2208_14228_b200/csrc/bt_libm.cuh) restates exactly that variant.
"""

from __future__ import annotations

import json
import os
import random
import struct
import sys
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.dont_write_bytecode = True

import bittrain  # noqa: E402
from bittrain import buckets, checkpoint, engine, model, prng, reduction, sampling, scenarios  # noqa: E402
from bittrain.runlog import float_to_hex, param_fingerprint  # noqa: E402

OUT = Path(__file__).resolve().parent
MASK64 = prng.MASK64


def fh(v: float) -> str:
    return float_to_hex(v)


def fhl(vals) -> list[str]:
    return [fh(v) for v in vals]


def rows_bytes(rows) -> bytes:
    out = bytearray()
    for x, y in rows:
        out += struct.pack(f"<{len(x)}d", *x)
        out += struct.pack("<d", y)
    return bytes(out)


def dump(name: str, doc) -> None:
    path = OUT / name
    with open(path, "w", encoding="utf-8") as fh_:
        json.dump(doc, fh_, indent=None, separators=(",", ":"), sort_keys=True)
        fh_.write("\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


# --------------------------------------------------------------------------
# prng.py (prng.py:27-93)
# --------------------------------------------------------------------------
def gen_prng():
    doc = {}
    streams = {}
    for seed in (0, 1, 42, 0xDEADBEEF, MASK64):
        s = seed
        outs = []
        for _ in range(50):
            s, v = prng.splitmix64_next(s)
            outs.append(format(v, "016x"))
        streams[format(seed, "016x")] = outs
    doc["splitmix64"] = streams
    s = 42
    uni = []
    for _ in range(20):
        s, u = prng.rng_uniform01(s)
        uni.append(fh(u))
    doc["uniform01_seed42"] = uni
    doc["derive_stream"] = [
        {"words": [format(w & MASK64, "016x") for w in words],
         "state": format(prng.derive_stream(*words), "016x")}
        for words in (
            (1, 2, 3), (1, 2, 4), (3, 2, 1), (prng.TAG_MODEL_INIT, 42), (prng.TAG_DATASET, 42),
            (prng.TAG_DROPOUT, 42, 0), (prng.TAG_DROPOUT, 42, 7), (prng.TAG_DATA_WORKER, 42, 0, 0, 0),
            (prng.TAG_DATA_WORKER, 42, 3, 31, 7), (prng.TAG_BUCKET_ARRIVAL, 4, 12, 1), (),
        )
    ]
    doc["dropout_stream_seed42"] = [
        format(prng.derive_stream(prng.TAG_DROPOUT, 42, r), "016x") for r in range(64)
    ]
    doc["worker_rng_seed42"] = [
        {"epoch": e, "local": l, "worker": w,
         "state": format(sampling.worker_rng(42, e, l, w), "016x")}
        for e in (0, 1, 5) for l in (0, 1, 31, 63) for w in (0, 3, 7)
    ]
    doc["fnv1a64"] = [
        {"hex": data.hex(), "hash": format(prng.fnv1a64(data), "016x")}
        for data in (b"", b"a", b"foobar", b"gpu_fast", b"gpu_mid", bytes(range(256)))
    ]
    doc["shuffled_range"] = [
        {"n": n, "state": format(st, "016x"), "perm": prng.shuffled_range(n, st)}
        for n, st in ((0, 99), (1, 99), (2, 7), (16, 42), (33, 7), (5, MASK64), (1024, 42), (1024, 43),
                      (1000, 11))
    ]
    doc["layout_arrival_perm"] = [
        {"n": n, "layout": [[k, t] for k, t in lay], "perm": buckets.layout_arrival_perm(n, lay)}
        for n, lay in (
            (161, [("gpu_a", 1)] * 4), (161, [("gpu_a", 2)] * 2), (161, [("gpu_fast", 4)]),
            (161, [("gpu_fast", 2), ("gpu_mid", 2)]), (16, [("x", 4)]),
        )
    ]
    dump("prng.json", doc)


# --------------------------------------------------------------------------
# reduction.py (reduction.py:20-84)
# --------------------------------------------------------------------------
def adversarial(n, seed):
    rng = random.Random(seed)
    return [rng.uniform(-1, 1) * 10 ** rng.randint(-12, 12) for _ in range(n)]


def gen_reduction():
    cases = []
    for n in (0, 1, 2, 3, 4, 5, 7, 8, 9, 16, 17, 31, 33, 64, 100):
        vals = adversarial(n, 1000 + n)
        if n == 1:
            vals = [-0.0]
        out = {"values": fhl(vals)}
        out["seq"] = fh(reduction.reduce_sum(vals, reduction.Sequential()))
        for f in (2, 3, 4, 5, 8, 16):
            out[f"tree{f}"] = fh(reduction.reduce_sum(vals, reduction.Tree(f)))
        cases.append(out)
    dump("reduction.json", {"cases": cases})


# --------------------------------------------------------------------------
# model.py forward_backward / sgd_step (model.py:107-213)
# --------------------------------------------------------------------------
def variant_of(tag: str):
    return reduction.Sequential() if tag == "seq" else reduction.Tree(int(tag[4:]))


def gen_model():
    fb = []
    rng = random.Random(2208)
    for case in range(40):
        rows = [1, 2, 3, 4, 5, 8, 16, 32][case % 8]
        tag = ["seq", "tree2", "tree3", "tree4"][case % 4]
        rate = [0.5, 0.0, 0.3, 0.5, 1.0, 0.75][case % 6]
        m = model.ToyModel([rng.uniform(-0.5, 0.5) for _ in range(model.PARAM_COUNT)])
        batch = [(tuple(rng.uniform(-1, 1) for _ in range(model.INPUT_DIM)), rng.uniform(-1, 1))
                 for _ in range(rows)]
        if case % 10 == 7:  # adversarial targets make batch reduction order observable
            batch = [(x, (-1.0) ** r * 10.0 ** (r + 2)) for r, (x, _) in enumerate(batch)]
        rank = case % 9
        dropout_rng = rng.getrandbits(64)
        stat = model.TrackedStat(rng.uniform(-1, 1), rng.randint(0, 50))
        loss, grads, rng2, stat2 = model.forward_backward(
            m, batch, rank, dropout_rng, stat, variant_of(tag), rate)
        fb.append({
            "params": fhl(m.values), "x": [fhl(x) for x, _ in batch], "y": fhl([y for _, y in batch]),
            "rank": rank, "rng": format(dropout_rng, "016x"), "stat_mean": fh(stat.running_mean),
            "stat_count": stat.update_count, "variant": tag, "rate": fh(rate),
            "out_loss": fh(loss), "out_grads": fhl(grads), "out_rng": format(rng2, "016x"),
            "out_stat_mean": fh(stat2.running_mean), "out_stat_count": stat2.update_count,
        })
    sgd = []
    for case in range(6):
        m = model.ToyModel([rng.uniform(-0.5, 0.5) for _ in range(model.PARAM_COUNT)])
        lr, mu = [(0.02, 0.9), (0.1, 0.0), (0.0, 0.9), (1.0, 0.5), (0.3, 0.99), (1e-3, 0.9)][case]
        vel = [rng.uniform(-1, 1) * 10 ** rng.randint(-6, 3) for _ in range(model.PARAM_COUNT)]
        g = adversarial(model.PARAM_COUNT, 77 + case)
        opt = model.OptState(lr, mu, vel)
        m2, o2 = model.sgd_step(m, opt, g)
        sgd.append({"params": fhl(m.values), "vel": fhl(vel), "lr": fh(lr), "mu": fh(mu),
                    "grads": fhl(g), "out_params": fhl(m2.values), "out_vel": fhl(o2.velocity)})
    init = {str(seed): fhl(model.ToyModel.init_random(seed).values) for seed in (42, 11, 77, 0)}
    dump("model.json", {"forward_backward": fb, "sgd_step": sgd, "init_random": init})


# --------------------------------------------------------------------------
# buckets.py allreduce (buckets.py:31-124)
# --------------------------------------------------------------------------
def gen_allreduce():
    cases = []
    for i, (nparams, nrep, cap, tag, shuffled) in enumerate((
        (16, 4, 16, "tree2", False), (16, 4, 3, "tree2", False), (16, 4, 5, "tree2", True),
        (16, 4, 5, "seq", True), (23, 5, 7, "seq", False), (23, 5, 7, "tree3", False),
        (161, 8, 64, "tree2", False), (161, 8, 64, "tree3", True), (161, 8, 64, "seq", False),
        (161, 1, 64, "tree2", False), (161, 3, 64, "tree2", False), (161, 16, 64, "tree2", False),
        (161, 6, 10, "tree4", True), (100, 64, 64, "tree2", False), (100, 13, 9, "tree5", True),
        (40, 2, 1, "tree2", False),
    )):
        reps = [adversarial(nparams, 500 + 31 * i + r) for r in range(nrep)]
        if shuffled:
            perm = buckets.layout_arrival_perm(nparams, [("gpu_a", nrep)])
            bm = buckets.rebuild_buckets_first_minibatch(perm, cap)
        else:
            bm = buckets.build_buckets_initial(nparams, cap)
        out = buckets.allreduce(reps, bm, variant_of(tag))
        cases.append({"replicas": [fhl(r) for r in reps], "capacity": cap,
                      "buckets": [list(b) for b in bm.buckets], "variant": tag, "out": fhl(out)})
    dump("allreduce.json", {"cases": cases})


# --------------------------------------------------------------------------
# sampling.py (sampling.py:24-207)
# --------------------------------------------------------------------------
def gen_sampling():
    doc = {}
    ds = sampling.make_dataset(42, 1024, 8)
    doc["dataset_42_1024"] = {"fnv": format(prng.fnv1a64(rows_bytes(ds)), "016x"),
                              "head": [fhl(list(x) + [y]) for x, y in ds[:4]],
                              "tail": [fhl(list(x) + [y]) for x, y in ds[-2:]]}
    ds64 = sampling.make_dataset(42, 64, 8)
    doc["dataset_42_64"] = [fhl(list(x) + [y]) for x, y in ds64]
    ep = []
    for (seed, n, nw, mb, epoch, shuffle) in ((42, 1024, 4, 4, 0, True), (42, 1024, 4, 4, 1, True),
                                              (42, 1024, 8, 4, 0, True), (42, 1024, 8, 4, 3, True),
                                              (42, 50, 4, 3, 3, True), (1, 16, 4, 1, 0, False),
                                              (11, 64, 4, 4, 2, True)):
        plan = sampling.SamplePlan(seed, epoch, n, nw, mb, shuffle)
        ep.append({"seed": seed, "n": n, "workers": nw, "micro": mb, "epoch": epoch,
                   "shuffle": shuffle, "lists": sampling.epoch_indices(plan)})
    doc["epoch_indices"] = ep
    # Pipeline batches (jitter applied) for the C1/C2 configs, first 3 steps and an epoch boundary.
    batches = []
    for nw in (4, 8):
        pipe = sampling.DataPipeline(42, 1024, nw, 4, jitter=0.1, worker_slots=2, prefetch_depth=2)
        spe = pipe.steps_per_epoch
        for step in range(spe + 2):
            for est in range(nw):
                rows = pipe.batch(est, step)
                if step < 3 or step >= spe - 1:
                    batches.append({"workers": nw, "step": step, "est": est,
                                    "rows": [fhl(list(x) + [y]) for x, y in rows]})
    doc["pipeline_batches"] = batches
    dump("sampling.json", doc)


# --------------------------------------------------------------------------
# Full runs through engine/scenarios (engine.py:202-336, scenarios.py:52-83)
# --------------------------------------------------------------------------
FANINS = {"gpu_fast": 2, "gpu_mid": 3}


def cfg(mode="d1", max_workers=4, **over):
    base = dict(seed=42, max_workers=max_workers, micro_batch=4, dataset_size=1024, lr=0.02,
                momentum=0.9, dropout_rate=0.5, jitter=0.1, bucket_capacity=64,
                determinism=engine.DeterminismMode.from_label(mode), device_fanins=FANINS)
    base.update(over)
    return engine.TrainRunConfig(**base)


def spec(kinds, restarts=()):
    return scenarios.RunSpec(tuple(engine.ExecutorSpec(k) for k in kinds),
                             tuple(scenarios.RestartEvent(s, tuple(engine.ExecutorSpec(k) for k in ks))
                                   for s, ks in restarts))


def run_doc(name, c, sp, steps, layout_desc):
    log, ts = scenarios.run_training(c, sp, steps)
    ex = ts.executors[0]
    return {
        "name": name,
        "config": {"seed": c.seed, "max_workers": c.max_workers, "micro_batch": c.micro_batch,
                   "dataset_size": c.dataset_size, "lr": fh(c.lr), "momentum": fh(c.momentum),
                   "dropout_rate": fh(c.dropout_rate), "jitter": fh(c.jitter),
                   "bucket_capacity": c.bucket_capacity, "determinism": c.determinism.label,
                   "devices": FANINS},
        "layout": layout_desc, "steps": steps,
        "losses": [r.losses and fhl(r.losses) for r in log.records],
        "param_hash": [r.param_hash for r in log.records],
        "final_params": fhl(ex.model.values), "final_velocity": fhl(ex.opt.velocity),
        "final_stats": [[fh(cx.stat.running_mean), cx.stat.update_count] for cx in ts.contexts],
        "final_dropout_rng": [format(cx.dropout_rng, "016x") for cx in ts.contexts],
        "final_ckpt_fnv": format(prng.fnv1a64(checkpoint.checkpoint_save(ts)), "016x"),
    }


def gen_runs():
    runs = []
    # C1: 4 ESTs on one executor, d1, 200 steps (fixtures/train_d1.yaml without its restart).
    runs.append(run_doc("c1_d1", cfg("d1", 4), spec(["gpu_fast"]), 200,
                        {"initial": ["gpu_fast"], "restarts": []}))
    # C2: 8 ESTs on 1/2/4/8 executors, 100 steps, d1 and d1d2; hashes must agree across layouts.
    for mode in ("d1", "d1d2"):
        docs = []
        for g in (1, 2, 4, 8):
            docs.append(run_doc(f"c2_{mode}_g{g}", cfg(mode, 8), spec(["gpu_fast"] * g), 100,
                                {"initial": ["gpu_fast"] * g, "restarts": []}))
        assert all(d["param_hash"] == docs[0]["param_hash"] for d in docs)
        assert all(d["losses"] == docs[0]["losses"] for d in docs)
        runs.append(docs[0] | {"name": f"c2_{mode}", "layouts_checked": [1, 2, 4, 8]})
    # fixtures/train_d1.yaml: 2 executors, restart onto 3 after step 100.
    runs.append(run_doc("train_d1_yaml", cfg("d1", 4), spec(["gpu_fast"] * 2, [(100, ["gpu_fast"] * 3)]),
                        200, {"initial": ["gpu_fast"] * 2, "restarts": [[100, ["gpu_fast"] * 3]]}))
    # Mixed device kinds (per-EST batch variants differ; allreduce uses executor 0's variant).
    runs.append(run_doc("mixed_d1", cfg("d1", 4), spec(["gpu_mid", "gpu_fast"]), 40,
                        {"initial": ["gpu_mid", "gpu_fast"], "restarts": []}))
    runs.append(run_doc("mixed_d1d2", cfg("d1d2", 4), spec(["gpu_mid", "gpu_fast"], [(20, ["gpu_fast"])]), 40,
                        {"initial": ["gpu_mid", "gpu_fast"], "restarts": [[20, ["gpu_fast"]]]}))
    # d0: bucket map rebuilt from the layout-keyed arrival order after the first post-boot step.
    runs.append(run_doc("d0_restart", cfg("d0", 4), spec(["gpu_fast"] * 4, [(10, ["gpu_fast"] * 2)]), 30,
                        {"initial": ["gpu_fast"] * 4, "restarts": [[10, ["gpu_fast"] * 2]]}))
    runs.append(run_doc("d0_plain", cfg("d0", 4), spec(["gpu_fast"] * 4), 30,
                        {"initial": ["gpu_fast"] * 4, "restarts": []}))
    # Small engine-test config (micro 2, 64 rows: epoch rollover every 8 steps), 16 ESTs.
    runs.append(run_doc("small_e16", cfg("d1", 16, micro_batch=2, dataset_size=64), spec(["gpu_fast"] * 3), 12,
                        {"initial": ["gpu_fast"] * 3, "restarts": []}))
    dump("runs.json", {"runs": runs})


def gen_checkpoint():
    blobs = []
    for mode, steps, nw, layout in (("d1", 5, 4, 2), ("d0", 3, 4, 2), ("d1d2", 0, 4, 2), ("d1", 2, 8, 3)):
        c = cfg(mode, nw, micro_batch=2, dataset_size=64)
        ts = engine.init_training(c, [engine.ExecutorSpec("gpu_fast")] * layout)
        for _ in range(steps):
            engine.run_minibatch(ts)
        blob = checkpoint.checkpoint_save(ts)
        blobs.append({"mode": mode, "steps": steps, "workers": nw, "executors": layout,
                      "config": {"micro_batch": 2, "dataset_size": 64}, "blob": blob.hex()})
    dump("checkpoint.json", {"blobs": blobs})


def gen_global_batch():
    """run_minibatch(ts, global_batch) with explicit rows (engine.py:261-282)."""
    out = []
    c = cfg("d1", 4, micro_batch=2, dataset_size=64)
    ts = engine.init_training(c, [engine.ExecutorSpec("gpu_fast")] * 2)
    rng = random.Random(3)
    for step in range(4):
        rows = [(tuple(rng.uniform(-1, 1) for _ in range(8)), rng.uniform(-1, 1)) for _ in range(8)]
        losses = engine.run_minibatch(ts, rows)
        out.append({"rows": [fhl(list(x) + [y]) for x, y in rows], "losses": fhl(losses),
                    "params": fhl(ts.executors[0].model.values)})
    dump("global_batch.json", {"steps": out, "config": {"seed": 42, "max_workers": 4, "micro_batch": 2,
                                                        "dataset_size": 64, "executors": 2}})


def gen_ladder():
    """The S1-S5 reproducibility ladder (scenarios.py:118-169) as the reference's
    own scenario tests configure it (test_scenarios.py:16-29): per mode, each
    level's two runs (per-step losses + param hashes) and the bitdiff verdict;
    plus the staged kind-change run and seeded random restart schedules."""
    from bittrain.runlog import bitdiff

    kinds = {"gpu_a": 2, "gpu_b": 3}
    steps = 16

    def cfg_for(mode):
        return engine.TrainRunConfig(seed=11, max_workers=4, micro_batch=4, dataset_size=64,
                                     determinism=engine.DeterminismMode.from_label(mode), device_fanins=kinds)

    def spec_doc(sp):
        return {"layout": [e.device_kind for e in sp.layout],
                "restarts": [[r.after_step, [e.device_kind for e in r.layout]] for r in sp.restarts]}

    def run_pair(c, sp_a, sp_b):
        la, ta = scenarios.run_training(c, sp_a, steps)
        lb, tb = scenarios.run_training(c, sp_b, steps)
        d = bitdiff(la, lb)
        return {"run_a": spec_doc(sp_a), "run_b": spec_doc(sp_b),
                "hash_a": [r.param_hash for r in la.records], "hash_b": [r.param_hash for r in lb.records],
                "losses_b": [fhl(r.losses) for r in lb.records],
                "final_equal": ta.executors[0].model.values == tb.executors[0].model.values,
                "divergence": None if d is None else {"step": d.step, "field": d.field, "worker": d.worker}}

    c0 = cfg_for("d1")
    doc = {"steps": steps, "kinds": kinds,
           "config": {"seed": 11, "max_workers": 4, "micro_batch": 4, "dataset_size": 64, "lr": fh(c0.lr),
                      "momentum": fh(c0.momentum), "dropout_rate": fh(c0.dropout_rate), "jitter": fh(c0.jitter),
                      "bucket_capacity": c0.bucket_capacity},
           "matrix": {}}
    for mode in ("d0", "d1", "d1d2"):
        c = cfg_for(mode)
        levels = []
        for sc in scenarios.default_matrix("gpu_a", "gpu_b", steps):
            levels.append({"level": sc.level, **run_pair(c, sc.run_a, sc.run_b)})
        rep = scenarios.run_matrix(c, scenarios.default_matrix("gpu_a", "gpu_b", steps), steps)
        assert [r.bitwise_equal for r in rep.results] == [lv["divergence"] is None and lv["final_equal"]
                                                          for lv in levels]
        doc["matrix"][mode] = {"levels": levels, "guaranteed": sorted(scenarios.guaranteed_levels(mode)),
                               "failed_guarantees": rep.failed_guarantees()}
    # test_scenarios.py:89-112: homogeneous shrink then a kind change
    ref4 = spec(["gpu_a"] * 4)
    staged = spec(["gpu_a"] * 4, [(6, ["gpu_a"] * 2), (11, ["gpu_a", "gpu_b"])])
    doc["staged"] = {m: run_pair(cfg_for(m), ref4, staged) for m in ("d1", "d1d2")}
    # test_scenarios.py:131-159: seeded random layouts and restart schedules
    rng = random.Random(2718)
    rand = []
    for mode, ks in (("d1", ["gpu_a"]), ("d1d2", ["gpu_a", "gpu_b"])):
        for _ in range(3):
            lay = [rng.choice(ks) for _ in range(rng.randint(1, 4))]
            rs = [(s, [rng.choice(ks) for _ in range(rng.randint(1, 4))])
                  for s in sorted(rng.sample(range(2, steps - 1), rng.randint(0, 2)))]
            rand.append({"mode": mode, **run_pair(cfg_for(mode), spec([ks[0]] * 4), spec(lay, rs))})
    doc["random"] = rand
    dump("ladder.json", doc)


def gen_cli():
    """The reference's own command line (cli.py:38-78): run logs (JSON lines), checkpoint bytes, and
    the reprocheck / bitdiff reports, byte for byte, for small configs and the train_d1 fixture."""
    import contextlib
    import io
    import tempfile

    import yaml
    from bittrain import cli

    def small(**over):
        doc = {"seed": 7, "max_workers": 4, "micro_batch": 4, "dataset_size": 128, "minibatches": 12,
               "determinism": "d1", "devices": {"gpu_fast": 2, "gpu_mid": 3},
               "layout": [{"device": "gpu_fast"}, {"device": "gpu_fast"}]}
        doc.update(over)
        return doc

    fixture = yaml.safe_load(open("/root/reference/pkg/fixtures/train_d1.yaml", encoding="utf-8"))
    out = {"train": [], "reprocheck": []}
    with tempfile.TemporaryDirectory() as td:
        def run(argv):
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                rc = cli.main(argv)
            return rc, buf.getvalue()

        cases = [("small_fast2", small()), ("small_mid2", small(layout=[{"device": "gpu_mid"}] * 2)),
                 ("small_fast1", small(layout=[{"device": "gpu_fast"}])),
                 ("small_e2", small(max_workers=2, layout=[{"device": "gpu_fast"}])),
                 ("small_dump", small(dump_params_every=4, minibatches=8)),
                 ("train_d1_fixture", fixture)]
        for name, doc in cases:
            cfg_path, log_path, ck_path = f"{td}/{name}.yaml", f"{td}/{name}.log", f"{td}/{name}.ckpt"
            with open(cfg_path, "w", encoding="utf-8") as fh:
                yaml.safe_dump(doc, fh)
            rc, text = run(["train", "--config", cfg_path, "--out", log_path, "--ckpt", ck_path])
            out["train"].append({"name": name, "doc": doc, "rc": rc, "stdout": text,
                                 "log": open(log_path, encoding="utf-8").read(),
                                 "ckpt": open(ck_path, "rb").read().hex()})
        logs = {c["name"]: f"{td}/{c['name']}.log" for c in out["train"]}
        out["bitdiff"] = []
        for a, b in (("small_fast2", "small_fast1"), ("small_fast2", "small_mid2"), ("small_fast2", "small_e2")):
            rc, text = run(["bitdiff", logs[a], logs[b]])
            out["bitdiff"].append({"a": a, "b": b, "rc": rc, "stdout": text})
        matrix = {"steps": 12,
                  "config": {"seed": 3, "max_workers": 4, "micro_batch": 4, "dataset_size": 128,
                             "devices": {"gpu_fast": 2, "gpu_mid": 3}},
                  "scenarios": [{"level": "S1", "run_a": {"layout": [{"device": "gpu_fast"}]},
                                 "run_b": {"layout": [{"device": "gpu_fast"}]}},
                                {"level": "S3", "run_a": {"layout": [{"device": "gpu_fast"}]},
                                 "run_b": {"layout": [{"device": "gpu_mid"}]}},
                                {"level": "S4", "run_a": {"layout": [{"device": "gpu_fast"}] * 4},
                                 "run_b": {"layout": [{"device": "gpu_fast"}] * 2,
                                           "restarts": [{"after_step": 6, "layout": [{"device": "gpu_fast"}] * 3}]}}]}
        mpath = f"{td}/matrix.yaml"
        with open(mpath, "w", encoding="utf-8") as fh:
            yaml.safe_dump(matrix, fh)
        for mode in ("d0", "d1", "d1d2"):
            rc, text = run(["reprocheck", "--mode", mode, "--matrix", mpath])
            out["reprocheck"].append({"mode": mode, "matrix": matrix, "rc": rc, "stdout": text})
    dump("cli.json", out)


if __name__ == "__main__":
    assert os.path.isdir(REF_SRC), "needs the read-only reference at /root/reference"
    if sys.argv[1:] == ["ladder"]:
        gen_ladder()
        sys.exit(0)
    if sys.argv[1:] == ["cli"]:
        gen_cli()
        sys.exit(0)
    gen_prng()
    gen_reduction()
    gen_model()
    gen_allreduce()
    gen_sampling()
    gen_runs()
    gen_checkpoint()
    gen_global_batch()
    gen_ladder()
    gen_cli()
