"""Training/matrix YAML parsing for the hot path (reference configio.py:180-251).

Only the train and matrix documents are in scope; the planner's pool,
profile, trace and metrics I/O serve the out-of-scope simulator.
"""

from __future__ import annotations

import yaml

from .engine import DeterminismMode, ExecutorSpec, TrainRunConfig
from .errors import ConfigError
from .scenarios import ReproScenario, RestartEvent, RunSpec


def _load_yaml(path):
    try:
        with open(path, encoding="utf-8") as fh:
            doc = yaml.safe_load(fh)
    except OSError as exc:
        raise ConfigError(f"cannot read {path}: {exc}") from exc
    except yaml.YAMLError as exc:
        raise ConfigError(f"{path}: invalid YAML: {exc}") from exc
    if not isinstance(doc, dict):
        raise ConfigError(f"{path}: expected a mapping at the top level")
    return doc


def _layout(entries) -> tuple:
    if not entries:
        raise ConfigError("layout must list at least one executor")
    out = []
    for e in entries:
        if "device" not in e:
            raise ConfigError("layout entries need a device kind")
        t = e.get("threads")
        out.append(ExecutorSpec(str(e["device"]), None if t is None else int(t)))
    return tuple(out)


def _restarts(entries) -> tuple:
    return tuple(RestartEvent(int(r["after_step"]), _layout(r["layout"])) for r in entries or [])


def parse_train_config(doc: dict):
    """-> (TrainRunConfig, RunSpec, steps, dump_every)."""
    try:
        cfg = TrainRunConfig(
            seed=int(doc["seed"]), max_workers=int(doc["max_workers"]),
            micro_batch=int(doc.get("micro_batch", 4)), dataset_size=int(doc.get("dataset_size", 1000)),
            lr=float(doc.get("lr", 0.02)), momentum=float(doc.get("momentum", 0.9)),
            dropout_rate=float(doc.get("dropout_rate", 0.5)), jitter=float(doc.get("jitter", 0.1)),
            bucket_capacity=int(doc.get("bucket_capacity", 64)), worker_slots=int(doc.get("worker_slots", 2)),
            prefetch_depth=int(doc.get("prefetch_depth", 2)), shuffle=bool(doc.get("shuffle", True)),
            determinism=DeterminismMode.from_label(str(doc.get("determinism", "d1"))),
            device_fanins={str(k): int(v) for k, v in doc["devices"].items()})
    except KeyError as exc:
        raise ConfigError(f"training config missing field {exc}") from exc
    spec = RunSpec(_layout(doc.get("layout")), _restarts(doc.get("restarts")))
    return cfg, spec, int(doc.get("minibatches", 100)), int(doc.get("dump_params_every", 0))


def load_train_config(path):
    return parse_train_config(_load_yaml(path))


def load_matrix(path):
    """-> (base TrainRunConfig, [ReproScenario], steps)."""
    doc = _load_yaml(path)
    base = dict(doc.get("config") or {})
    base.setdefault("layout", [{"device": next(iter(base.get("devices", {"x": 0})))}])
    cfg, _, _, _ = parse_train_config(base)
    scenarios = []
    for s in doc.get("scenarios", []):
        a, b = s["run_a"], s["run_b"]
        scenarios.append(ReproScenario(str(s["level"]), RunSpec(_layout(a["layout"]), _restarts(a.get("restarts"))),
                                       RunSpec(_layout(b["layout"]), _restarts(b.get("restarts")))))
    if not scenarios:
        raise ConfigError(f"{path}: no scenarios")
    return cfg, scenarios, int(doc.get("steps", 100))
