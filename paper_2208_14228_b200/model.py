"""The reference MLP (model.py:1-213) with device-resident state.

Shape and flat parameter order are the reference's: w1 (input-major,
[8][16]), b1[16], w2[16], b2 -> 161 binary64 parameters.  Forward/backward
and the SGD update run in the sm_100a library (bt_mlp.cu / bt_reduce.cu) with
the reference's pinned evaluation order and glibc's tanh, so results are
bit-identical to the reference on the same inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native
from .device import (DeviceVector, Flags, i64_to_u64, ptr, require_cuda, stream, to_dev, u64_to_i64)
from .errors import InputError
from .reduction import ReduceVariant, fanin_code

INPUT_DIM = 8
HIDDEN_DIM = 16
W1_OFF = 0
B1_OFF = INPUT_DIM * HIDDEN_DIM
W2_OFF = B1_OFF + HIDDEN_DIM
B2_OFF = W2_OFF + HIDDEN_DIM
PARAM_COUNT = B2_OFF + 1  # 161
RANK_EPSILON = 2.0**-40
STAT_DECAY = 0.9

Batch = list[tuple[tuple[float, ...], float]]


def _as_param_tensor(values) -> torch.Tensor:
    if isinstance(values, DeviceVector):
        return values.t
    if isinstance(values, torch.Tensor):
        if values.is_cuda and values.dtype == torch.float64 and values.is_contiguous():
            return values  # already a device vector (on whichever GPU holds it): a view, not a copy
        t = values.to(device=require_cuda(), dtype=torch.float64)
        return t if t.is_contiguous() else t.contiguous()
    return to_dev(list(values))


class ToyModel:
    """Flat parameter vector held in HBM; `.values` is a list-like view."""

    __slots__ = ("_t",)

    def __init__(self, values):
        t = _as_param_tensor(values)
        if t.numel() != PARAM_COUNT:
            raise InputError(f"expected {PARAM_COUNT} parameters, got {t.numel()}")
        self._t = t

    @property
    def values(self) -> DeviceVector:
        return DeviceVector(self._t)

    @values.setter
    def values(self, vals) -> None:
        self._t.copy_(_as_param_tensor(vals))

    @property
    def tensor(self) -> torch.Tensor:
        return self._t

    @classmethod
    def zeros(cls) -> "ToyModel":
        require_cuda()
        return cls(torch.zeros(PARAM_COUNT, dtype=torch.float64, device="cuda"))

    @classmethod
    def init_random(cls, seed: int, scale: float = 0.5) -> "ToyModel":
        """(u*2-1)*scale per parameter from derive_stream(TAG_MODEL_INIT, seed)  (model.py:58-66)."""
        require_cuda()
        t = torch.empty(PARAM_COUNT, dtype=torch.float64, device="cuda")
        _native.check(_native.lib().bt_init_random(seed & (2**64 - 1), float(scale), PARAM_COUNT, ptr(t), stream()))
        return cls(t)

    def copy(self) -> "ToyModel":
        return ToyModel(self._t.clone())

    def __eq__(self, other) -> bool:
        return isinstance(other, ToyModel) and self.values == other.values

    def __repr__(self) -> str:
        return f"ToyModel({self.values.tolist()!r})"


class OptState:
    """Momentum-SGD state: lr, momentum and a device velocity vector."""

    __slots__ = ("lr", "momentum", "_t")

    def __init__(self, lr: float, momentum: float, velocity):
        self.lr = lr
        self.momentum = momentum
        t = _as_param_tensor(velocity)
        if t.numel() != PARAM_COUNT:
            raise InputError(f"expected {PARAM_COUNT} velocity slots, got {t.numel()}")
        self._t = t

    @property
    def velocity(self) -> DeviceVector:
        return DeviceVector(self._t)

    @velocity.setter
    def velocity(self, vals) -> None:
        self._t.copy_(_as_param_tensor(vals))

    @property
    def tensor(self) -> torch.Tensor:
        return self._t

    @classmethod
    def fresh(cls, lr: float, momentum: float) -> "OptState":
        require_cuda()
        return cls(lr, momentum, torch.zeros(PARAM_COUNT, dtype=torch.float64, device="cuda"))

    def copy(self) -> "OptState":
        return OptState(self.lr, self.momentum, self._t.clone())

    def __eq__(self, other) -> bool:
        return (isinstance(other, OptState) and (self.lr, self.momentum) == (other.lr, other.momentum)
                and self.velocity == other.velocity)


@dataclass(frozen=True)
class TrackedStat:
    """Running mean that mixes in the worker rank (model.py:88-104).

    Inside the step the update runs on the device (bt_mlp.cu stage D); this
    value type is what the API hands out and checkpoints carry."""

    running_mean: float = 0.0
    update_count: int = 0

    def updated(self, batch_mean: float, virtual_rank: int) -> "TrackedStat":
        mixed = batch_mean + virtual_rank * RANK_EPSILON
        return TrackedStat(self.running_mean * STAT_DECAY + 0.1 * mixed, self.update_count + 1)


def rows_tensor(batch: Batch, expect_width: int = INPUT_DIM) -> torch.Tensor:
    """Host rows [(x tuple, y)] -> device [n][9] (x then y, the dataset row layout)."""
    flat = []
    for x, y in batch:
        if len(x) != expect_width:
            raise InputError(f"expected input width {expect_width}, got {len(x)}")
        flat.extend(x)
        flat.append(y)
    return to_dev(flat).view(len(batch), INPUT_DIM + 1)


def forward_backward(model: ToyModel, batch: Batch, virtual_rank: int, dropout_rng: int, stat: TrackedStat,
                     variant: ReduceVariant, dropout_rate: float = 0.5):
    """One forward/backward pass on the device (model.py:107-196).

    Returns ``(loss, grads, dropout_rng', stat')`` with grads as a Python list,
    like the reference.  Pure: the model is not modified.
    """
    nrows = len(batch)
    if nrows == 0:
        raise InputError("empty micro-batch")
    if nrows > 256:
        raise InputError("micro-batch larger than 256 rows is not supported by the device kernel")
    rows = rows_tensor(batch)
    params = model.tensor if isinstance(model, ToyModel) else _as_param_tensor(model)
    fan = torch.tensor([fanin_code(variant)], dtype=torch.int32, device="cuda")
    rng = torch.tensor([u64_to_i64(dropout_rng)], dtype=torch.int64, device="cuda")
    mean = torch.tensor([stat.running_mean], dtype=torch.float64, device="cuda")
    cnt = torch.tensor([stat.update_count], dtype=torch.int64, device="cuda")
    loss = torch.empty(1, dtype=torch.float64, device="cuda")
    grads = torch.empty(PARAM_COUNT, dtype=torch.float64, device="cuda")
    flags = Flags()
    _native.check(_native.lib().bt_fwd_bwd_mlp_f64(
        ptr(params), ptr(rows), 1, 0, 1, nrows, ptr(fan), float(dropout_rate), int(virtual_rank), ptr(rng),
        ptr(mean), ptr(cnt), ptr(loss), ptr(grads), ptr(flags.t), stream()), "forward_backward")
    flags.raise_if_set("forward_backward")
    return (float(loss.item()), grads.tolist(), i64_to_u64(int(rng.item())),
            TrackedStat(float(mean.item()), int(cnt.item())))


def sgd_step(model: ToyModel, opt: OptState, grads) -> tuple[ToyModel, OptState]:
    """v <- mu*v + g; p <- p - lr*v on the device (model.py:199-213).

    Out of place: on a non-finite gradient NumericError is raised and the
    inputs are untouched (the reference raises before returning new objects)."""
    g = grads.t if isinstance(grads, DeviceVector) else _as_param_tensor(grads)
    if g.numel() != PARAM_COUNT:
        raise InputError(f"expected {PARAM_COUNT} gradients, got {g.numel()}")
    po = torch.empty(PARAM_COUNT, dtype=torch.float64, device="cuda")
    vo = torch.empty(PARAM_COUNT, dtype=torch.float64, device="cuda")
    flags = Flags()
    _native.check(_native.lib().bt_sgd_step_f64(ptr(model.tensor), ptr(opt.tensor), ptr(g), PARAM_COUNT,
                                                float(opt.lr), float(opt.momentum), ptr(po), ptr(vo),
                                                ptr(flags.t), stream()), "sgd_step")
    st, detail, _ = flags.status()
    if st == 5:
        from .errors import NumericError

        raise NumericError(f"non-finite gradient at parameter {detail}: {g[detail].item()!r}")
    if st:
        flags.raise_if_set("sgd_step")
    return ToyModel(po), OptState(opt.lr, opt.momentum, vo)


__all__ = ["INPUT_DIM", "HIDDEN_DIM", "W1_OFF", "B1_OFF", "W2_OFF", "B2_OFF", "PARAM_COUNT", "RANK_EPSILON",
           "STAT_DECAY", "Batch", "ToyModel", "OptState", "TrackedStat", "forward_backward", "sgd_step"]
