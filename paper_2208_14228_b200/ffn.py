"""Per-EST transformer FFN training step -- the C4 model-stack slice.

A BERT-base FFN sublayer (d_model 768 -> d_ff 3072 -> 768, GELU (tanh form, as BERT), dropout)
trained data-parallel by E virtual workers (ESTs), EasyScale-style:

* every EST's randomness (its synthetic tokens and targets, its dropout masks)
  is keyed by (seed, EST rank, step), never by the launch or the GPU
  (the reference keys dropout the same way, model.py:151-161);
* the dense products run on the deterministic tcgen05 GEMM (csrc/bt_gemm.cu):
  row-independent products (forward, dD) for a whole group of ESTs at once --
  a row's bits do not depend on which rows share the launch -- and one weight
  gradient per EST (batched GEMM over the EST's own tokens);
* the per-EST gradients are summed by the fixed-order reducer (csrc/bt_reduce.cu,
  EST-rank order, fused /E and momentum SGD on fp32 master weights).

So the trained weights are bit-identical however the ESTs are grouped into
launches (`groups=`) -- the same property the multi-GPU mapping needs: a GPU
holding a contiguous EST block runs exactly one such group.

There is no reference implementation of this model: parity is
against a float64 restatement with the same bf16 rounding points
(tests/test_gpu_ffn.py), at a stated tolerance.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native
from .device import Flags, require_cuda, stream
from .errors import ConfigError, NumericError
from .gemm import gemm_bf16, gemm_bf16_at_b

_P = 64  # partial loss sums per EST (bt_ffn_out)


def _init_uniform(seed: int, n: int, scale: float) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_init_random(seed & (2**64 - 1), scale, n, out.data_ptr(), stream()))
    return out.float()


class FFNJob:
    """E ESTs x `tokens` tokens each, one FFN sublayer, momentum SGD on fp32 master weights."""

    def __init__(self, ests: int, tokens: int, d_model: int = 768, d_ff: int = 3072, seed: int = 42,
                 lr: float = 1e-2, momentum: float = 0.9, dropout: float = 0.1, fanin: int = 0, fused: bool = True):
        require_cuda()
        if tokens % 128 or d_model % 128 or d_ff % 128:
            raise ConfigError("tokens, d_model and d_ff must be multiples of 128")
        if ests > _native.BT_MAX_TABLE:
            raise ConfigError(f"at most {_native.BT_MAX_TABLE} ESTs per job")
        if fanin not in (0, 2) or (fanin == 2 and ests & (ests - 1)):
            raise ConfigError("allreduce variant: Sequential (0) or Tree(2) with a power-of-two EST count")
        self.E, self.Te, self.D, self.F = ests, tokens, d_model, d_ff
        self.seed, self.lr, self.mu, self.p, self.fanin = seed, lr, momentum, dropout, fanin
        self.fused = fused  # element ops in the GEMM epilogues (False: standalone kernels, same math)
        D, F = d_model, d_ff
        self.W1 = _init_uniform(seed, F * D, D ** -0.5).view(F, D)
        self.b1 = torch.zeros(F, device="cuda")
        self.W2 = _init_uniform(seed + 1, D * F, F ** -0.5).view(D, F)
        self.b2 = torch.zeros(D, device="cuda")
        self.params = [self.W1, self.b1, self.W2, self.b2]
        self.vel = [torch.zeros_like(t) for t in self.params]
        self.step_idx = 0
        self.flags = Flags()
        self._ws = {}
        self._grads = [torch.empty(ests, t.numel(), dtype=torch.float32, device="cuda") for t in self.params]
        self._refresh_bf16()

    # -- bf16 operand copies of the master weights (W2^T for the dD product)
    def _refresh_bf16(self):
        L, s = _native.lib(), stream()
        if not hasattr(self, "W1h"):
            self.W1h = torch.empty(self.F, self.D, dtype=torch.bfloat16, device="cuda")
            self.W2h = torch.empty(self.D, self.F, dtype=torch.bfloat16, device="cuda")
            self.W2t = torch.empty(self.F, self.D, dtype=torch.bfloat16, device="cuda")
        _native.check(L.bt_cast_f32_bf16(self.W1.data_ptr(), self.W1.numel(), self.W1h.data_ptr(), s))
        _native.check(L.bt_cast_f32_bf16(self.W2.data_ptr(), self.W2.numel(), self.W2h.data_ptr(), s))
        _native.check(L.bt_transpose_to_bf16(self.W2.data_ptr(), 1, 1, self.D, self.F, self.W2t.data_ptr(), s))

    def _workspace(self, n: int) -> dict:
        """Activation / scratch buffers of an n-EST group, allocated once and reused every step."""
        ws = self._ws.get(n)
        if ws is None:
            D, F, Te, T = self.D, self.F, self.Te, n * self.Te
            bf, f32 = dict(dtype=torch.bfloat16, device="cuda"), dict(dtype=torch.float32, device="cuda")
            ws = {"X": torch.empty(T, D, **bf), "tgt": torch.empty(T, D, **f32), "Hpre": torch.empty(T, F, **bf),
                  "D": torch.empty(T, F, **bf), "Y": torch.empty(T, D, **f32), "dY": torch.empty(T, D, **bf),
                  "dH": torch.empty(T, F, **bf), "part": torch.empty(n * _P, **f32),
                  "colsum": torch.empty(n * -(-Te // 64) * F, **f32)}
            if not self.fused:
                ws["H"] = torch.empty(T, F, **f32)
            self._ws[n] = ws
        return ws

    def _group(self, base: int, n: int, grads: list, losses: torch.Tensor, capture: dict | None = None):
        """Forward/backward of ESTs [base, base+n): per-EST gradients into grads[*][base:base+n]."""
        L, s = _native.lib(), stream()
        D, F, Te, T = self.D, self.F, self.Te, n * self.Te
        seed, step, p = self.seed & (2**64 - 1), self.step_idx, self.p
        w = self._workspace(n)
        X, tgt, Hpre, Dact, dY, dH = w["X"], w["tgt"], w["Hpre"], w["D"], w["dY"], w["dH"]
        _native.check(L.bt_ffn_data(seed, step, base, n, Te, D, X.data_ptr(), tgt.data_ptr(), s))
        if self.fused:  # X W1^T with bias + GELU + dropout in the GEMM epilogue
            _native.check(L.bt_gemm_bf16_ffn(X.data_ptr(), self.W1h.data_ptr(), Hpre.data_ptr(), T, F, D, 1,
                                             self.b1.data_ptr(), None, Dact.data_ptr(), seed, step, base, Te, p, 0,
                                             s), "ffn forward GEMM")
        else:
            gemm_bf16(X, self.W1h, out=w["H"])                         # [T][F] = X W1^T
            _native.check(L.bt_ffn_fwd_act(w["H"].data_ptr(), self.b1.data_ptr(), seed, step, base, n, Te, F, p,
                                           Hpre.data_ptr(), Dact.data_ptr(), s))
        gemm_bf16(Dact, self.W2h, out=w["Y"])                          # [T][D] = dropout(gelu) W2^T
        _native.check(L.bt_ffn_out(w["Y"].data_ptr(), self.b2.data_ptr(), tgt.data_ptr(), n, Te, D, dY.data_ptr(),
                                   w["part"].data_ptr(), losses[base:].data_ptr(), s))
        if self.fused:  # dY W2 with dropout' and GELU' in the GEMM epilogue
            _native.check(L.bt_gemm_bf16_ffn(dY.data_ptr(), self.W2t.data_ptr(), dH.data_ptr(), T, F, D, 2, None,
                                             Hpre.data_ptr(), None, seed, step, base, Te, p, 0, s),
                          "ffn backward GEMM")
        else:
            gemm_bf16(dY, self.W2t, out=w["H"])                        # [T][F] = dY W2
            _native.check(L.bt_ffn_bwd_act(w["H"].data_ptr(), Hpre.data_ptr(), seed, step, base, n, Te, F, p,
                                           dH.data_ptr(), s))
        if capture is not None:
            capture.update(X=X.clone(), D=Dact.clone(), dY=dY.clone(), dH=dH.clone())
        gW1, gb1, gW2, gb2 = grads
        # per-EST weight gradients, K = the EST's own tokens, operands read MN-major from the activations
        gemm_bf16_at_b(dH.view(n, Te, F), X.view(n, Te, D), out=gW1[base:base + n])      # dW1_e = dH_e^T X_e
        gemm_bf16_at_b(dY.view(n, Te, D), Dact.view(n, Te, F), out=gW2[base:base + n])   # dW2_e = dY_e^T D_e
        _native.check(L.bt_colsum_bf16(dH.data_ptr(), n, Te, F, gb1[base:].data_ptr(), w["colsum"].data_ptr(), s))
        _native.check(L.bt_colsum_bf16(dY.data_ptr(), n, Te, D, gb2[base:].data_ptr(), w["colsum"].data_ptr(), s))

    def step(self, groups: list[int] | None = None, capture: dict | None = None) -> torch.Tensor:
        """One mini-batch of all E ESTs; `groups` = EST counts per launch group (default: one group).
        Returns the per-EST losses [E] (fp32, on device)."""
        groups = groups or [self.E]
        if sum(groups) != self.E or min(groups) < 1:
            raise ConfigError(f"groups {groups} must partition {self.E} ESTs")
        E = self.E
        grads = self._grads
        losses = torch.empty(E, dtype=torch.float32, device="cuda")
        base = 0
        for n in groups:
            self._group(base, n, grads, losses, capture if len(groups) == 1 else None)
            base += n
        if capture is not None:
            capture["grads"] = [g.clone() for g in grads]
        self._reduce_update(grads)
        self.step_idx += 1
        self._refresh_bf16()
        return losses

    def _reduce_update(self, grads):
        """Fixed EST-rank-order sum, /E, momentum SGD (bt_reduce_update, f32, strided slots)."""
        L, s = _native.lib(), stream()
        for g, prm, vel in zip(grads, self.params, self.vel):
            a = _native.ReduceArgs()
            a.dtype, a.mode, a.E, a.fanin, a.n = _native.DTYPE_F32, _native.REDUCE_UPDATE, self.E, self.fanin, prm.numel()
            for k in range(self.E):  # a pointer table (the 16-byte-vector fast path), EST-rank order
                a.grads[k] = g[k].data_ptr()
            a.param, a.vel, a.param_out, a.vel_out = prm.data_ptr(), vel.data_ptr(), prm.data_ptr(), vel.data_ptr()
            a.lr, a.mu, a.flags = self.lr, self.mu, self.flags.t.data_ptr()
            _native.check(L.bt_reduce_update(C.byref(a), s), "ffn reduce_update")
        st, _, _ = self.flags.status()
        if st:
            self.flags.reset()
            raise NumericError("ffn: non-finite synchronized gradient")

    def flops_per_step(self) -> float:
        """5 GEMMs of 2*T*D*F flops each (forward x2, dD, dW1, dW2; no dX for the first layer)."""
        return 5 * 2.0 * self.E * self.Te * self.D * self.F
