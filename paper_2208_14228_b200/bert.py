"""Per-EST BERT encoder training step -- C4 (BASELINE.json configs[3]).

A post-LN BERT encoder (BERT-base: 12 layers, d_model 768, 12 heads of 64,
FFN 3072, sequence 128, hidden and attention-probability dropout 0.1) trained
data-parallel by E virtual workers (ESTs), EasyScale-style:

* every EST's randomness (its synthetic inputs and targets, every dropout
  mask) is keyed by (seed, EST rank, step, layer, element), never by the
  launch or the GPU -- the reference keys dropout by rank the same way
  (model.py:151-161);
* the dense products run on the deterministic tcgen05 GEMM (csrc/bt_gemm.cu):
  row-independent products (forward, dX) for a whole launch group of ESTs at
  once -- a row's bits do not depend on which rows share the launch -- and one
  weight gradient per EST (batched GEMM over the EST's own tokens, written
  straight into the EST's gradient slot); attention, LayerNorm and the loss
  are csrc/bt_bert.cu, each with a reduction shape fixed by the EST's data;
* the per-EST gradients [E][P] are summed by the fixed-order reducer
  (csrc/bt_reduce.cu: EST-rank order, fused /E and momentum SGD on the fp32
  master weights) -- one launch over all P parameters.

So the trained weights are bit-identical however the ESTs are grouped into
launches (`groups=`), which is what mapping them onto 1/2/4/8 GPUs does: a GPU
holding a contiguous EST block runs exactly one such group.

Input and output layers (head="mlm", the default; csrc/bt_embed.cu): synthetic token ids from
splitmix64 mod the vocabulary (30522), word + position embeddings, and BERT's masked-LM
objective -- `npred` (20) masked positions per 128-token sequence, [MASK] inputs there, a decoder
tied to the word embedding (logits = y_m W_emb^T + b over the vocabulary, tcgen05 GEMMs) and a
softmax cross-entropy; the embedding gradient (tied decoder GEMM + a per-leaf sorted segment sum of
the input-side rows, no atomics) lands in the gradient slot like every other parameter.  (Not
modelled: token-type embeddings, the embedding LayerNorm and the MLM transform layer.)
head="mse": a per-token regression on synthetic embedded inputs (the round-1 head).  There is no
reference implementation of this model: parity is against a float64 restatement of
every stage with the same bf16 rounding points (tests/test_gpu_bert.py).
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _native
from .device import Flags, require_cuda, stream
from .errors import ConfigError, NumericError

_LAYER = ("Wqkv", "bqkv", "Wo", "bo", "g1", "be1", "W1", "b1", "W2", "b2", "g2", "be2")
_MATS = ("Wqkv", "Wo", "W1", "W2")
# b1 gradient partials from the FFN backward GEMM's epilogue (BT_BERT_CS=0: the standalone column-sum pass,
# kept for A/B measurements)
_FUSED_CS = os.environ.get("BT_BERT_CS", "1") != "0"
# attention-dropout keep bits written by the forward, read by the backward (BT_ATTN_BITS=0: the backward
# draws the masks again -- A/B measurements)
_ATTN_BITS = os.environ.get("BT_ATTN_BITS", "1") != "0"


def _init_uniform(seed: int, n: int, scale: float) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_init_random(seed & (2**64 - 1), scale, n, out.data_ptr(), stream()))
    return out.float()


class BertJob:
    """E ESTs x `seqs` sequences of 128 tokens each, `layers` encoder layers, momentum SGD."""

    def __init__(self, ests: int, seqs: int = 8, layers: int = 12, d_model: int = 768, heads: int = 12,
                 d_ff: int = 3072, seed: int = 42, lr: float = 1e-3, momentum: float = 0.9, p_hidden: float = 0.1,
                 p_attn: float = 0.1, fanin: int = 0, eps: float = 1e-12, est_base: int = 0,
                 est_count: int | None = None, est_group: int = 1, optimizer: str = "sgd",
                 adam_beta2: float = 0.999, adam_eps: float = 1e-8, graph: bool = True, head: str = "mlm",
                 vocab: int = 30522, npred: int = 20, mask_id: int = 103):
        """`est_base` / `est_count`: this process computes ESTs [est_base, est_base + est_count) of the E
        (one rank of a multi-GPU job, `attach_peer`); default all E.
        `est_group` (g): gradient leaf group.  g = 1: one gradient buffer per EST, summed by the reducer in
        EST-rank order.  g > 1: the weight/bias/LN gradients of ESTs [g*j, g*j+g) are accumulated in one
        buffer in a canonical order -- the GEMM's ascending K over EST g*j's tokens, then g*j+1's, ... --
        before the rank-ordered reducer runs over the E/g leaves (EasyScale's per-worker gradient
        accumulation with a pinned order).  Bit-identical for every mapping whose GPU blocks are whole
        leaf groups (E=32, g=4: 1/2/4/8 GPUs), with g-fold less gradient traffic.
        `optimizer`: "sgd" (momentum SGD, the reference's update) or "adam" (beta1 = momentum; fused into
        the reducer's final pass as well, bias corrections from the step count).
        `graph`: after one eager step, the whole step (all launch groups, the reducer, the bf16 weight
        refresh, the device step counter) is captured once as a CUDA graph and replayed -- no per-kernel
        host launches; every kernel reads the step from the device counter, so replays are exact.
        `head`: "mlm" (token ids, embeddings, masked-LM cross-entropy over `vocab` with `npred` masked
        positions per sequence) or "mse" (regression on synthetic embedded inputs)."""
        require_cuda()
        if heads * 64 != d_model or d_model % 256 or d_model > 1024 or d_ff % 256:
            raise ConfigError("d_model = 64 * heads, a multiple of 256 (<= 1024); d_ff a multiple of 256")
        if ests > _native.BT_MAX_TABLE or ests < 1:
            raise ConfigError(f"1..{_native.BT_MAX_TABLE} ESTs per job")
        if fanin not in (0, 2):
            raise ConfigError("allreduce variant: Sequential (0) or Tree(2)")
        if seqs < 1 or layers < 1:
            raise ConfigError("seqs and layers must be >= 1")
        self.E, self.S, self.L, self.D, self.H, self.F = ests, seqs, layers, d_model, heads, d_ff
        self.est0, self.En = est_base, ests if est_count is None else est_count
        if self.est0 < 0 or self.En < 1 or self.est0 + self.En > ests:
            raise ConfigError(f"local EST block [{est_base}, +{est_count}) outside the {ests} ESTs")
        self.g = est_group
        if self.g < 1 or ests % self.g or self.En % self.g or self.est0 % self.g:
            raise ConfigError(f"gradient leaf group {est_group} must divide E and the local EST block")
        if fanin == 2 and (ests // self.g) & (ests // self.g - 1):
            raise ConfigError("Tree(2) needs a power-of-two number of gradient leaves")
        if head not in ("mlm", "mse"):
            raise ConfigError(f"head {head!r}: 'mlm' or 'mse'")
        if head == "mlm" and not (2 <= vocab and 1 <= npred <= 32 and 0 <= mask_id < vocab):
            raise ConfigError("mlm head: vocab >= 2, 1 <= npred <= 32, mask_id in the vocabulary")
        self.head, self.V, self.NP, self.mask_id = head, vocab, npred, mask_id
        self.Vp = -(-vocab // 256) * 256  # padded vocabulary (GEMM tiles); the padding rows stay zero
        self.peer = None
        self.Te = seqs * 128
        self.seed, self.lr, self.mu, self.fanin = seed, lr, momentum, fanin
        self.ph, self.pa, self.eps = p_hidden, p_attn, eps
        D, F = d_model, d_ff
        shapes = {"Wqkv": (3 * D, D), "bqkv": (3 * D,), "Wo": (D, D), "bo": (D,), "g1": (D,), "be1": (D,),
                  "W1": (F, D), "b1": (F,), "W2": (D, F), "b2": (D,), "g2": (D,), "be2": (D,)}
        self.shapes = shapes
        self.eoff = {}  # mlm head: Wemb [Vp][D], Pemb [128][D], bdec [Vp] ahead of the layers
        o = 0
        if head == "mlm":
            shapes.update({"Wemb": (self.Vp, D), "Pemb": (128, D), "bdec": (self.Vp,)})
            for k in ("Wemb", "Pemb", "bdec"):
                self.eoff[k] = o
                o += int(torch.Size(shapes[k]).numel())
        self.off = []  # per layer: name -> flat offset (floats; all multiples of 256)
        for _ in range(layers):
            d = {}
            for k in _LAYER:
                d[k] = o
                o += int(torch.Size(shapes[k]).numel())
            self.off.append(d)
        self.P = o
        self.params = torch.zeros(self.P, dtype=torch.float32, device="cuda")
        for l in range(layers):
            for i, k in enumerate(_MATS):
                rows, cols = shapes[k]
                self.view(l, k).copy_(_init_uniform(seed * 1000003 + 16 * l + i, rows * cols, cols ** -0.5)
                                      .view(rows, cols))
            self.view(l, "g1").fill_(1.0)
            self.view(l, "g2").fill_(1.0)
        if head == "mlm":  # the embeddings (uniform, BERT's 0.02 scale); padding rows and the bias zero
            self.eview("Wemb")[:vocab].copy_(_init_uniform(seed * 1000003 + 7919, vocab * D, 0.02).view(vocab, D))
            self.eview("Pemb").copy_(_init_uniform(seed * 1000003 + 7927, 128 * D, 0.02).view(128, D))
        self.vel = torch.zeros_like(self.params)
        if optimizer not in ("sgd", "adam"):
            raise ConfigError(f"optimizer {optimizer!r}: 'sgd' or 'adam'")
        self.adam = (adam_beta2, adam_eps) if optimizer == "adam" else None
        self.vel2 = torch.zeros_like(self.params) if self.adam else None
        self.grads = torch.empty(self.En // self.g, self.P, dtype=torch.float32, device="cuda")  # gradient leaves
        # bf16 image of every parameter at the same offsets (the GEMM operands: W [out][in] as stored --
        # K-major for the forward, MN-major (B stored [K][N]) for the dX products, so no transposed copy)
        self.pb = torch.empty(self.P, dtype=torch.bfloat16, device="cuda")
        self.step_idx = 0
        self._step_dev = torch.zeros(1, dtype=torch.int64, device="cuda")  # == step_idx, read by the kernels
        self.flags = Flags()
        self._ws = {}
        self.graph = graph and est_count is None  # CUDA-graph replay of the whole step (single process)
        self._graph, self._gwarm = None, False
        self._refresh_bf16()

    # ------------------------------------------------------------------ views
    def view(self, layer: int, name: str, t: torch.Tensor | None = None) -> torch.Tensor:
        """Parameter `name` of `layer` as a view of the flat fp32 buffer (or of row e of grads)."""
        t = self.params if t is None else t
        o, shape = self.off[layer][name], self.shapes[name]
        return t[o:o + int(torch.Size(shape).numel())].view(shape)

    def eview(self, name: str, t: torch.Tensor | None = None) -> torch.Tensor:
        """Embedding-layer parameter (Wemb / Pemb / bdec) as a view of the flat buffer (or a gradient row)."""
        t = self.params if t is None else t
        o, shape = self.eoff[name], self.shapes[name]
        return t[o:o + int(torch.Size(shape).numel())].view(shape)

    def _ep(self, k):
        return self.params.data_ptr() + 4 * self.eoff[k]

    def _eg(self, base, k):  # local EST `base`'s gradient leaf for an embedding-layer parameter
        return self.grads.data_ptr() + 4 * ((base // self.g) * self.P + self.eoff[k])

    def _wb(self, l, k):
        return self.pb.data_ptr() + 2 * self.off[l][k]

    def _ewb(self, k):
        return self.pb.data_ptr() + 2 * self.eoff[k]

    def _p(self, l, k):
        return self.params.data_ptr() + 4 * self.off[l][k]

    def _g(self, base, l, k):  # local EST `base`'s gradient leaf for (layer, name); leaf j at + j*P floats
        return self.grads.data_ptr() + 4 * ((base // self.g) * self.P + self.off[l][k])

    def _refresh_bf16(self):
        _native.check(_native.lib().bt_cast_f32_bf16(self.params.data_ptr(), self.P, self.pb.data_ptr(), stream()),
                      "bert weight cast")

    # -------------------------------------------------------------- workspace
    def _workspace(self, n: int) -> dict:
        ws = self._ws.get(n)
        if ws is not None:
            return ws
        D, F, Te, T, L = self.D, self.F, self.Te, n * self.Te, self.L
        bf, f32 = dict(dtype=torch.bfloat16, device="cuda"), dict(dtype=torch.float32, device="cuda")
        ws = {
            "layers": [{"xb": torch.empty(T, D, **bf), "qkv": torch.empty(T, 3 * D, **bf),
                        "ctx": torch.empty(T, D, **bf), "hs1": torch.empty(T, D, **f32), "st1": torch.empty(T, 2, **f32),
                        "h1b": torch.empty(T, D, **bf), "Hpre": torch.empty(T, F, **bf),
                        "Dact": torch.empty(T, F, **bf), "hs2": torch.empty(T, D, **f32),
                        "st2": torch.empty(T, 2, **f32),
                        "ast": torch.empty(T * self.H, 2, **f32),  # attention row statistics
                        "amask": torch.empty(T * self.H, 4, dtype=torch.int32, device="cuda")}  # keep bits
                       for _ in range(L)],
            "x32": torch.empty(T, D, **f32), "y32": torch.empty(T, D, **f32),
            "brb": torch.empty(T, D, **bf), "ytop": torch.empty(T, D, **bf),
            "tgt": torch.empty(T, D, **f32), "dy1": [torch.empty(T, D, **bf) for _ in range(2)],
            "dres": [torch.empty(T, D, **f32) for _ in range(2)],
            "dbr": torch.empty(T, D, **bf), "dHpre": torch.empty(T, F, **bf), "dctx": torch.empty(T, D, **bf),
            "dqkv": torch.empty(T, 3 * D, **bf), "lnpart": torch.empty(n * (Te // 16) * 3 * D, **f32),
            "colsum": torch.empty(max(n * -(-Te // 32) * max(3 * D, F),
                                      (n // self.g) * -(-(self.g * self.S * self.NP) // 64) * self.Vp), **f32),
            "msepart": torch.empty(n * 64, **f32),
        }
        if self.head == "mlm":
            R, i32 = n * self.S * self.NP, dict(dtype=torch.int32, device="cuda")
            ws.update({"ids": torch.empty(T, **i32), "mrow": torch.empty(R, **i32), "mlabel": torch.empty(R, **i32),
                       "ym": torch.empty(R, D, **bf), "logits": torch.empty(R, self.Vp, **f32),
                       "dlogits": torch.empty(R, self.Vp, **bf), "rowloss": torch.empty(R, **f32),
                       "dym": torch.empty(R, D, **bf)})
            ni, nf = C.c_int64(), C.c_int64()
            _native.check(_native.lib().bt_bert_embed_grad_scratch(n // self.g, self.g * Te, D, C.byref(ni),
                                                                   C.byref(nf)), "embedding scratch")
            ws.update({"eg_int": torch.empty(ni.value, **i32), "eg_part": torch.empty(nf.value, **f32)})
        self._ws[n] = ws
        return ws

    # ------------------------------------------------------------- launchers
    def _gemm(self, a, b, c, M, N, K, out_bf16=False, bias=None, batch=1, sa=0, sb=0, sc=0):
        _native.check(_native.lib().bt_gemm_bf16_tn_ex(a, b, c, batch, M, N, K, sa, sb, sc, 1 if out_bf16 else 0,
                                                       bias, 0, stream()), "bert gemm")

    def _dx(self, a, w, c, M, N, K):
        """dX = dY . W with W [K = out][N = in] read as stored (B MN-major: bit-identical to dY . (W^T)^T)."""
        _native.check(_native.lib().bt_gemm_bf16_ex(a, w, c, 1, M, N, K, 0, 0, 0, 1, None, 2, 0, stream()),
                      "bert dX gemm")

    def _wgrad(self, ws, n, dy, x, rows_out, cols_in, dst):
        """Weight gradient of each gradient leaf, dW_j = dy_j^T x_j ([rows_out][cols_in], K = the leaf's
        tokens in EST order), read MN-major straight from the token-major activations and written into
        the leaf's slot (stride P): one batched launch, no transposed copies."""
        K = self.g * self.Te
        _native.check(_native.lib().bt_gemm_bf16_ex(dy, x, dst, n // self.g, rows_out, cols_in, K, rows_out * K,
                                                     cols_in * K, self.P, 0, None, 1, 0, stream()),
                      "bert weight-gradient gemm")

    def _group(self, lb: int, n: int, losses: torch.Tensor, capture: dict | None = None):
        """Forward/backward of local ESTs [lb, lb+n) (global ranks est0 + lb ...): per-EST gradients into
        grads[lb:lb+n]; every random draw keyed by the GLOBAL rank."""
        L, s = _native.lib(), stream()
        base, gg = self.est0 + lb, self.g
        sp = self._step_dev.data_ptr()  # the step counter lives on the device (CUDA-graph replays)
        D, F, H, Te, T, NL = self.D, self.F, self.H, self.Te, n * self.Te, self.L
        seed, step = self.seed & (2**64 - 1), self.step_idx
        ws = self._workspace(n)
        lay = ws["layers"]
        if self.head == "mlm":  # token ids + masked positions, then word + position embeddings
            _native.check(L.bt_bert_tokens(seed, step, sp, base, n, self.S, self.V, self.NP, self.mask_id,
                                           ws["ids"].data_ptr(), ws["mrow"].data_ptr(), ws["mlabel"].data_ptr(), s),
                          "bert tokens")
            _native.check(L.bt_bert_embed_fwd(ws["ids"].data_ptr(), self._ep("Wemb"), self._ep("Pemb"), T, D,
                                              ws["x32"].data_ptr(), lay[0]["xb"].data_ptr(), s), "bert embedding")
        else:
            _native.check(L.bt_bert_data(seed, step, base, n, Te, D, ws["x32"].data_ptr(), lay[0]["xb"].data_ptr(),
                                         ws["tgt"].data_ptr(), sp, s))
        x32 = ws["x32"]
        for l in range(NL):
            w = lay[l]
            self._gemm(w["xb"].data_ptr(), self._wb(l, "Wqkv"), w["qkv"].data_ptr(), T, 3 * D, D, out_bf16=True,
                       bias=self._p(l, "bqkv"))
            _native.check(L.bt_bert_attn_ex2(0, w["qkv"].data_ptr(), None, w["ctx"].data_ptr(), n, Te, D, H, base, NL,
                                             l, seed, step, self.pa, sp, w["ast"].data_ptr(),
                                             w["amask"].data_ptr() if _ATTN_BITS else None, s), "attention forward")
            self._gemm(w["ctx"].data_ptr(), self._wb(l, "Wo"), ws["brb"].data_ptr(), T, D, D, out_bf16=True)
            if l == 0:  # the embedding input is stored fp32; later residuals are recomputed (bt_bert_ln_fwd_rc)
                _native.check(L.bt_bert_ln_fwd(x32.data_ptr(), ws["brb"].data_ptr(), self._p(l, "bo"),
                                               self._p(l, "g1"), self._p(l, "be1"), w["hs1"].data_ptr(),
                                               w["st1"].data_ptr(), None, w["h1b"].data_ptr(), n, Te,
                                               D, base, NL, l, 0, seed, step, self.ph, self.eps, sp, s), "layernorm 1")
            else:
                pw = lay[l - 1]
                _native.check(L.bt_bert_ln_fwd_rc(pw["hs2"].data_ptr(), pw["st2"].data_ptr(), self._p(l - 1, "g2"),
                                                  self._p(l - 1, "be2"), ws["brb"].data_ptr(), self._p(l, "bo"),
                                                  self._p(l, "g1"), self._p(l, "be1"), w["hs1"].data_ptr(),
                                                  w["st1"].data_ptr(), None, w["h1b"].data_ptr(), n, Te, D, base, NL, l,
                                                  0, seed, step, self.ph, self.eps, sp, s), "layernorm 1")
            _native.check(L.bt_gemm_bf16_ffn(w["h1b"].data_ptr(), self._wb(l, "W1"), w["Hpre"].data_ptr(), T, F, D, 1,
                                             self._p(l, "b1"), None, w["Dact"].data_ptr(), seed, step, base, Te, 0.0,
                                             0, s), "ffn forward GEMM")
            self._gemm(w["Dact"].data_ptr(), self._wb(l, "W2"), ws["brb"].data_ptr(), T, D, F, out_bf16=True)
            # the fp32 LayerNorm-2 output is kept only where it is read: the loss (last layer), captures
            keep = l == NL - 1 or (capture is not None and l == 0)
            y32 = ws["y32"]
            yb = lay[l + 1]["xb"] if l + 1 < NL else ws["ytop"]
            _native.check(L.bt_bert_ln_fwd_rc(w["hs1"].data_ptr(), w["st1"].data_ptr(), self._p(l, "g1"),
                                              self._p(l, "be1"), ws["brb"].data_ptr(), self._p(l, "b2"),
                                              self._p(l, "g2"), self._p(l, "be2"), w["hs2"].data_ptr(),
                                              w["st2"].data_ptr(), y32.data_ptr() if keep else None, yb.data_ptr(), n,
                                              Te, D, base, NL, l, 1, seed, step, self.ph, self.eps, sp, s),
                          "layernorm 2")
            if capture is not None and l == 0:
                capture.update({k: w[k].clone() for k in ("xb", "qkv", "ctx", "hs1", "st1", "h1b", "Hpre", "Dact",
                                                          "hs2", "st2")})
                capture.update(x32=x32.clone(), y32=y32.clone())
            x32 = y32
        # gradients between GEMMs bf16 (A: into LN2', Db: into LN1'), residual-path gradients fp32 (B, Cb)
        (A, Db), (B, Cb) = ws["dy1"], ws["dres"]
        if self.head == "mlm":
            self._mlm_head(ws, n, lb, losses, capture)
        else:
            _native.check(L.bt_bert_mse(x32.data_ptr(), ws["tgt"].data_ptr(), n, Te, D, A.data_ptr(),
                                        ws["msepart"].data_ptr(), losses[lb:].data_ptr(), s))
        if capture is not None:
            capture.update(ytop=x32.clone(), tgt=ws["tgt"].clone())
        dy2 = None
        part = ws["lnpart"].data_ptr()
        for l in reversed(range(NL)):
            w = lay[l]
            if capture is not None and l == 0:
                capture.update(dy1_top=A.clone(), dy2_top=None if dy2 is None else dy2.clone())
            _native.check(L.bt_bert_ln_bwd(A.data_ptr(), None if dy2 is None else dy2.data_ptr(), w["hs2"].data_ptr(),
                                           w["st2"].data_ptr(), self._p(l, "g2"), Cb.data_ptr(), ws["dbr"].data_ptr(),
                                           part, n, Te, D, base, NL, l, 1, seed, step, self.ph, sp, s), "layernorm 2'")
            _native.check(L.bt_bert_ln_fold(part, n // gg, gg * Te, D, self._g(lb, l, "g2"), self._g(lb, l, "be2"),
                                            self._g(lb, l, "b2"), self.P, s))
            if capture is not None and l == 0:
                capture.update(dg=Cb.clone(), do=ws["dbr"].clone())
            # dHpre = (dbr . W2) * gelu'(h), with the b1 gradient's 32-row column partials from the epilogue
            _native.check(L.bt_gemm_bf16_ffn_cs(ws["dbr"].data_ptr(), self._wb(l, "W2"), ws["dHpre"].data_ptr(), T, F,
                                                D, 2 | 0x100, None, w["Hpre"].data_ptr(), None,
                                                ws["colsum"].data_ptr() if _FUSED_CS else None, seed, step, base, Te,
                                                0.0, 0, s),
                          "ffn backward GEMM")
            self._dx(ws["dHpre"].data_ptr(), self._wb(l, "W1"), Db.data_ptr(), T, D, F)
            self._wgrad(ws, n, ws["dbr"].data_ptr(), w["Dact"].data_ptr(), D, F, self._g(lb, l, "W2"))
            self._wgrad(ws, n, ws["dHpre"].data_ptr(), w["h1b"].data_ptr(), F, D, self._g(lb, l, "W1"))
            if _FUSED_CS:
                _native.check(L.bt_colsum_fold(ws["colsum"].data_ptr(), n // gg, gg * Te // 32, F,
                                               self._g(lb, l, "b1"), self.P, s), "b1 gradient")
            else:
                _native.check(L.bt_colsum_bf16_strided(ws["dHpre"].data_ptr(), n // gg, gg * Te, F,
                                                       self._g(lb, l, "b1"), self.P, ws["colsum"].data_ptr(), s))
            if capture is not None and l == 0:
                capture.update(dHpre=ws["dHpre"].clone(), dh1=Db.clone())
            _native.check(L.bt_bert_ln_bwd(Db.data_ptr(), Cb.data_ptr(), w["hs1"].data_ptr(), w["st1"].data_ptr(),
                                           self._p(l, "g1"), B.data_ptr(), ws["dbr"].data_ptr(), part, n, Te, D, base,
                                           NL, l, 0, seed, step, self.ph, sp, s), "layernorm 1'")
            _native.check(L.bt_bert_ln_fold(part, n // gg, gg * Te, D, self._g(lb, l, "g1"), self._g(lb, l, "be1"),
                                            self._g(lb, l, "bo"), self.P, s))
            self._dx(ws["dbr"].data_ptr(), self._wb(l, "Wo"), ws["dctx"].data_ptr(), T, D, D)
            self._wgrad(ws, n, ws["dbr"].data_ptr(), w["ctx"].data_ptr(), D, D, self._g(lb, l, "Wo"))
            _native.check(L.bt_bert_attn_ex2(1, w["qkv"].data_ptr(), ws["dctx"].data_ptr(), ws["dqkv"].data_ptr(), n,
                                             Te, D, H, base, NL, l, seed, step, self.pa, sp, w["ast"].data_ptr(),
                                             w["amask"].data_ptr() if _ATTN_BITS else None, s),
                          "attention backward")
            if capture is not None and l == 0:
                capture.update(dh=B.clone(), da=ws["dbr"].clone(), dctx=ws["dctx"].clone(), dqkv=ws["dqkv"].clone())
            self._dx(ws["dqkv"].data_ptr(), self._wb(l, "Wqkv"), A.data_ptr(), T, D, 3 * D)
            self._wgrad(ws, n, ws["dqkv"].data_ptr(), w["xb"].data_ptr(), 3 * D, D, self._g(lb, l, "Wqkv"))
            _native.check(L.bt_colsum_bf16_strided(ws["dqkv"].data_ptr(), n // gg, gg * Te, 3 * D,
                                                   self._g(lb, l, "bqkv"), self.P, ws["colsum"].data_ptr(), s))
            dy2 = B
        if capture is not None:
            capture["dx"] = A.clone()
            capture["dx_res"] = B.clone()
        if self.head == "mlm":  # the embedding gradient: dx = A (bf16) + B (fp32 residual path)
            _native.check(L.bt_bert_embed_grad(A.data_ptr(), B.data_ptr(), ws["ids"].data_ptr(), n // gg, gg * Te, D,
                                               ws["eg_int"].data_ptr(), ws["eg_part"].data_ptr(),
                                               self._eg(lb, "Wemb"), self._eg(lb, "Pemb"), self.P, s),
                          "embedding gradient")

    def _mlm_head(self, ws, n: int, lb: int, losses: torch.Tensor, capture: dict | None) -> None:
        """Masked-LM head of local ESTs [lb, lb+n): gather the masked rows of the top layer's output, logits
        against the tied word embedding (+ bias) on the tensor cores, softmax cross-entropy (per-EST mean
        over its masked rows), then dy_m = dlogits W_emb scattered back to the masked rows (A), the decoder
        weight gradient dlogits^T y_m and bias column sums into each gradient leaf."""
        L, s = _native.lib(), stream()
        D, T, Vp, gg = self.D, n * self.Te, self.Vp, self.g
        R, per = n * self.S * self.NP, self.S * self.NP
        A = ws["dy1"][0]
        ym, lg, dl = ws["ym"], ws["logits"], ws["dlogits"]
        _native.check(L.bt_rows_gather(ws["ytop"].data_ptr(), ws["mrow"].data_ptr(), R, D, ym.data_ptr(), s), "mlm gather")
        self._gemm(ym.data_ptr(), self._ewb("Wemb"), lg.data_ptr(), R, Vp, D, bias=self._ep("bdec"))
        _native.check(L.bt_bert_mlm_ce(lg.data_ptr(), ws["mlabel"].data_ptr(), R, self.V, Vp, n, per, dl.data_ptr(),
                                       ws["rowloss"].data_ptr(), losses[lb:].data_ptr(), s), "mlm cross-entropy")
        self._dx(dl.data_ptr(), self._ewb("Wemb"), ws["dym"].data_ptr(), R, D, Vp)
        _native.check(L.bt_rows_scatter(ws["dym"].data_ptr(), ws["mrow"].data_ptr(), R, self.NP, T, D, A.data_ptr(), s),
                      "mlm scatter")
        K = gg * per  # decoder weight gradient per leaf: dlogits_j^T y_m_j (MN-major operands, K = the leaf's rows)
        _native.check(L.bt_gemm_bf16_ex(dl.data_ptr(), ym.data_ptr(), self._eg(lb, "Wemb"), n // gg, Vp, D, K, Vp * K,
                                        D * K, self.P, 0, None, 1, 0, s), "mlm decoder weight gradient")
        _native.check(L.bt_colsum_bf16_strided(dl.data_ptr(), n // gg, K, Vp, self._eg(lb, "bdec"), self.P,
                                               ws["colsum"].data_ptr(), s), "mlm decoder bias gradient")
        if capture is not None:
            capture.update({k: ws[k].clone() for k in ("ids", "mrow", "mlabel", "ym", "logits", "dlogits", "dym")})
            capture["ytop_b"] = ws["ytop"].clone()

    # ------------------------------------------------------------------ step
    def step(self, groups: list[int] | None = None, capture: dict | None = None, check: bool = True) -> torch.Tensor:
        """One mini-batch of this process's ESTs; `groups` = EST counts per launch group (default: one group).
        Returns the local per-EST losses [est_count] (fp32, on device).  check=False defers the host-side
        non-finite check (no per-step synchronisation; `check_status()` later): the update is guarded on the
        device either way -- a non-finite step and every step after it leave the weights unchanged."""
        groups = groups or [self.En]
        if sum(groups) != self.En or min(groups) < 1 or any(n % self.g for n in groups):
            raise ConfigError(f"groups {groups} must partition {self.En} ESTs into whole gradient leaves of {self.g}")
        replay = self.graph and capture is None and self.peer is None and self.adam is None and groups == [self.En]
        if replay and self._gwarm:
            if self._graph is None:  # capture once (the captured work runs at the first replay)
                self._gloss = torch.empty(self.En, dtype=torch.float32, device="cuda")
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self._body(groups, self._gloss)
                self._graph = g
            self._graph.replay()
            self._post(check)
            return self._gloss.clone()
        losses = torch.empty(self.En, dtype=torch.float32, device="cuda")
        self._body(groups, losses, capture)
        self._post(check)
        self._gwarm = self._gwarm or replay
        return losses

    def _body(self, groups, losses, capture=None):
        """Everything a step puts on the stream (capturable: no host synchronisation, no allocation)."""
        base = 0
        for n in groups:
            self._group(base, n, losses, capture if len(groups) == 1 else None)
            base += n
        if capture is not None:
            capture["grads"] = self.grads.clone()
        self._reduce_update()
        self._refresh_bf16()
        self._step_dev.add_(1)

    def _post(self, check: bool = True):
        """Host side of a step: the non-finite check (one status read) and the step count."""
        self.step_idx += 1
        if check:
            self.check_status()

    def check_status(self):
        """The non-finite check of every step since the last one (the status words are sticky)."""
        if self.peer is not None:
            self.peer.check()
            return
        st, _, _ = self.flags.status()
        if st:
            self.flags.reset()
            raise NumericError("bert: non-finite synchronized gradient")

    def _stage(self) -> torch.Tensor:
        """Staging buffer of the guarded update (the synchronized gradients, checked before any write)."""
        st = getattr(self, "_stage_buf", None)
        if st is None or st.numel() != self.P:
            st = self._stage_buf = torch.empty(self.P, dtype=torch.float32, device="cuda")
        return st

    def fingerprint(self) -> str:
        """FNV fingerprint of the fp32 master weights (runlog.device_fingerprint: 64 KB slices hashed on the
        GPU, then on the host) -- the model-stack counterpart of the reference's per-step param_hash."""
        from .runlog import device_fingerprint

        return device_fingerprint(self.params)

    def run_log(self, steps: int, log=None, every: int = 1, groups=None):
        """`steps` mini-batches recorded like the reference's run_training (scenarios.py:69-80): per step
        the per-EST losses (binary64 hex on disk) and, every `every` steps (sampled: the weights are
        hundreds of MB), the weight fingerprint; returns the RunLog (comparable with runlog.bitdiff)."""
        from .runlog import RunLog, RunRecord

        if log is None:
            log = RunLog(self.E, "d1", self.seed)
        for _ in range(steps):
            losses = self.step(groups) if groups is not None else self.step()
            n = self.step_idx
            h = self.fingerprint() if every and n % every == 0 else ""
            log.add(RunRecord(n, [float(x) for x in losses.tolist()], h))
        return log

    def attach_peer(self, group=None):
        """Multi-GPU (one process per GPU, torch.distributed initialised, rank r holding the r-th contiguous
        EST block): the exchange becomes paper_2208_14228_b200.peer.PeerGroupReducer over CUDA IPC --
        Tree(2): each rank's subtree partial, then the owner of each parameter shard folds the G partials
        with NVLink peer loads (the same association as the flat tree); Sequential: the owner reads all E
        slots in rank order.  Fused /E + momentum SGD, updated shard stored into every replica."""
        from .hier import RankBuffers
        from .peer import PeerGroupReducer

        loc = RankBuffers(self.grads, self.params, self.vel, torch.cuda.current_stream(), vel2=self.vel2)
        self.peer = PeerGroupReducer(loc, self.E // self.g, "rank_tree2" if self.fanin == 2 else "sequential", None,
                                     self.lr, self.mu, group, divisor=self.E, adam=self.adam)

    def _reduce_update(self):
        """Fixed EST-rank-order sum of the E gradient slots, /E, momentum SGD: one launch over all P
        (or, across processes, the peer-memory reducer)."""
        if self.peer is not None:
            self.peer.step()
            return
        if self.En != self.E:
            raise ConfigError("a partial EST block needs attach_peer() for the exchange")
        a = _native.ReduceArgs()
        leaves = self.E // self.g
        a.dtype, a.mode, a.E, a.fanin, a.n = _native.DTYPE_F32, _native.REDUCE_UPDATE, leaves, self.fanin, self.P
        a.divisor = self.E
        for k in range(leaves):
            a.grads[k] = self.grads.data_ptr() + 4 * k * self.P
        p, v = self.params.data_ptr(), self.vel.data_ptr()
        a.param, a.vel, a.param_out, a.vel_out = p, v, p, v
        a.lr, a.mu, a.flags = self.lr, self.mu, self.flags.t.data_ptr()
        a.stage = self._stage().data_ptr()  # guarded: a non-finite step changes nothing (model.py:207-209)
        if self.adam is not None:
            t = self.step_idx + 1
            a.mode = _native.REDUCE_ADAM
            a.vel2 = a.vel2_out = self.vel2.data_ptr()
            a.beta2, a.eps = self.adam
            a.bc1, a.bc2 = 1.0 / (1.0 - self.mu ** t), 1.0 / (1.0 - self.adam[0] ** t)
        _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()), "bert reduce_update")

    # ---------------------------------------------------------------- sizes
    def gemm_flops_per_step(self) -> float:
        """Dense-layer flops: forward 2*T*P_w, backward dX + dW 4*T*P_w (P_w = weight-matrix params); the
        masked-LM decoder adds 6 * R * Vp * D (R = masked rows)."""
        pw = sum(int(torch.Size(self.shapes[k]).numel()) for k in _MATS) * self.L
        head = 6.0 * self.En * self.S * self.NP * self.Vp * self.D if self.head == "mlm" else 0.0
        return 6.0 * self.En * self.Te * pw + head

    def attn_flops_per_step(self) -> float:
        """QK^T and PV: 4*128*128*64 per (sequence, head) forward; backward recomputes S (+1) and does 4 more."""
        per = 4 * 128 * 128 * 64 / 2  # one 128x128x64 product = 2*128*128*64 flops
        return (2 + 5) * per * self.En * self.S * self.H * self.L
