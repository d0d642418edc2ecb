"""Per-EST ResNet-18 training step with BatchNorm and elastic rescale -- C3
(BASELINE.json configs[2]).

CIFAR ResNet-18 (3x3 stem, 4 stages x 2 BasicBlocks of widths 64-128-256-512,
1x1 stride-2 downsample shortcuts, 4x4 average pool, 10-way linear head,
softmax cross-entropy) trained data-parallel by E ESTs of B images each.
The EasyScale properties it keeps (paper §3.2, D1):

* per-EST state -- each EST's BatchNorm running statistics and its sampler
  cursor -- lives in HBM slots indexed by the EST's rank and travels with the
  EST: `rescale(G)` redistributes the slots onto a new number of "GPUs"
  (launch groups of contiguous EST blocks, `engine.assign_ranks`) with the
  128-bit slot-copy kernel (bt_est_slot_copy), the context switch of
  SURVEY §7 D5;
* every EST normalises with its own micro-batch statistics (no cross-EST
  BatchNorm), all randomness is keyed by (seed, EST rank, EST cursor), every
  reduction has a shape fixed by the EST's own data, and the per-EST gradients
  are summed by the fixed-order reducer -- so losses, weights and BN statistics
  are bit-identical for any mapping and across an 8 -> 4 -> 2 rescale
  (tests/test_gpu_resnet.py).

Convolutions are im2col GEMMs on the deterministic tcgen05 kernel; dX is the
transposed convolution as an im2col gather (no scatter-add), dW one MN-major
batched GEMM per EST.  The stem's 3 input channels are zero-padded to 8.
There is no reference implementation of this model.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from . import _native
from .device import Flags, require_cuda, stream
from .errors import ConfigError, NumericError

WIDTHS = (64, 128, 256, 512)
CLASSES = 10


def _init_uniform(seed: int, n: int, scale: float) -> torch.Tensor:
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().bt_init_random(seed & (2**64 - 1), scale, n, out.data_ptr(), stream()))
    return out.float()


def _round8(n: int) -> int:
    return (n + 7) // 8 * 8


def est_blocks(ests: int, gpus: int) -> list[tuple[int, int]]:
    """(first EST, count) per GPU: the reference's EST -> executor mapper (engine.assign_ranks,
    engine.py:169-199: contiguous blocks, balanced, larger shares first)."""
    from .engine import ExecutorSpec, assign_ranks

    if gpus < 1:
        raise ConfigError(f"{gpus} GPUs")
    return [(ranks[0], len(ranks)) for _, ranks in assign_ranks([ExecutorSpec("gpu")] * gpus, ests)]


class _Conv:
    def __init__(self, name, ci, co, k, s, hin):
        self.name, self.ci, self.co, self.k, self.s, self.hin = name, ci, co, k, s, hin
        self.p = k // 2
        self.hout = (hin + 2 * self.p - k) // s + 1
        self.taps = k * k
        self.K = self.taps * ci


class ResNetJob:
    """E ESTs x B images (32 x 32 x 3), ResNet-18 with per-EST BatchNorm, momentum SGD, `groups` "GPUs"."""

    def __init__(self, ests: int = 16, batch: int = 32, gpus: int = 8, seed: int = 42, lr: float = 0.02,
                 momentum: float = 0.9, fanin: int = 0, eps: float = 1e-5, est_base: int = 0,
                 est_count: int | None = None, graph: bool = True):
        """`gpus`: launch groups ("GPUs") of this process's ESTs.  `est_base` / `est_count`: this process
        holds ESTs [est_base, est_base + est_count) of the E (one rank of a multi-GPU job, `attach_peer`)."""
        require_cuda()
        if ests < 1 or ests > _native.BT_MAX_TABLE:
            raise ConfigError(f"1..{_native.BT_MAX_TABLE} ESTs per job")
        if fanin not in (0, 2) or (fanin == 2 and ests & (ests - 1)):
            raise ConfigError("allreduce variant: Sequential (0) or Tree(2) with a power-of-two EST count")
        self.E, self.B, self.seed, self.lr, self.mu, self.fanin, self.eps = ests, batch, seed, lr, momentum, fanin, eps
        self.est0, self.En = est_base, ests if est_count is None else est_count
        if self.est0 < 0 or self.En < 1 or self.est0 + self.En > ests:
            raise ConfigError(f"local EST block [{est_base}, +{est_count}) outside the {ests} ESTs")
        self.peer = None
        self.graph = graph
        convs = [_Conv("stem", 8, 64, 3, 1, 32)]
        blocks = []
        ci, h = 64, 32
        for si, w in enumerate(WIDTHS):
            for bi in range(2):
                s = 2 if (si > 0 and bi == 0) else 1
                a = _Conv(f"l{si + 1}.{bi}.a", ci, w, 3, s, h)
                b = _Conv(f"l{si + 1}.{bi}.b", w, w, 3, 1, a.hout)
                d = _Conv(f"l{si + 1}.{bi}.d", ci, w, 1, s, h) if (s != 1 or ci != w) else None
                convs += [a, b] + ([d] if d else [])
                blocks.append((a, b, d))
                ci, h = w, a.hout
        self.convs, self.blocks = convs, blocks
        # flat fp32 parameters: per conv W [Co][taps][Ci], gamma [Co], beta [Co]; then fc W [10][512], b [10]
        self.off, o = {}, 0
        for cv in convs:
            self.off[cv.name] = (o, o + _round8(cv.co * cv.K), o + _round8(cv.co * cv.K) + _round8(cv.co))
            o += _round8(cv.co * cv.K) + 2 * _round8(cv.co)
        self.off_fc = (o, o + CLASSES * 512)
        o += CLASSES * 512 + _round8(CLASSES)
        self.P = _round8(o)
        self.params = torch.zeros(self.P, dtype=torch.float32, device="cuda")
        for i, cv in enumerate(convs):
            w0, g0, _ = self.off[cv.name]
            fan_in = cv.taps * (3 if cv.name == "stem" else cv.ci)
            w = _init_uniform(seed * 7919 + i, cv.co * cv.K, (6.0 / fan_in) ** 0.5).view(cv.co, cv.taps, cv.ci)
            if cv.name == "stem":
                w[:, :, 3:] = 0.0  # padded input channels
            self.params[w0:w0 + cv.co * cv.K] = w.reshape(-1)
            self.params[g0:g0 + cv.co] = 1.0
        self.params[self.off_fc[0]:self.off_fc[0] + CLASSES * 512] = _init_uniform(seed * 7919 + 999, CLASSES * 512,
                                                                                   (1.0 / 512) ** 0.5)
        self.vel = torch.zeros_like(self.params)
        self.grads = torch.zeros(self.En, self.P, dtype=torch.float32, device="cuda")  # padding stays 0
        # BatchNorm channel offsets inside an EST's running-statistics slot
        self.bn_off, c = {}, 0
        for cv in convs:
            self.bn_off[cv.name] = c
            c += cv.co
        self.CBN = c
        # bf16 operand copies of the conv weights: wb [Co][taps*Ci] (forward), wt [Ci][taps][Co] (dX)
        tot = sum(cv.co * cv.K for cv in convs)
        self.wb = torch.empty(tot, dtype=torch.bfloat16, device="cuda")
        self.wt = torch.empty(tot, dtype=torch.bfloat16, device="cuda")
        self.woff, m = {}, 0
        for cv in convs:
            self.woff[cv.name] = m
            m += cv.co * cv.K
        n = len(convs)
        self._cast = [(C.c_void_p * n)(), (C.c_void_p * n)(), (C.c_void_p * n)(), (C.c_int32 * n)(),
                      (C.c_int32 * n)(), (C.c_int32 * n)(), (C.c_int32 * n)()]
        for i, cv in enumerate(convs):
            self._cast[0][i] = self.params.data_ptr() + 4 * self.off[cv.name][0]
            self._cast[1][i] = self.wb.data_ptr() + 2 * self.woff[cv.name]
            self._cast[2][i] = self.wt.data_ptr() + 2 * self.woff[cv.name]
            self._cast[3][i], self._cast[4][i], self._cast[5][i] = cv.co, cv.taps, cv.ci
            self._cast[6][i] = 1  # stride-1 dX = a forward convolution of dz with the flipped filter
        # stride-2 dX by output parity class: per (conv, class) the taps that reach it, as a stride-1
        # convolution of dz (offsets (a + p - kh) / 2 from 0) with a class filter [Ci][Tc][Co] (bf16)
        self.cls, ents, m = {}, [], 0
        for cv in convs:
            if cv.s != 2:
                continue
            lst = []
            for a in (0, 1):
                for b in (0, 1):
                    th = sorted((kh for kh in range(cv.k) if (a + cv.p - kh) % 2 == 0), key=lambda kh: -kh)
                    tw = sorted((kw for kw in range(cv.k) if (b + cv.p - kw) % 2 == 0), key=lambda kw: -kw)
                    if not th or not tw:
                        lst.append(None)
                        continue
                    assert [(a + cv.p - kh) // 2 for kh in th] == list(range(len(th)))
                    assert [(b + cv.p - kw) // 2 for kw in tw] == list(range(len(tw)))
                    src = [kh * cv.k + kw for kh in th for kw in tw]
                    lst.append((len(th), len(tw), m))
                    ents.append((cv, src, m))
                    m += cv.ci * len(src) * cv.co
            self.cls[cv.name] = lst
        self.wcls = torch.empty(max(m, 1), dtype=torch.bfloat16, device="cuda")
        k = len(ents)
        self._taps = [(C.c_void_p * k)(), (C.c_void_p * k)(), (C.c_int32 * k)(), (C.c_int32 * k)(),
                      (C.c_int32 * k)(), (C.c_int32 * k)(), (C.c_int32 * (9 * k))(), k]
        for i, (cv, src, off) in enumerate(ents):
            self._taps[0][i] = self.params.data_ptr() + 4 * self.off[cv.name][0]
            self._taps[1][i] = self.wcls.data_ptr() + 2 * off
            self._taps[2][i], self._taps[3][i], self._taps[4][i], self._taps[5][i] = cv.co, cv.taps, cv.ci, len(src)
            for t, v in enumerate(src):
                self._taps[6][9 * i + t] = v
        self.flags = Flags()
        self.step_idx = 0
        self._ws = {}
        # per-EST slots, held by the "GPU" (launch group) that owns the EST
        self.G = 0
        self.slots = []
        self._place(gpus, initial=True)
        self._refresh_bf16()

    # ------------------------------------------------------------ EST slots
    def layout(self, gpus: int) -> list[tuple[int, int]]:
        return est_blocks(self.En, gpus)

    def _new_slots(self, n: int) -> dict:
        return {"run_mean": torch.zeros(n, self.CBN, dtype=torch.float32, device="cuda"),
                "run_var": torch.ones(n, self.CBN, dtype=torch.float32, device="cuda"),
                "cursor": torch.zeros(n, dtype=torch.int64, device="cuda")}

    def _slot_set(self, gpus: int) -> list[dict]:
        """The slot buffers of layout `gpus` (one set per layout, allocated once: a layout's CUDA graph
        keeps pointing at them, so re-entering a layout replays its graph)."""
        if gpus not in self._slot_sets:
            self._slot_sets[gpus] = [self._new_slots(n) for _, n in self.layout(gpus)]
        return self._slot_sets[gpus]

    def _copy_plan(self, g0: int, g1: int):
        """(dst, src, bytes, count) ctypes arrays moving every EST's slot bytes from layout g0 to g1."""
        key = (g0, g1)
        if key not in self._plans:
            owner = {}
            for g, (base, n) in enumerate(self.layout(g0)):
                for k in range(n):
                    owner[base + k] = (g, k)
            old, new = self._slot_set(g0), self._slot_set(g1)
            dst, src, nb = [], [], []
            for g, (base, n) in enumerate(self.layout(g1)):
                for k in range(n):
                    og, ok = owner[base + k]
                    for name in ("run_mean", "run_var", "cursor"):
                        d, s_ = new[g][name][k], old[og][name][ok]
                        dst.append(d.data_ptr())
                        src.append(s_.data_ptr())
                        nb.append(d.numel() * d.element_size())
            cnt = len(dst)
            self._plans[key] = ((C.c_void_p * cnt)(*dst), (C.c_void_p * cnt)(*src), (C.c_int64 * cnt)(*nb), cnt)
        return self._plans[key]

    def _place(self, gpus: int, initial: bool = False):
        if initial:
            self._slot_sets, self._plans, self._graphs = {}, {}, {}
            self.slots, self.G = self._slot_set(gpus), gpus
            self._graph, self._gwarm = None, False
            return
        if gpus == self.G:
            return
        # the EST context switch: every EST's slot bytes move to its new owner in ONE launch
        dst, src, nb, cnt = self._copy_plan(self.G, gpus)
        _native.check(_native.lib().bt_est_slot_copy(dst, src, nb, cnt, stream()), "EST slot copy")
        self.slots, self.G = self._slot_set(gpus), gpus
        self._graph = self._graphs.get(gpus)  # a prepared / previously captured layout replays at once
        self._gwarm = self._graph is not None

    def rescale(self, gpus: int):
        """Elastic rescale onto `gpus` launch groups: per-EST slots move, parameters are replicated."""
        self._place(gpus)

    def prepare(self, gpus: int) -> None:
        """Stage layout `gpus` before a rescale needs it (EasyScale's planner knows the next layout): its slot
        buffers, the copy plans from/to the current layout, the launch groups' workspaces and the CUDA graph
        of its step -- captured, not run, so the training state does not move.  A later rescale(gpus) is then
        one slot-copy launch and the next step a graph replay."""
        if not self.graph or self.peer is not None or gpus in self._graphs:
            return
        for _, n in self.layout(gpus):
            self._workspace(n)
        for g in set(self._slot_sets) | {self.G}:  # copy plans to and from every staged layout
            if g != gpus:
                self._copy_plan(g, gpus)
                self._copy_plan(gpus, g)
        cur = (self.slots, self.G)
        self.slots, self.G = self._slot_set(gpus), gpus
        try:
            self._capture(gpus)
        finally:
            self.slots, self.G = cur

    def _capture(self, gpus: int):
        self._stage()  # allocated outside the graph's private pool
        gloss = torch.empty(self.En, dtype=torch.float32, device="cuda")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._body(gloss)
        self._graphs[gpus] = (g, gloss)
        return self._graphs[gpus]

    def est_state(self) -> dict:
        """Per-EST slots gathered in EST-rank order (for comparisons across mappings)."""
        return {k: torch.cat([s[k] for s in self.slots]) for k in ("run_mean", "run_var", "cursor")}

    def implicit(self, cv) -> bool:
        """Convolution as an implicit GEMM (TMA im2col loads, bt_gemm_conv): 64-channel-block inputs and
        64-pixel EST blocks; the stem (3 -> 8 padded channels) keeps the explicit im2col.  BT_CONV_EXPLICIT=1
        forces the explicit im2col path (the same tiles and K order: the same bits)."""
        return cv.ci % 64 == 0 and (self.B * cv.hout ** 2) % 64 == 0 and os.environ.get("BT_CONV_EXPLICIT") != "1"

    def implicit_dx(self, cv) -> bool:
        """The input gradient as an implicit GEMM: a stride-1 convolution over dz (stride 1: the whole
        gradient; stride 2: one output parity class), input channels cv.co, output pixels dz's grid."""
        return cv.co % 64 == 0 and (self.B * cv.hout ** 2) % 64 == 0 and os.environ.get("BT_CONV_EXPLICIT") != "1"

    def splits(self, cv) -> int:
        """Pinned pixel splits of an EST's weight-gradient reduction (a function of the shape only)."""
        return max(1, (self.B * cv.hout ** 2) // 2048)

    # ------------------------------------------------------------ workspace
    def _refresh_bf16(self):
        c, t = self._cast, self._taps
        _native.check(_native.lib().bt_cnn_conv_weights(c[0], c[1], c[2], c[3], c[4], c[5], c[6], len(c[3]), stream()),
                      "conv weight cast")
        if t[7]:
            _native.check(_native.lib().bt_cnn_filter_taps(t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], stream()),
                          "class filters")

    def _workspace(self, n: int) -> dict:
        ws = self._ws.get(n)
        if ws is not None:
            return ws
        B = self.B
        bf, f32 = dict(dtype=torch.bfloat16, device="cuda"), dict(dtype=torch.float32, device="cuda")
        col = 0  # the dX gathers of explicit fallbacks (stride 1: 9 taps; stride 2: a class's <= 4 taps)
        for cv in self.convs:
            if cv.name != "stem" and not self.implicit_dx(cv):
                col = max(col, n * B * cv.hout ** 2 * cv.taps * cv.co)
        ws = {"img": torch.empty(n * B * 1024 * 8, **bf), "labels": torch.empty(n * B, dtype=torch.int32, device="cuda"),
              "col": torch.empty(col, **bf), "loss": torch.empty(n, **f32)}
        for cv in self.convs:
            R = n * B * cv.hout ** 2
            ws[cv.name] = {"z": torch.empty(R * cv.co, **bf), "y": torch.empty(R * cv.co, **bf),
                           "mean": torch.empty(n * cv.co, **f32), "rstd": torch.empty(n * cv.co, **f32)}
            if not self.implicit(cv):  # explicit forward im2col, kept for the dW product
                ws[cv.name]["col"] = torch.empty(R * cv.K, **bf)
        big = max(n * B * cv.hin ** 2 * max(cv.ci, cv.co) for cv in self.convs)
        ws["g"] = [torch.empty(big, **bf) for _ in range(4)]
        ws["wpart"] = torch.empty(max(n * self.splits(cv) * cv.co * cv.K for cv in self.convs), **f32)
        ws["sg"] = torch.empty(n * 512, **f32)
        ws["sgx"] = torch.empty(n * 512, **f32)
        chunks = max((B * cv.hout ** 2 + 255) // 256 for cv in self.convs)
        ws["part"] = torch.empty(n * chunks * 2 * 512, **f32)
        self._ws[n] = ws
        return ws

    # ------------------------------------------------------------ layers
    def _conv_fwd(self, ws, cv, x, n, z):
        L, s = _native.lib(), stream()
        R = n * self.B * cv.hout ** 2
        wb = self.wb.data_ptr() + 2 * self.woff[cv.name]
        if self.implicit(cv):
            _native.check(L.bt_gemm_conv(0, x.data_ptr(), n * self.B, cv.hin, cv.hin, cv.ci, cv.hout, cv.hout, cv.k,
                                         cv.k, cv.s, cv.p, wb, z.data_ptr(), cv.co, 1, 0, 0, 1, s), "conv (implicit)")
            return
        col = ws[cv.name]["col"]
        _native.check(L.bt_cnn_im2col(x.data_ptr(), col.data_ptr(), n * self.B, cv.hin, cv.hin, cv.ci, cv.hout,
                                      cv.hout, cv.k, cv.k, cv.s, cv.p, 0, s), "im2col")
        _native.check(L.bt_gemm_bf16_ex(col.data_ptr(), wb, z.data_ptr(), 1, R, cv.co, cv.K, 0, 0, 0, 1, None, 0, 0, s),
                      "conv gemm")

    def _bn_fwd(self, ws, cv, n, gslot, res=None, relu=True, out=None):
        L, s = _native.lib(), stream()
        w = ws[cv.name]
        Re = self.B * cv.hout ** 2
        _, g0, b0 = self.off[cv.name]
        sl = self.slots[gslot]
        rm = sl["run_mean"].data_ptr() + 4 * self.bn_off[cv.name]
        rv = sl["run_var"].data_ptr() + 4 * self.bn_off[cv.name]
        _native.check(L.bt_cnn_bn_stats(0, w["z"].data_ptr(), None, None, w["mean"].data_ptr(), w["rstd"].data_ptr(),
                                        None, None, ws["part"].data_ptr(), rm, rv, self.CBN, None, None, 0, n, Re,
                                        cv.co, self.eps, s), "bn stats")
        out = w["y"] if out is None else out
        _native.check(L.bt_cnn_bn_apply(w["z"].data_ptr(), None if res is None else res.data_ptr(),
                                        w["mean"].data_ptr(), w["rstd"].data_ptr(),
                                        self.params.data_ptr() + 4 * g0, self.params.data_ptr() + 4 * b0, n, Re,
                                        cv.co, 1 if relu else 0, out.data_ptr(), s), "bn apply")

    def _bn_bwd(self, ws, cv, n, base, dy, y, dz):
        """dz of BN(z) whose (block) output y got gradient dy (through the ReLU mask of y)."""
        L, s = _native.lib(), stream()
        w = ws[cv.name]
        Re = self.B * cv.hout ** 2
        _, g0, b0 = self.off[cv.name]
        gp = self.grads.data_ptr() + 4 * base * self.P
        _native.check(L.bt_cnn_bn_stats(2, w["z"].data_ptr(), dy.data_ptr(), y.data_ptr(), w["mean"].data_ptr(),
                                        w["rstd"].data_ptr(), ws["sg"].data_ptr(), ws["sgx"].data_ptr(),
                                        ws["part"].data_ptr(), None, None, 0, gp + 4 * g0, gp + 4 * b0, self.P, n, Re,
                                        cv.co, self.eps, s), "bn backward sums")
        _native.check(L.bt_cnn_bn_bwd(w["z"].data_ptr(), dy.data_ptr(), y.data_ptr(), w["mean"].data_ptr(),
                                      w["rstd"].data_ptr(), ws["sg"].data_ptr(), ws["sgx"].data_ptr(),
                                      self.params.data_ptr() + 4 * g0, n, Re, cv.co, dz.data_ptr(), s), "bn backward")

    def _conv_bwd(self, ws, cv, n, base, x, dz, dx):
        """dW_e into each EST's gradient slot (implicit GEMM over the EST's output pixels, or the forward's
        explicit im2col) and, if dx is given, the input gradient (`_dx`: stride 2 returns its parity
        classes)."""
        L, s, B = _native.lib(), stream(), self.B
        Re = B * cv.hout ** 2
        gdst = self.grads.data_ptr() + 4 * (base * self.P + self.off[cv.name][0])
        # fixed split-K: the EST's pixels in `sp` pinned splits of >= 2048 (more output tiles in flight),
        # partials folded in split order
        sp = self.splits(cv)
        Rs = Re // sp
        # one split: the product lands in the EST's gradient slot directly (batch stride P)
        part, pst = (ws["wpart"].data_ptr(), cv.co * cv.K) if sp > 1 else (gdst, self.P)
        if self.implicit(cv):
            _native.check(L.bt_gemm_conv(1, x.data_ptr(), n * B, cv.hin, cv.hin, cv.ci, cv.hout, cv.hout, cv.k, cv.k,
                                         cv.s, cv.p, dz.data_ptr(), part, cv.co, n * sp, Rs, pst, 0, s),
                          "conv dW (implicit)")
        else:
            _native.check(L.bt_gemm_bf16_ex(dz.data_ptr(), ws[cv.name]["col"].data_ptr(), part, n * sp, cv.co, cv.K,
                                            Rs, Rs * cv.co, Rs * cv.K, pst, 0, None, 1, 0, s), "conv dW gemm")
        if sp > 1:
            _native.check(L.bt_fold_splits(part, n, sp, cv.co * cv.K, gdst, self.P, s), "dW split fold")
        if dx is None:
            return None
        return self._dx(ws, cv, n, dz, dx)

    def _dx(self, ws, cv, n, dz, dx):
        """Stride 1: dx = a forward convolution of dz with the flipped filter.  Stride 2: the four output
        parity classes, each a stride-1 convolution of dz with its class filter, into the four quarters
        of `dx`'s buffer; returns their pointers (None for a class no tap reaches) for bt_cnn_add_s2."""
        if cv.s == 1:
            wt = self.wt.data_ptr() + 2 * self.woff[cv.name]
            self._conv_s1(ws, cv, n, dz.data_ptr(), cv.k, cv.k, cv.k - 1 - cv.p, wt, dx.data_ptr())
            return None
        q = n * self.B * cv.hout ** 2 * cv.ci  # one class's elements
        out = []
        for i, c in enumerate(self.cls[cv.name]):
            if c is None:
                out.append(None)
                continue
            kh, kw, off = c
            dst = dx.data_ptr() + 2 * i * q
            self._conv_s1(ws, cv, n, dz.data_ptr(), kh, kw, 0, self.wcls.data_ptr() + 2 * off, dst)
            out.append(dst)
        return out

    def _conv_s1(self, ws, cv, n, src, kh, kw, pad, w, dst):
        """A stride-1 convolution over dz's grid (cv.hout square, cv.co channels) into cv.ci channels."""
        L, s, B, h = _native.lib(), stream(), self.B, cv.hout
        if self.implicit_dx(cv):
            _native.check(L.bt_gemm_conv(0, src, n * B, h, h, cv.co, h, h, kh, kw, 1, pad, w, dst, cv.ci, 1, 0, 0, 1, s),
                          "conv dX (implicit)")
            return
        _native.check(L.bt_cnn_im2col(src, ws["col"].data_ptr(), n * B, h, h, cv.co, h, h, kh, kw, 1, pad, 0, s),
                      "dX im2col")
        _native.check(L.bt_gemm_bf16_ex(ws["col"].data_ptr(), w, dst, 1, n * B * h * h, cv.ci, kh * kw * cv.co, 0, 0,
                                        0, 1, None, 0, 0, s), "conv dX gemm")

    def _group(self, gslot: int, base: int, n: int, losses: torch.Tensor, capture: dict | None):
        L, s, B = _native.lib(), stream(), self.B
        ws = self._workspace(n)
        sl = self.slots[gslot]
        _native.check(L.bt_cnn_data(self.seed & (2**64 - 1), sl["cursor"].data_ptr(), self.est0 + base, n, B,
                                    ws["img"].data_ptr(), ws["labels"].data_ptr(), s))
        stem = self.convs[0]
        self._conv_fwd(ws, stem, ws["img"], n, ws["stem"]["z"])
        self._bn_fwd(ws, stem, n, gslot)
        x = ws["stem"]["y"]
        ins = []
        for a, b, d in self.blocks:
            ins.append(x)
            self._conv_fwd(ws, a, x, n, ws[a.name]["z"])
            self._bn_fwd(ws, a, n, gslot)
            self._conv_fwd(ws, b, ws[a.name]["y"], n, ws[b.name]["z"])
            res = x
            if d is not None:
                self._conv_fwd(ws, d, x, n, ws[d.name]["z"])
                self._bn_fwd(ws, d, n, gslot, relu=False)
                res = ws[d.name]["y"]
            self._bn_fwd(ws, b, n, gslot, res=res)
            x = ws[b.name]["y"]
        gp = self.grads.data_ptr() + 4 * base * self.P
        g = ws["g"]
        fw, fb = self.off_fc
        _native.check(L.bt_cnn_head(x.data_ptr(), ws["labels"].data_ptr(), self.params.data_ptr() + 4 * fw,
                                    self.params.data_ptr() + 4 * fb, n, B, gp + 4 * fw, gp + 4 * fb, self.P,
                                    losses[base:].data_ptr(), g[0].data_ptr(), s), "head")
        if capture is not None:
            capture.update(img=ws["img"].clone(), labels=ws["labels"].clone(),
                           **{f"{k}_{cv.name}": ws[cv.name][k].clone() for cv in self.convs[:4] + self.convs[-2:]
                              for k in ("z", "y", "mean", "rstd")}, top=x.clone(),
                           dtop=g[0][:x.numel()].clone())
        dy = g[0]  # gradient of the current block output
        for (a, b, d), xin in zip(reversed(self.blocks), reversed(ins)):
            out = ws[b.name]["y"]
            dzb, dya, dza, dxa = g[1], g[2], g[1], g[3]
            self._bn_bwd(ws, b, n, base, dy, out, dzb)
            self._conv_bwd(ws, b, n, base, ws[a.name]["y"], dzb, dya)
            self._bn_bwd(ws, a, n, base, dya, ws[a.name]["y"], dza)
            ca = self._conv_bwd(ws, a, n, base, xin, dza, dxa)
            if d is None:  # identity shortcut: dx = dxa + dy [out > 0]
                _native.check(L.bt_cnn_add(dxa.data_ptr(), dy.data_ptr(), out.data_ptr(), n * B * a.hin ** 2 * a.ci,
                                           dy.data_ptr(), s))
            else:  # stride-2 block: both gradients arrive as parity classes, interleaved by the add
                self._bn_bwd(ws, d, n, base, dy, out, g[2])
                cd = self._conv_bwd(ws, d, n, base, xin, g[2], g[1])
                if a.s == 2:
                    _native.check(L.bt_cnn_add_s2((C.c_void_p * 4)(*ca), (C.c_void_p * 4)(*cd), dy.data_ptr(), n * B,
                                                  a.hout, a.hout, a.ci, s), "stride-2 dX classes + shortcut")
                else:
                    _native.check(L.bt_cnn_add(dxa.data_ptr(), g[1].data_ptr(), None, n * B * a.hin ** 2 * a.ci,
                                               dy.data_ptr(), s))
        self._bn_bwd(ws, stem, n, base, dy, ws["stem"]["y"], g[1])
        self._conv_bwd(ws, stem, n, base, ws["img"], g[1], None)
        sl["cursor"].add_(1)  # every EST of the group consumed one micro-batch

    # ------------------------------------------------------------ step
    def step(self, capture: dict | None = None, check: bool = True) -> torch.Tensor:
        """One mini-batch of this process's ESTs on the current layout; per-EST losses [est_count].
        After one eager step on a layout, the whole step (every launch group, the reducer, the weight
        refresh, the cursor advance) is captured as a CUDA graph and replayed until the next rescale."""
        replay = self.graph and capture is None and self.peer is None
        if replay and self._gwarm:
            if self._graph is None:  # capture once per layout (the captured work runs at the first replay)
                self._graph = self._capture(self.G)
            g, gloss = self._graph
            g.replay()
            self._post(check)
            return gloss.clone()
        losses = torch.empty(self.En, dtype=torch.float32, device="cuda")
        self._body(losses, capture)
        self._post(check)
        self._gwarm = self._gwarm or replay
        return losses

    def _body(self, losses, capture=None):
        """Everything a step puts on the stream (capturable: no host synchronisation, no allocation)."""
        for g, (base, n) in enumerate(self.layout(self.G)):
            self._group(g, base, n, losses, capture if self.G == 1 else None)
        if capture is not None:
            capture["grads"] = self.grads.clone()
        if self.peer is not None:  # across processes: the peer-memory reducer
            self.peer.step()
        else:
            if self.En != self.E:
                raise ConfigError("a partial EST block needs attach_peer() for the exchange")
            a = _native.ReduceArgs()
            a.dtype, a.mode, a.E, a.fanin, a.n = _native.DTYPE_F32, _native.REDUCE_UPDATE, self.E, self.fanin, self.P
            for k in range(self.E):
                a.grads[k] = self.grads.data_ptr() + 4 * k * self.P
            p, v = self.params.data_ptr(), self.vel.data_ptr()
            a.param, a.vel, a.param_out, a.vel_out = p, v, p, v
            a.lr, a.mu, a.flags = self.lr, self.mu, self.flags.t.data_ptr()
            a.stage = self._stage().data_ptr()  # guarded: a non-finite step changes nothing (model.py:207-209)
            _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()), "resnet reduce_update")
        self._refresh_bf16()

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
            raise NumericError("resnet: non-finite synchronized gradient")

    def flops_per_step(self) -> float:
        """Convolution + head flops of one mini-batch (forward 2*R*Co*K, backward dX and dW 2x that)."""
        f = 0.0
        for cv in self.convs:
            f += 6.0 * self.En * self.B * cv.hout ** 2 * cv.co * (cv.taps * (3 if cv.name == "stem" else cv.ci))
        return f

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

    def run_log(self, steps: int, log=None, every: int = 1):
        """`steps` mini-batches recorded like the reference's run_training (scenarios.py:69-80): per step
        the per-EST losses (binary64 hex on disk) and, every `every` steps (sampled: the weights are
        hundreds of MB), the weight fingerprint; returns the RunLog (comparable with runlog.bitdiff)."""
        from .runlog import RunLog, RunRecord

        if log is None:
            log = RunLog(self.E, "d1", self.seed)
        for _ in range(steps):
            losses = self.step()
            n = self.step_idx
            h = self.fingerprint() if every and n % every == 0 else ""
            log.add(RunRecord(n, [float(x) for x in losses.tolist()], h))
        return log

    def attach_peer(self, group=None):
        """Multi-GPU (one process per GPU, torch.distributed initialised, rank r holding the r-th contiguous
        EST block): the exchange becomes paper_2208_14228_b200.peer.PeerGroupReducer over CUDA IPC (Tree(2):
        hierarchical partials + owner fold over NVLink; Sequential: owner reads all E slots in rank order)."""
        from .hier import RankBuffers
        from .peer import PeerGroupReducer

        loc = RankBuffers(self.grads, self.params, self.vel, torch.cuda.current_stream())
        self.peer = PeerGroupReducer(loc, self.E, "rank_tree2" if self.fanin == 2 else "sequential", None, self.lr,
                                     self.mu, group)
