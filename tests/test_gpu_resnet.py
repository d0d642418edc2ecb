"""Per-EST ResNet-18 step with BatchNorm and elastic rescale (C3, BASELINE.json configs[2]; needs a B200).

* Elastic rescale (the EasyScale S1/S2/S4 property, bit for bit): 16 ESTs trained on 8 "GPUs"
  (launch groups), rescaled to 4 and then 2 mid-training -- per-EST BatchNorm running statistics and
  sampler cursors moved by the slot-copy kernel -- give the same losses, weights, momentum and per-EST
  BN statistics as the uninterrupted 1-GPU run.
* Parity (no reference implementation exists for this model): the stem and first block
  stage by stage against float64 restatements fed with the captured bf16 inputs (conv: <= 1% of bf16
  outputs differ by one ulp; BN statistics and running statistics rel. error <= 1e-5); the whole
  network's per-EST loss against a float64 restatement with the same forward bf16 rounding points
  (rel. error <= 2e-3 after 20 layers of bf16 activations); the head and the last BasicBlock's
  backward stage by stage from the captured tensors (fc gradients <= 1e-4, BN dgamma/dbeta <= 1e-4,
  per-EST conv weight gradient rel. Frobenius error <= 5e-3).
"""

import ctypes as C

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

pytestmark = pytest.mark.gpu

SMALL = dict(ests=16, batch=4, seed=7, lr=0.05, momentum=0.9)
BENCHED = dict(ests=2, batch=32, seed=7, lr=0.05, momentum=0.9)  # the benched per-EST shape (C3: 32 images)


@pytest.fixture(scope="module")
def rn():
    assert torch.cuda.is_available()
    from paper_2208_14228_b200 import resnet as mod

    return mod


def _bits(t):
    return t.detach().contiguous().view(torch.int32).cpu().numpy()


def test_rescale_8_4_2_matches_uninterrupted_run(rn):
    a = rn.ResNetJob(gpus=8, **SMALL)
    b = rn.ResNetJob(gpus=1, **SMALL)
    la, lb = [], []
    for gpus in (8, 4, 2):
        if gpus != 8:
            a.rescale(gpus)
        for _ in range(2):
            la.append(a.step().clone())
            lb.append(b.step().clone())
    for x, y in zip(la, lb):
        assert np.array_equal(_bits(x), _bits(y))
    assert np.array_equal(_bits(a.params), _bits(b.params))
    assert np.array_equal(_bits(a.vel), _bits(b.vel))
    sa, sb = a.est_state(), b.est_state()
    for k in ("run_mean", "run_var"):
        assert np.array_equal(_bits(sa[k]), _bits(sb[k])), k
    assert torch.equal(sa["cursor"], sb["cursor"]) and int(sa["cursor"][0]) == 6
    assert a.G == 2 and len(a.slots) == 2


def test_uneven_layout_and_tree_reducer(rn):
    a = rn.ResNetJob(gpus=3, fanin=2, **SMALL)  # 6 + 5 + 5 ESTs
    b = rn.ResNetJob(gpus=1, fanin=2, **SMALL)
    for _ in range(2):
        assert np.array_equal(_bits(a.step()), _bits(b.step()))
    assert np.array_equal(_bits(a.params), _bits(b.params))


def test_same_batch_loss_decreases(rn):
    job = rn.ResNetJob(gpus=1, **dict(SMALL, lr=0.05))
    first = job.step().mean().item()
    for _ in range(3):
        job.slots[0]["cursor"].zero_()  # replay micro-batch 0 of every EST
        last = job.step().mean().item()
    assert last < first, (first, last)


def _d(t):
    return t.detach().double().cpu()


def _bf(x):
    return x.to(torch.bfloat16).double()


def _close_bf16(got, want, what, frac=1e-2, rel=5e-3):
    got, want = _d(got), want.double()
    mism = (got != _bf(want)).double().mean().item()
    err = ((got - want).norm() / (want.norm() + 1e-30)).item()
    assert mism <= frac and err <= rel, (what, mism, err)


def _close(got, want, what, rel):
    got, want = _d(got), want.double()
    err = ((got - want).norm() / (want.norm() + 1e-30)).item()
    assert err <= rel, (what, err)


def _conv_w(job, cv, p):
    w0 = job.off[cv.name][0]
    return _d(p[w0:w0 + cv.co * cv.K]).view(cv.co, cv.k, cv.k, cv.ci).permute(0, 3, 1, 2)  # OIHW


def _nchw(t, n, h, c):
    return _d(t).view(n, h, h, c).permute(0, 3, 1, 2)


@pytest.mark.parametrize("cfg", [SMALL, BENCHED], ids=["batch4", "batch32"])
def test_stem_and_block_stages_match_float64(rn, cfg):
    job = rn.ResNetJob(gpus=1, **cfg)
    P0 = job.params.clone()
    cap = {}
    job.step(capture=cap)
    E, B, eps = job.E, job.B, job.eps
    N = E * B
    stem = job.convs[0]
    x = _nchw(cap["img"], N, 32, 8)
    assert bool((x[:, 3:] == 0).all()) and float(x[:, :3].abs().max()) <= 1.0
    z_ref = Fn.conv2d(x, _bf(_conv_w(job, stem, P0)), padding=1)
    z = _nchw(cap["z_stem"], N, 32, 64)
    _close_bf16(z, z_ref, "stem conv")
    # per-EST batch statistics over the EST's own B x 32 x 32 pixels
    zc = z.view(E, B, 64, 1024).permute(0, 2, 1, 3).reshape(E, 64, -1)
    mean, var = zc.mean(-1), zc.var(-1, unbiased=False)
    _close(cap["mean_stem"].view(E, 64), mean, "bn mean", 1e-5)
    _close(cap["rstd_stem"].view(E, 64), 1 / torch.sqrt(var + eps), "bn rstd", 1e-5)
    g0, b0 = job.off["stem"][1:]
    gam, bet = _d(P0[g0:g0 + 64]), _d(P0[b0:b0 + 64])
    y_ref = torch.relu(gam.view(1, 64, 1, 1) * (z - mean.repeat_interleave(B, 0).view(N, 64, 1, 1))
                       * (1 / torch.sqrt(var + eps)).repeat_interleave(B, 0).view(N, 64, 1, 1) + bet.view(1, 64, 1, 1))
    _close_bf16(_nchw(cap["y_stem"], N, 32, 64), y_ref, "bn + relu")
    st = job.est_state()
    R = B * 1024
    _close(st["run_mean"][:, :64], 0.1 * mean, "running mean", 1e-5)
    _close(st["run_var"][:, :64], 0.9 + 0.1 * var * R / (R - 1), "running var", 1e-5)
    a = job.convs[1]
    za_ref = Fn.conv2d(_nchw(cap["y_stem"], N, 32, 64), _bf(_conv_w(job, a, P0)), padding=1)
    _close_bf16(_nchw(cap[f"z_{a.name}"], N, 32, 64), za_ref, "block conv a")


def _restate_loss(job, P, img, labels):
    """float64 ResNet-18 with the kernels' forward bf16 rounding points; per-EST BatchNorm statistics."""
    E, B, eps = job.E, job.B, job.eps
    N = E * B

    def bn(z, cv, relu=True, res=None):
        g0, b0 = job.off[cv.name][1:]
        zz = z.view(E, B, cv.co, -1).transpose(1, 2).reshape(E, cv.co, -1)
        m = zz.mean(-1).repeat_interleave(B, 0).view(N, cv.co, 1, 1)
        v = zz.var(-1, unbiased=False).repeat_interleave(B, 0).view(N, cv.co, 1, 1)
        y = P[g0:g0 + cv.co].view(1, -1, 1, 1) * (z - m) / torch.sqrt(v + eps) + P[b0:b0 + cv.co].view(1, -1, 1, 1)
        if res is not None:
            y = y + res
        return _bf(torch.relu(y) if relu else y)

    def conv(x, cv):
        w0 = job.off[cv.name][0]
        w = P[w0:w0 + cv.co * cv.K].view(cv.co, cv.k, cv.k, cv.ci).permute(0, 3, 1, 2)
        return _bf(Fn.conv2d(x, _bf(w), stride=cv.s, padding=cv.p))

    x = bn(conv(img, job.convs[0]), job.convs[0])
    for a, b, d in job.blocks:
        h = bn(conv(x, a), a)
        res = x if d is None else bn(conv(x, d), d, relu=False)
        x = bn(conv(h, b), b, res=res)
    pooled = x.mean((2, 3))
    fw, fb = job.off_fc
    logits = pooled @ P[fw:fw + 5120].view(10, 512).T + P[fb:fb + 10]
    ce = Fn.cross_entropy(logits, labels, reduction="none")
    return ce.view(E, B).mean(1)


@pytest.mark.parametrize("cfg", [SMALL, BENCHED], ids=["batch4", "batch32"])
def test_loss_and_last_block_gradients_match_float64(rn, cfg):
    """Whole-network loss vs the float64 restatement; the head and the last BasicBlock's backward
    (ReLU mask, BatchNorm backward with per-EST statistics, per-EST conv weight gradient) stage by
    stage from the captured bf16 tensors."""
    job = rn.ResNetJob(gpus=1, **cfg)
    P0 = job.params.clone()
    cap = {}
    losses = job.step(capture=cap)
    E, B, eps = job.E, job.B, job.eps
    N = E * B
    img = _nchw(cap["img"], N, 32, 8)
    labels = cap["labels"].long().cpu()
    assert int(labels.min()) >= 0 and int(labels.max()) <= 9
    with torch.no_grad():
        ref = _restate_loss(job, _d(P0), img, labels)
    _close(losses, ref, "per-EST loss (20 layers of bf16 activations)", 2e-3)
    g = cap["grads"].double().cpu()
    # head: avgpool + fc + CE from the captured block output
    top = _d(cap["top"]).view(N, 16, 512)
    pooled = top.mean(1).requires_grad_(True)
    fw, fb = job.off_fc
    W = _d(P0[fw:fw + 5120]).view(10, 512).requires_grad_(True)
    bvec = _d(P0[fb:fb + 10]).requires_grad_(True)
    ce = Fn.cross_entropy(pooled @ W.T + bvec, labels, reduction="none").view(E, B).mean(1)
    _close(losses, ce.detach(), "head loss", 1e-5)
    for e in (0, E - 1):
        gw, gb, gp = torch.autograd.grad(ce[e], (W, bvec, pooled), retain_graph=True)
        _close(g[e, fw:fw + 5120], gw.reshape(-1), f"fc grad est {e}", 1e-4)
        _close(g[e, fb:fb + 10], gb, f"fc bias grad est {e}", 1e-4)
    (gpool,) = torch.autograd.grad(ce.sum(), pooled)
    dtop = _d(cap["dtop"]).view(N, 16, 512)
    _close_bf16(dtop, (gpool / 16).unsqueeze(1).expand(N, 16, 512), "head dx")
    # last block, conv b: g = dtop [out > 0]; BN backward with the EST's own statistics; dW_e
    a, b = job.convs[-2], job.convs[-1]
    z = _d(cap[f"z_{b.name}"]).view(E, B * 16, 512)
    mean, rstd = _d(cap[f"mean_{b.name}"]).view(E, 1, 512), _d(cap[f"rstd_{b.name}"]).view(E, 1, 512)
    gmask = (dtop * (top > 0)).view(E, B * 16, 512)
    xh = (z - mean) * rstd
    gam = _d(P0[job.off[b.name][1]:job.off[b.name][1] + 512])
    R = B * 16
    dz = gam * rstd * (gmask - gmask.sum(1, keepdim=True) / R - xh * (gmask * xh).sum(1, keepdim=True) / R)
    ya = _d(cap[f"y_{a.name}"]).view(N, 4, 4, 512).permute(0, 3, 1, 2)
    col = Fn.unfold(ya, 3, padding=1).view(E, B, 512, 9, 16)  # (ci, tap) x position
    col = col.permute(0, 1, 4, 3, 2).reshape(E, R, 9 * 512)     # rows (n, pos), columns (tap, ci)
    dzb = _bf(dz)
    lo, g0, b0 = job.off[b.name]
    for e in (0, E - 1):
        _close(g[e, b0:b0 + 512], gmask[e].sum(0), f"dbeta est {e}", 1e-5)
        _close(g[e, g0:g0 + 512], (gmask[e] * xh[e]).sum(0), f"dgamma est {e}", 1e-4)
        _close(g[e, lo:g0], (dzb[e].T @ col[e]).reshape(-1), f"conv dW est {e}", 5e-3)


def test_implicit_gemm_convolutions_equal_explicit_im2col(rn, monkeypatch):
    """TMA im2col-mode convolutions (bt_gemm_conv: forward, weight gradient, stride-1 dX) load the same
    tiles in the same K order as the explicit im2col + GEMM path: identical bits over several steps."""
    a = rn.ResNetJob(gpus=2, **SMALL)
    la = [a.step().clone() for _ in range(2)]
    monkeypatch.setenv("BT_CONV_EXPLICIT", "1")
    b = rn.ResNetJob(gpus=2, **SMALL)
    lb = [b.step().clone() for _ in range(2)]
    monkeypatch.delenv("BT_CONV_EXPLICIT")
    for x, y in zip(la, lb):
        assert np.array_equal(_bits(x), _bits(y))
    assert np.array_equal(_bits(a.params), _bits(b.params))


@pytest.mark.parametrize("ci,co,k,s,hw", [(64, 64, 3, 1, 8), (64, 128, 3, 2, 8), (128, 256, 1, 2, 8), (64, 64, 3, 1, 32), (256, 256, 3, 1, 8)])
def test_convolution_products_match_float64(rn, ci, co, k, s, hw):
    """The implicit-GEMM convolution (bt_gemm_conv: TMA im2col loads), its weight gradient and the dX
    paths (stride 1: forward convolution of dz with the tap-reversed filter; stride 2: the transposed
    gather, and the zero insertion of dz convolved at stride 1) against torch's float64 conv2d / conv2d_weight / conv2d_input on the same bf16 values:
    fp32-accumulation error only (rel. Frobenius <= 1e-5 for fp32 outputs, bf16 rounding for bf16)."""
    from torch.nn.grad import conv2d_input, conv2d_weight

    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    L = _native.lib()
    N, p = 4, k // 2
    ho = (hw + 2 * p - k) // s + 1
    g = torch.Generator(device="cuda").manual_seed(ci + co + k)
    x = torch.randn(N, hw, hw, ci, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(co, k, k, ci, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    dz = torch.randn(N, ho, ho, co, device="cuda", generator=g).to(torch.bfloat16)
    wt = w.permute(3, 1, 2, 0).contiguous()  # [Ci][kh][kw][Co]
    x64, w64, dz64 = (t.double().cpu() for t in (x.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), dz.permute(0, 3, 1, 2)))
    # forward (fp32 out)
    z = torch.empty(N * ho * ho, co, device="cuda")
    _native.check(L.bt_gemm_conv(0, x.data_ptr(), N, hw, hw, ci, ho, ho, k, k, s, p, w.data_ptr(), z.data_ptr(), co,
                                 1, 0, 0, 0, stream()))
    zref = torch.nn.functional.conv2d(x64, w64, stride=s, padding=p).permute(0, 2, 3, 1).reshape(-1, co)
    _close(z, zref, "conv forward", 1e-5)
    # weight gradient, one batch entry per 2 images (an "EST"), fp32 out
    R = 2 * ho * ho
    if R % 64 == 0:
        dw = torch.empty(2, co, k * k * ci, device="cuda")
        _native.check(L.bt_gemm_conv(1, x.data_ptr(), N, hw, hw, ci, ho, ho, k, k, s, p, dz.data_ptr(), dw.data_ptr(),
                                     co, 2, R, co * k * k * ci, 0, stream()))
        for e in range(2):
            sl = slice(2 * e, 2 * e + 2)
            ref = conv2d_weight(x64[sl], w64.shape, dz64[sl], stride=s, padding=p).permute(0, 2, 3, 1).reshape(co, -1)
            _close(dw[e], ref, f"conv dW entry {e}", 1e-5)
    # dX
    dxref = conv2d_input(x64.shape, w64, dz64, stride=s, padding=p).permute(0, 2, 3, 1).reshape(-1, ci)
    dx = torch.empty(N * hw * hw, ci, device="cuda")
    if s == 1:  # forward convolution of dz with the tap-reversed filter
        wflip = torch.flip(w.view(co, k, k, ci), dims=(1, 2)).permute(3, 1, 2, 0).contiguous()
        _native.check(L.bt_gemm_conv(0, dz.data_ptr(), N, ho, ho, co, hw, hw, k, k, 1, p, wflip.data_ptr(),
                                     dx.data_ptr(), ci, 1, 0, 0, 0, stream()))
    else:  # transposed-convolution gather + GEMM
        col = torch.empty(N * hw * hw, k * k * co, dtype=torch.bfloat16, device="cuda")
        _native.check(L.bt_cnn_im2col(dz.data_ptr(), col.data_ptr(), N, ho, ho, co, hw, hw, k, k, s, p, 1, stream()))
        _native.check(L.bt_gemm_bf16_ex(col.data_ptr(), wt.data_ptr(), dx.data_ptr(), 1, N * hw * hw, ci, k * k * co,
                                        0, 0, 0, 0, None, 0, 0, stream()))
    _close(dx, dxref, "conv dX", 1e-5)
    if s != 1:  # the step's path: four output parity classes, each a stride-1 convolution of dz
        wf = w.float().reshape(co, k * k, ci).contiguous()  # master layout [Co][taps][Ci]
        cls, outs = [], []
        for a in (0, 1):
            for b in (0, 1):
                th = sorted((t for t in range(k) if (a + p - t) % 2 == 0), key=lambda t: -t)
                tw = sorted((t for t in range(k) if (b + p - t) % 2 == 0), key=lambda t: -t)
                if not th or not tw:
                    cls.append(None)
                    continue
                src = [u * k + v for u in th for v in tw]
                wc = torch.empty(ci, len(src), co, dtype=torch.bfloat16, device="cuda")
                tm = (C.c_int32 * 9)(*(src + [0] * (9 - len(src))))
                _native.check(L.bt_cnn_filter_taps((C.c_void_p * 1)(wf.data_ptr()), (C.c_void_p * 1)(wc.data_ptr()),
                                                   (C.c_int32 * 1)(co), (C.c_int32 * 1)(k * k), (C.c_int32 * 1)(ci),
                                                   (C.c_int32 * 1)(len(src)), tm, 1, stream()))
                ref = w.view(co, k * k, ci)[:, src, :].permute(2, 1, 0)
                torch.cuda.synchronize()
                assert torch.equal(wc, ref)
                o = torch.empty(N, ho, ho, ci, dtype=torch.bfloat16, device="cuda")
                _native.check(L.bt_gemm_conv(0, dz.data_ptr(), N, ho, ho, co, ho, ho, len(th), len(tw), 1, 0,
                                             wc.data_ptr(), o.data_ptr(), ci, 1, 0, 0, 1, stream()))
                outs.append(o)
                cls.append(o.data_ptr())
        dxc = torch.empty(N, hw, hw, ci, dtype=torch.bfloat16, device="cuda")
        _native.check(L.bt_cnn_add_s2((C.c_void_p * 4)(*cls), None, dxc.data_ptr(), N, ho, ho, ci, stream()))
        _close_bf16(dxc.reshape(-1, ci), dxref, "conv dX (parity classes)")
    if s != 1:  # the zero-insertion alternative: a stride-1 implicit convolution of the zero-inserted dz
        up = torch.empty(N, hw, hw, co, dtype=torch.bfloat16, device="cuda")
        _native.check(L.bt_cnn_upsample(dz.data_ptr(), N, ho, ho, co, s, up.data_ptr(), stream()))
        upref = torch.zeros_like(up)
        upref[:, ::s, ::s, :] = dz
        assert torch.equal(up, upref)
        wflip = torch.flip(w.view(co, k, k, ci), dims=(1, 2)).permute(3, 1, 2, 0).contiguous()
        dx2 = torch.empty(N * hw * hw, ci, device="cuda")
        _native.check(L.bt_gemm_conv(0, up.data_ptr(), N, hw, hw, co, hw, hw, k, k, 1, k - 1 - p, wflip.data_ptr(),
                                     dx2.data_ptr(), ci, 1, 0, 0, 0, stream()))
        _close(dx2, dxref, "conv dX (zero insertion)", 1e-5)


@pytest.mark.parametrize("co,hw,out_bf16", [(64, 32, 1), (64, 32, 0), (32, 16, 1), (64, 16, 0)])
def test_halo_convolution_equals_im2col_path(co, hw, out_bf16, monkeypatch):
    """The halo form (three row-halo boxes per tile, the kh taps as views) issues the im2col path's
    UMMAs on the same rows: identical bits, bf16 and fp32 outputs, Co = 64 and Co < 64."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    L = _native.lib()
    N = 6
    g = torch.Generator(device="cuda").manual_seed(co + hw)
    x = torch.randn(N, hw, hw, 64, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(co, 9 * 64, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    dt = torch.bfloat16 if out_bf16 else torch.float32
    outs = []
    for halo in (True, False):
        if halo:
            monkeypatch.delenv("BT_CONV_HALO0", raising=False)
        else:
            monkeypatch.setenv("BT_CONV_HALO0", "1")
        z = torch.full((N * hw * hw, co), float("nan"), device="cuda", dtype=dt)
        _native.check(L.bt_gemm_conv(0, x.data_ptr(), N, hw, hw, 64, hw, hw, 3, 3, 1, 1, w.data_ptr(), z.data_ptr(),
                                     co, 1, 0, 0, out_bf16, stream()))
        outs.append(z)
    torch.cuda.synchronize()
    assert not torch.isnan(outs[0]).any()
    assert torch.equal(outs[0].view(torch.int16 if out_bf16 else torch.int32),
                       outs[1].view(torch.int16 if out_bf16 else torch.int32))


@pytest.mark.parametrize("ci,co,k,s", [(256, 256, 3, 1), (256, 512, 3, 2), (128, 256, 1, 2)])
def test_weight_gradient_pair_tiles_equal_single_cta(ci, co, k, s, monkeypatch):
    """The weight gradient on 256 x 256 CTA-pair tiles (im2col B halves loaded by each CTA of the pair)
    equals the 1-CTA form bit for bit (same per-element K order); shapes that do not tile fall back."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    L = _native.lib()
    N, hw, p = 8, 8, k // 2
    ho = (hw + 2 * p - k) // s + 1
    g = torch.Generator(device="cuda").manual_seed(ci + co)
    x = torch.randn(N, hw, hw, ci, device="cuda", generator=g).to(torch.bfloat16)
    dz = torch.randn(N, ho, ho, co, device="cuda", generator=g).to(torch.bfloat16)
    R = 4 * ho * ho
    if R % 64:
        pytest.skip("rows per entry not a multiple of 64")
    outs = []
    for pair in (True, False):
        if pair:
            monkeypatch.delenv("BT_CONV_WG_PAIR0", raising=False)
        else:
            monkeypatch.setenv("BT_CONV_WG_PAIR0", "1")
        dw = torch.full((2, co, k * k * ci), float("nan"), device="cuda")
        _native.check(L.bt_gemm_conv(1, x.data_ptr(), N, hw, hw, ci, ho, ho, k, k, s, p, dz.data_ptr(), dw.data_ptr(),
                                     co, 2, R, co * k * k * ci, 0, stream()))
        outs.append(dw)
    torch.cuda.synchronize()
    assert not torch.isnan(outs[0]).any()
    assert torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))


@pytest.mark.parametrize("ci,co,k,s,out_bf16", [(256, 256, 3, 1, 1), (128, 256, 3, 2, 0), (512, 512, 3, 1, 1)])
def test_forward_convolution_pair_tiles_equal_single_cta(ci, co, k, s, out_bf16, monkeypatch):
    """The forward implicit convolution on CTA-pair tiles (each CTA loads its 128 pixels' im2col boxes and
    its half of the filter rows) equals the 1-CTA form bit for bit."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    L = _native.lib()
    N, hw, p = 16, 8, k // 2
    ho = (hw + 2 * p - k) // s + 1
    g = torch.Generator(device="cuda").manual_seed(ci + co + s)
    x = torch.randn(N, hw, hw, ci, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(co, k * k * ci, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    dt = torch.bfloat16 if out_bf16 else torch.float32
    outs = []
    for pair in (True, False):
        if pair:
            monkeypatch.delenv("BT_CONV_FWD_PAIR0", raising=False)
        else:
            monkeypatch.setenv("BT_CONV_FWD_PAIR0", "1")
        z = torch.full((N * ho * ho, co), float("nan"), device="cuda", dtype=dt)
        _native.check(L.bt_gemm_conv(0, x.data_ptr(), N, hw, hw, ci, ho, ho, k, k, s, p, w.data_ptr(), z.data_ptr(),
                                     co, 1, 0, 0, out_bf16, stream()))
        outs.append(z)
    torch.cuda.synchronize()
    assert not torch.isnan(outs[0]).any()
    iv = torch.int16 if out_bf16 else torch.int32
    assert torch.equal(outs[0].view(iv), outs[1].view(iv))


def test_cuda_graph_replay_equals_eager_across_rescale(rn):
    """The captured ResNet step replays bit-identically to eager execution, and a rescale (new slot
    buffers and launch groups) re-captures: graph runs through 4 -> 2 GPUs equal the eager run."""
    a = rn.ResNetJob(gpus=4, graph=True, **SMALL)
    b = rn.ResNetJob(gpus=4, graph=False, **SMALL)
    for gpus in (4, 2):
        if gpus != 4:
            a.rescale(gpus)
            b.rescale(gpus)
        for _ in range(3):
            assert np.array_equal(_bits(a.step()), _bits(b.step()))
    assert a._graph is not None and np.array_equal(_bits(a.params), _bits(b.params))
    sa, sb = a.est_state(), b.est_state()
    assert np.array_equal(_bits(sa["run_var"]), _bits(sb["run_var"])) and torch.equal(sa["cursor"], sb["cursor"])


def test_run_log_across_rescale(rn):
    """C3's run log (per-EST losses + weight fingerprint every step) is identical for 8 -> 4 -> 2 launch
    groups with the EST context switches and for the uninterrupted single group (runlog.bitdiff)."""
    from paper_2208_14228_b200.runlog import bitdiff

    a = rn.ResNetJob(gpus=8, **SMALL)
    b = rn.ResNetJob(gpus=1, **SMALL)
    la = a.run_log(2)
    a.rescale(4)
    a.run_log(2, la)
    a.rescale(2)
    a.run_log(2, la)
    lb = b.run_log(6)
    assert bitdiff(la, lb) is None and len(la.records) == 6 and all(r.param_hash for r in la.records)


def test_prepared_rescale_replays_staged_graphs_and_reenters_layouts(rn):
    """ResNetJob.prepare stages a layout's slot buffers, copy plans and step graph (captured, not run --
    the training state does not move); the rescale is then one slot-copy launch and the next step a
    replay.  8 -> 4 -> 2 -> 8 -> 4 with staged graphs (the last two re-enter cached layouts) equals the
    uninterrupted run bit for bit: weights, momentum, per-EST BN statistics and cursors."""
    a = rn.ResNetJob(gpus=8, **SMALL)
    b = rn.ResNetJob(gpus=1, **SMALL)
    p0 = a.params.clone()
    for g in (4, 2):
        a.prepare(g)
    assert torch.equal(a.params, p0) and set(a._graphs) == {4, 2}
    la, lb = [], []
    for gpus in (8, 4, 2, 8, 4):
        if gpus != a.G:
            a.rescale(gpus)
            assert a.G == gpus and (gpus == 8 or a._graph is a._graphs[gpus])
        for _ in range(2):
            la.append(a.step().clone())
            lb.append(b.step().clone())
    for x, y in zip(la, lb):
        assert np.array_equal(_bits(x), _bits(y))
    assert np.array_equal(_bits(a.params), _bits(b.params)) and np.array_equal(_bits(a.vel), _bits(b.vel))
    sa, sb = a.est_state(), b.est_state()
    for k in ("run_mean", "run_var"):
        assert np.array_equal(_bits(sa[k]), _bits(sb[k])), k
    assert torch.equal(sa["cursor"], sb["cursor"]) and int(sa["cursor"][0]) == 10


@pytest.mark.parametrize("n_img,rpb,hw,ci,co", [(4, 2048, 32, 64, 64), (2, 1024, 32, 64, 64), (3, 1024, 32, 64, 64),
                                               (8, 512, 16, 128, 128), (6, 256, 16, 128, 128), (4, 512, 16, 64, 128),
                                               (2, 1024, 32, 128, 64)])
def test_weight_gradient_halo_equals_im2col_path(n_img, rpb, hw, ci, co, monkeypatch):
    """The 3x3 / stride-1 weight gradient in halo form (per (split, kw, 64-channel block): a {64 ch, W px,
    64/W + 2 rows} box whose three kh views, W rows apart, are ONE N = 192 MN-major operand) issues the
    im2col form's products in the same K order per output element: identical fp32 bits at W = 32 / 16,
    64 / 128 channels in and out, including splits that straddle images."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    L = _native.lib()
    H = W = hw
    g = torch.Generator(device="cuda").manual_seed(n_img * 7 + rpb + ci + co)
    x = torch.randn(n_img, H, W, ci, device="cuda", generator=g).to(torch.bfloat16)
    dz = (torch.randn(n_img * H * W, co, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    batch = n_img * H * W // rpb
    K = 9 * ci
    outs = []
    for halo in (True, False):
        if halo:
            monkeypatch.delenv("BT_CONV_WG_HALO0", raising=False)
        else:
            monkeypatch.setenv("BT_CONV_WG_HALO0", "1")
        c = torch.full((batch, co, K), float("nan"), device="cuda")
        _native.check(L.bt_gemm_conv(1, x.data_ptr(), n_img, H, W, ci, H, W, 3, 3, 1, 1, dz.data_ptr(), c.data_ptr(),
                                     co, batch, rpb, co * K, 0, stream()))
        outs.append(c)
    torch.cuda.synchronize()
    assert not torch.isnan(outs[0]).any()
    ref = torch.einsum("bpo,bpk->bok", dz.float().view(batch, rpb, co),
                       torch.stack([Fn.pad(x.float(), (0, 0, 1, 1, 1, 1))[:, kh:kh + H, kw:kw + W, :]
                                    for kh in range(3) for kw in range(3)], 3).view(batch, rpb, K))
    assert ((outs[0] - ref).norm() / ref.norm()).item() < 1e-5
    assert torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))
