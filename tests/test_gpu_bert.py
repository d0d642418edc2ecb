"""Per-EST BERT encoder step (C4, BASELINE.json configs[3]; needs a B200).

* Mapping invariance (the EasyScale property, bit for bit): the same E ESTs
  grouped into launches in different ways -- what mapping them onto 1/2/4/8
  GPUs does -- give identical losses and weights after several steps.
* Parity (there is no reference implementation of this model):
  every stage of layer 0's forward and backward, the loss, and every per-EST
  gradient against a float64 restatement fed with the captured bf16 inputs of
  that stage, with the same bf16 rounding points and the same counter-keyed
  dropout masks (regenerated here from splitmix64).  Tolerances, stated:
  fp32 outputs rel. Frobenius error <= 1e-4 (2e-3 where a bf16 GEMM output
  feeds them: a rounding flip there moves one input by one bf16 ulp); bf16 outputs: <= 1% of elements
  differ (one bf16 ulp, fp32-vs-fp64 accumulation) and rel. error <= 5e-3;
  per-EST gradients rel. Frobenius error <= 5e-3.
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

C_GELU = math.sqrt(2 / math.pi)


def _gelu(x):
    """GELU, tanh form (the original BERT code's activation)"""
    return 0.5 * x * (1 + torch.tanh(C_GELU * (x + 0.044715 * x ** 3)))


def _gelu_grad(x):
    t = torch.tanh(C_GELU * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * C_GELU * (1 + 3 * 0.044715 * x * x)

SMALL = dict(ests=4, seqs=2, layers=2, d_model=256, heads=4, d_ff=512, seed=3, lr=0.01, momentum=0.9,
             p_hidden=0.1, p_attn=0.1, vocab=1000)
# the benched C4 shapes (BERT-base: d 768, 12 heads, FFN 3072, seq 128): the CTA-pair GEMM with the
# 16-warp GELU epilogue at N = 3072 / K = 768, LayerNorm at D = 768, tcgen05 attention at 12 heads
BASE = dict(ests=2, seqs=2, layers=2, d_model=768, heads=12, d_ff=3072, seed=3, lr=0.01, momentum=0.9,
            p_hidden=0.1, p_attn=0.1)

GAMMA = np.uint64(0x9E3779B97F4A7C15)
TAG_HDROP = 0x4245_5254_4844_5250
TAG_ADROP = 0x4245_5254_4144_5250


def _mix64(x):
    x = x ^ (x >> np.uint64(30))
    x = x * np.uint64(0xBF58476D1CE4E5B9)
    x = x ^ (x >> np.uint64(27))
    x = x * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _draws(s0, n):
    with np.errstate(over="ignore"):
        return _mix64(np.uint64(s0) + (n.astype(np.uint64) + np.uint64(1)) * GAMMA)


def _keep(raw_quads, j, p):
    """scale per unit from the quad draw: unit j uses the 16-bit field j % 4 (bits [16 (j % 4), +16))"""
    field = (raw_quads >> (np.uint64(16) * (j % 4).astype(np.uint64))) & np.uint64(0xFFFF)
    thr = np.uint64(math.ceil(p * 2 ** 16))
    return np.where(field < thr, 0.0, 1.0 / (1.0 - p))


@pytest.fixture(scope="module")
def bert():
    assert torch.cuda.is_available()
    from paper_2208_14228_b200 import bert as mod

    return mod


def _bits(t):
    return t.detach().contiguous().view(torch.int32).cpu().numpy()


def test_groupings_are_bitwise_identical(bert):
    runs = {}
    for groups in ([4], [2, 2], [1, 1, 1, 1], [1, 3]):
        job = bert.BertJob(**SMALL)
        losses = [job.step(groups).clone() for _ in range(3)]
        runs[tuple(groups)] = (losses, job.params.clone(), job.vel.clone())
    ref_l, ref_p, ref_v = runs[(4,)]
    for key, (losses, params, vel) in runs.items():
        for a, b in zip(losses, ref_l):
            assert np.array_equal(_bits(a), _bits(b)), key
        assert np.array_equal(_bits(params), _bits(ref_p)), key
        assert np.array_equal(_bits(vel), _bits(ref_v)), key


def test_tree_reducer_groupings_and_repeat(bert):
    a, b = bert.BertJob(fanin=2, **SMALL), bert.BertJob(fanin=2, **SMALL)
    for _ in range(2):
        assert np.array_equal(_bits(a.step([2, 2])), _bits(b.step()))
    assert np.array_equal(_bits(a.params), _bits(b.params))


def test_losses_decrease(bert):
    # (the regression head: the masked-LM targets are fresh uniform token ids every step -- nothing to learn)
    job = bert.BertJob(**dict(SMALL, lr=0.05, p_hidden=0.0, p_attn=0.0, head="mse"))
    first = job.step().mean().item()
    for _ in range(8):
        last = job.step().mean().item()
    assert last < first


def _d(t):
    return t.detach().double().cpu()


def _bf(x):
    return x.to(torch.bfloat16).double()


def _close_bf16(got, want, what, frac=1e-2, rel=5e-3):
    got, want = _d(got), want.double()
    assert got.shape == want.shape, what
    mism = (got != _bf(want)).double().mean().item()
    err = ((got - want).norm() / (want.norm() + 1e-30)).item()
    assert mism <= frac and err <= rel, (what, mism, err)


def _close(got, want, what, rel=1e-4):
    got, want = _d(got), want.double()
    err = ((got - want).norm() / (want.norm() + 1e-30)).item()
    assert err <= rel, (what, err)


def _ln(x, g, b, eps):
    mean = x.mean(-1, keepdim=True)
    var = ((x - mean) ** 2).mean(-1, keepdim=True)
    rstd = 1 / torch.sqrt(var + eps)
    return (x - mean) * rstd * g + b, mean.squeeze(-1), rstd.squeeze(-1)


def _ln_bwd(dy, x, g, eps):
    mean = x.mean(-1, keepdim=True)
    rstd = 1 / torch.sqrt(((x - mean) ** 2).mean(-1, keepdim=True) + eps)
    xh = (x - mean) * rstd
    gg = dy * g
    return (gg - gg.mean(-1, keepdim=True) - xh * (gg * xh).mean(-1, keepdim=True)) * rstd, xh


@pytest.mark.parametrize("cfg", [SMALL, BASE], ids=["small", "bert_base_dims"])
def test_layer0_stages_match_float64_restatement(bert, cfg):
    from paper_2208_14228_b200._native import host_derive_stream

    job = bert.BertJob(**dict(cfg, head="mse"))  # the encoder on synthetic embedded inputs (MLM head: below)
    P0 = job.params.clone()
    cap = {}
    losses = job.step(capture=cap)
    E, Te, D, H, F, NL = job.E, job.Te, job.D, job.H, job.F, job.L
    S, seed, step, ph, pa, eps = job.S, job.seed, 0, job.ph, job.pa, job.eps
    T = E * Te
    W = {k: _d(job.view(0, k, P0)) for k in bert._LAYER}

    def hidden_scale(site, l=0):
        sc = np.empty((T, D))
        for e in range(E):
            s0 = host_derive_stream(TAG_HDROP, seed, e)
            tl = np.arange(Te)[:, None]
            j = np.arange(D)[None, :]
            n0 = ((((step * NL + l) * 2 + site) * Te + tl) * D + j) >> 2
            sc[e * Te:(e + 1) * Te] = _keep(_draws(s0, n0), j, ph)
        return torch.from_numpy(sc)

    def attn_scale(l=0):
        """one draw per (16-row block, row g < 8, column pair): four 16-bit fields, field
        ((i >> 3) & 1) * 2 + (j & 1) decides (i, j); dropped iff field < ceil(p * 2^16)"""
        sc = np.empty((E, S, H, 128, 128))
        i = np.arange(128)[:, None]
        j = np.arange(128)[None, :]
        cnt = ((i >> 4) * 8 + (i & 7)) * 64 + (j >> 1)
        field = ((i >> 3) & 1) * 2 + (j & 1)
        thr = np.uint64(math.ceil(pa * 65536))
        for e in range(E):
            s0 = host_derive_stream(TAG_ADROP, seed, e)
            for sl in range(S):
                for h in range(H):
                    nb = ((((step * NL + l) * S + sl) * H + h) * 4096)
                    raw = _draws(s0, nb + cnt)
                    f = (raw >> (np.uint64(16) * field.astype(np.uint64))) & np.uint64(0xFFFF)
                    sc[e, sl, h] = np.where(f < thr, 0.0, 1.0 / (1.0 - pa))
        return torch.from_numpy(sc).view(E * S, H, 128, 128)

    # ---- forward, layer 0
    xb, x32 = _d(cap["xb"]), _d(cap["x32"])
    assert torch.equal(xb, x32)  # the synthetic input is bf16-exact
    qkv_ref = xb @ _bf(W["Wqkv"]).T + W["bqkv"]
    _close_bf16(cap["qkv"], qkv_ref, "qkv")
    qkv = _d(cap["qkv"]).view(E * S, 128, 3, H, 64).permute(2, 0, 3, 1, 4)  # [3][seq][head][128][64]
    q, k, v = qkv[0], qkv[1], qkv[2]
    P = torch.softmax(q @ k.transpose(-1, -2) / 8, -1)
    am = attn_scale()
    drop_frac = (am == 0).double().mean().item()
    assert abs(drop_frac - pa) < 0.01, drop_frac
    Pd = _bf(P * am)
    ctx_ref = (Pd @ v).permute(0, 2, 1, 3).reshape(T, D)
    _close_bf16(cap["ctx"], ctx_ref, "ctx")
    ctx = _d(cap["ctx"])
    hm1 = hidden_scale(0)
    hs1_ref = x32 + (_bf(ctx @ _bf(W["Wo"]).T) + W["bo"]) * hm1  # branch GEMM output rounded to bf16
    _close(cap["hs1"], hs1_ref, "ln1 input", rel=2e-3)
    hs1 = _d(cap["hs1"])
    h1, mean1, rstd1 = _ln(hs1, W["g1"], W["be1"], eps)
    _close(cap["st1"][:, 0], mean1, "ln1 mean", rel=1e-5)
    _close(cap["st1"][:, 1], rstd1, "ln1 rstd", rel=1e-5)
    _close_bf16(cap["h1b"], h1, "ln1 out")
    h1b = _d(cap["h1b"])
    hpre = h1b @ _bf(W["W1"]).T + W["b1"]
    _close_bf16(cap["Hpre"], _gelu_grad(hpre), "gelu' kept for the backward")
    _close_bf16(cap["Dact"], _gelu(hpre), "gelu")
    hm2 = hidden_scale(1)
    hs2_ref = h1 + (_bf(_d(cap["Dact"]) @ _bf(W["W2"]).T) + W["b2"]) * hm2
    _close(cap["hs2"], hs2_ref, "ln2 input", rel=2e-3)
    # ---- loss head
    ytop, tgt = _d(cap["ytop"]), _d(cap["tgt"])
    diff = ytop - tgt
    loss_ref = (0.5 * diff ** 2).view(E, Te * D).sum(1) / Te
    assert torch.allclose(_d(losses), loss_ref, rtol=1e-5), (losses, loss_ref)
    # ---- backward, layer 0
    dy1 = _d(cap["dy1_top"])
    dy2 = _d(cap["dy2_top"])
    hs2 = _d(cap["hs2"])
    dg_ref, xh2 = _ln_bwd(dy1 + dy2, hs2, W["g2"], eps)
    _close(cap["dg"], dg_ref, "ln2 backward")
    do_ref = _d(cap["dg"]) * hm2
    _close_bf16(cap["do"], do_ref, "ffn-out dropout'")
    do = _d(cap["do"])
    gelu_g = _d(cap["Hpre"])  # the stored gelu'(h)
    _close_bf16(cap["dHpre"], (do @ _bf(W["W2"])) * gelu_g, "dHpre")
    dHpre = _d(cap["dHpre"])
    _close_bf16(cap["dh1"], dHpre @ _bf(W["W1"]), "dh1")
    dyl1 = _d(cap["dh1"]) + _d(cap["dg"])
    dh_ref, xh1 = _ln_bwd(dyl1, hs1, W["g1"], eps)
    _close(cap["dh"], dh_ref, "ln1 backward")
    _close_bf16(cap["da"], _d(cap["dh"]) * hm1, "attn-out dropout'")
    da = _d(cap["da"])
    _close_bf16(cap["dctx"], da @ _bf(W["Wo"]), "dctx")
    dctx = _d(cap["dctx"]).view(E * S, 128, H, 64).permute(0, 2, 1, 3)
    dPd = dctx @ v.transpose(-1, -2)
    dP = dPd * am
    dS = _bf(P * (dP - (dP * P).sum(-1, keepdim=True)) / 8)
    dq_ref, dk_ref, dv_ref = dS @ k, dS.transpose(-1, -2) @ q, Pd.transpose(-1, -2) @ dctx
    dqkv_ref = torch.stack([dq_ref, dk_ref, dv_ref]).permute(1, 3, 0, 2, 4).reshape(T, 3 * D)
    _close_bf16(cap["dqkv"], dqkv_ref, "attention backward", frac=2e-2, rel=1e-2)
    dqkv = _d(cap["dqkv"])
    _close_bf16(cap["dx"], dqkv @ _bf(W["Wqkv"]), "dx")
    # ---- per-EST gradients of layer 0
    g = cap["grads"]
    for e in range(E):
        r = slice(e * Te, (e + 1) * Te)
        want = {
            "Wqkv": dqkv[r].T @ xb[r], "bqkv": dqkv[r].sum(0),
            "Wo": da[r].T @ ctx[r], "bo": (_d(cap["dh"])[r] * hm1[r]).sum(0),
            "g1": (dyl1[r] * xh1[r]).sum(0), "be1": dyl1[r].sum(0),
            "W1": dHpre[r].T @ h1b[r], "b1": dHpre[r].sum(0),
            "W2": do[r].T @ _d(cap["Dact"])[r], "b2": (_d(cap["dg"])[r] * hm2[r]).sum(0),
            "g2": ((dy1 + dy2)[r] * xh2[r]).sum(0), "be2": (dy1 + dy2)[r].sum(0),
        }
        for name, w_ in want.items():
            _close(job.view(0, name, g[e]), w_, f"grad {name} est {e}", rel=5e-3)
    # ---- fixed-order mean + momentum SGD (v0 = 0: v = mean_e g_e, p' = p - lr v)
    mean_g = _d(g).mean(0)
    _close(job.vel, mean_g, "velocity", rel=1e-6)
    _close(job.params - P0, -job.lr * mean_g, "update", rel=1e-4)


def test_gradient_leaf_groups(bert):
    """est_group=2: ESTs (0,1), (2,3) accumulate into one gradient leaf each (GEMM K over EST 2j's then
    2j+1's tokens); mapping-invariant for launch groups of whole leaves, the reducer's mean still over
    E; leaf gradients equal the sum of the per-EST gradients within fp32 accumulation error."""
    from paper_2208_14228_b200.errors import ConfigError

    a = bert.BertJob(est_group=2, **SMALL)
    b = bert.BertJob(est_group=2, **SMALL)
    for _ in range(2):
        assert np.array_equal(_bits(a.step([2, 2])), _bits(b.step([4])))
    assert np.array_equal(_bits(a.params), _bits(b.params))
    with pytest.raises(ConfigError):
        a.step([1, 3])
    one, two = bert.BertJob(**SMALL), bert.BertJob(est_group=2, **SMALL)
    c1, c2 = {}, {}
    l1, l2 = one.step(capture=c1), two.step(capture=c2)
    assert np.array_equal(_bits(l1), _bits(l2))  # the forward is per EST either way
    g1, g2 = c1["grads"].double(), c2["grads"].double()
    for j in range(2):
        want = g1[2 * j] + g1[2 * j + 1]
        assert ((g2[j] - want).norm() / want.norm()).item() < 1e-5
    assert ((two.params.double() - one.params.double()).norm() / one.params.double().norm()).item() < 1e-6


def test_adam_update(bert):
    """optimizer="adam": the reducer's final pass applies Adam (bias-corrected, beta1 = momentum) --
    mapping-invariant bits like SGD, and the first update equals a float64 Adam step of the captured
    mean gradient within fp32 rounding."""
    a = bert.BertJob(optimizer="adam", **dict(SMALL, lr=1e-3))
    b = bert.BertJob(optimizer="adam", **dict(SMALL, lr=1e-3))
    p0 = a.params.clone()
    cap = {}
    a.step(capture=cap)
    b.step([1, 3])
    assert np.array_equal(_bits(a.params), _bits(b.params)) and np.array_equal(_bits(a.vel2), _bits(b.vel2))
    g = _d(cap["grads"]).mean(0)
    m, s = 0.1 * g, 0.001 * g * g
    want = _d(p0) - 1e-3 * (m / 0.1) / (torch.sqrt(s / 0.001) + 1e-8)
    _close(a.params, want, "adam step", rel=1e-6)
    for _ in range(2):
        assert np.array_equal(_bits(a.step()), _bits(b.step([2, 2])))
    assert np.array_equal(_bits(a.params), _bits(b.params))


def test_cuda_graph_replay_equals_eager(bert):
    """The captured step (one CUDA graph: every launch group, the reducer, the weight refresh, the device
    step counter) replays bit-identically to eager execution, step after step."""
    a = bert.BertJob(graph=True, **SMALL)
    b = bert.BertJob(graph=False, **SMALL)
    for _ in range(4):
        assert np.array_equal(_bits(a.step()), _bits(b.step()))
    assert a._graph is not None and b._graph is None
    assert np.array_equal(_bits(a.params), _bits(b.params)) and int(a._step_dev.item()) == 4


def test_tcgen05_attention_forward_matches_mma_sync(bert, monkeypatch):
    """The tcgen05 attention forward (bt_attn_tc.cu: S and PV on the 5th-gen tensor cores, one softmax
    row per thread) and the mma.sync forward apply the same keyed dropout masks to the same softmax:
    their ctx agree to bf16 rounding (<= 1% of elements one ulp apart), each is run-to-run bitwise
    stable, and the tcgen05 path keeps the grouping invariance."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    job = bert.BertJob(**SMALL)
    cap = {}
    job.step(capture=cap)
    qkv = cap["qkv"]
    E, Te, D, H = job.E, job.Te, job.D, job.H
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("BT_ATTN_TC", mode)
        o = torch.empty(E * Te, D, dtype=torch.bfloat16, device="cuda")
        _native.check(_native.lib().bt_bert_attn(0, qkv.data_ptr(), None, o.data_ptr(), E, Te, D, H, 0, job.L, 0,
                                                 job.seed, 0, job.pa, None, stream()))
        o2 = torch.empty_like(o)
        _native.check(_native.lib().bt_bert_attn(0, qkv.data_ptr(), None, o2.data_ptr(), E, Te, D, H, 0, job.L, 0,
                                                 job.seed, 0, job.pa, None, stream()))
        assert torch.equal(o.view(torch.int16), o2.view(torch.int16))
        outs[mode] = o
    monkeypatch.delenv("BT_ATTN_TC")
    a, b = _d(outs["1"]), _d(outs["0"])
    assert torch.equal(a, _d(cap["ctx"]))  # the step used the tcgen05 path
    assert (a != b).double().mean().item() <= 1e-2
    assert ((a - b).norm() / b.norm()).item() <= 5e-3


def test_tcgen05_attention_backward_matches_mma_sync(bert, monkeypatch):
    """The tcgen05 attention backward (bt_attn_tc.cu: S, dP, dQ, dK, dV as UMMAs, the forward's exact
    softmax recomputation, K-major tiles read MN-major for the transposed products) agrees with the
    mma.sync backward to bf16 rounding and is run-to-run bitwise stable."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    job = bert.BertJob(**SMALL)
    cap = {}
    job.step(capture=cap)
    qkv, dctx = cap["qkv"], cap["dctx"]
    E, Te, D, H = job.E, job.Te, job.D, job.H
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("BT_ATTN_TC", mode)
        res = []
        for _ in range(2):
            o = torch.empty(E * Te, 3 * D, dtype=torch.bfloat16, device="cuda")
            _native.check(_native.lib().bt_bert_attn(1, qkv.data_ptr(), dctx.data_ptr(), o.data_ptr(), E, Te, D, H,
                                                     0, job.L, 0, job.seed, 0, job.pa, None, stream()))
            res.append(o)
        assert torch.equal(res[0].view(torch.int16), res[1].view(torch.int16))
        outs[mode] = res[0]
    monkeypatch.delenv("BT_ATTN_TC")
    a, b = _d(outs["1"]), _d(outs["0"])
    assert torch.equal(a, _d(cap["dqkv"]))  # the step used the tcgen05 path
    for part in range(3):
        x, y = a[:, part * D:(part + 1) * D], b[:, part * D:(part + 1) * D]
        assert (x != y).double().mean().item() <= 3e-2, part
        assert ((x - y).norm() / y.norm()).item() <= 1e-2, part


def test_layernorm_residual_recompute_equals_stored(bert):
    """bt_bert_ln_fwd_rc (the residual recomputed from the previous LayerNorm's input, statistics and
    affine parameters) gives the bits of bt_bert_ln_fwd fed the previous LayerNorm's stored fp32 output."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    L = _native.lib()
    E, Te, D = 2, 128, 768
    T = E * Te
    g = torch.Generator(device="cuda").manual_seed(5)
    f32 = dict(device="cuda", dtype=torch.float32)

    def rnd(*shape, scale=1.0):
        return torch.randn(*shape, generator=g, **f32) * scale

    x0, b0 = rnd(T, D), rnd(T, D).to(torch.bfloat16)
    bias0, g0, be0 = rnd(D, scale=0.1), 1 + rnd(D, scale=0.1), rnd(D, scale=0.1)
    bias1, g1, be1 = rnd(D, scale=0.1), 1 + rnd(D, scale=0.1), rnd(D, scale=0.1)
    b1 = rnd(T, D).to(torch.bfloat16)
    hs0, st0, y0, yb0 = torch.empty(T, D, **f32), torch.empty(T, 2, **f32), torch.empty(T, D, **f32), \
        torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    args = (E, Te, D, 0, 2, 0, 1, 42, 3, 0.1, 1e-5, None, stream())
    _native.check(L.bt_bert_ln_fwd(x0.data_ptr(), b0.data_ptr(), bias0.data_ptr(), g0.data_ptr(), be0.data_ptr(),
                                   hs0.data_ptr(), st0.data_ptr(), y0.data_ptr(), yb0.data_ptr(), *args))
    outs = []
    for rc in (False, True):
        hs, st = torch.empty(T, D, **f32), torch.empty(T, 2, **f32)
        y, yb = torch.empty(T, D, **f32), torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
        if rc:
            _native.check(L.bt_bert_ln_fwd_rc(hs0.data_ptr(), st0.data_ptr(), g0.data_ptr(), be0.data_ptr(),
                                              b1.data_ptr(), bias1.data_ptr(), g1.data_ptr(), be1.data_ptr(),
                                              hs.data_ptr(), st.data_ptr(), y.data_ptr(), yb.data_ptr(), *args))
        else:
            _native.check(L.bt_bert_ln_fwd(y0.data_ptr(), b1.data_ptr(), bias1.data_ptr(), g1.data_ptr(),
                                           be1.data_ptr(), hs.data_ptr(), st.data_ptr(), y.data_ptr(), yb.data_ptr(),
                                           *args))
        outs.append((hs, st, y, yb))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a.view(torch.int16 if a.dtype == torch.bfloat16 else torch.int32),
                           b.view(torch.int16 if b.dtype == torch.bfloat16 else torch.int32))


TAG_TOK = 0x4245_5254_544F_4B4E
TAG_MASK = 0x4245_5254_4D41_534B


@pytest.mark.parametrize("g", [1, 2])
def test_mlm_head_and_embeddings_match_float64(bert, g):
    """Token ids / masked positions regenerated from splitmix64 (bit-exact); the word + position
    embedding (exact fp32 adds); logits against the tied embedding + bias, the per-EST masked-LM
    cross-entropy, dlogits, dy at the masked rows; the per-leaf decoder weight and bias gradients;
    and the embedding gradient (tied decoder part + the sorted segment sum of dx rows, no atomics)
    and the position-embedding gradient -- against a float64 restatement of the captured tensors."""
    from paper_2208_14228_b200._native import host_derive_stream

    job = bert.BertJob(est_group=g, **dict(SMALL, vocab=1000, npred=20))
    P0 = job.params.clone()
    cap = {}
    losses = job.step(capture=cap)
    E, S, Te, D, V, Vp, NPd = job.E, job.S, job.Te, job.D, job.V, job.Vp, job.NP
    # ---- ids and masked positions (the partial Fisher-Yates + sort), bit for bit
    ids_want, mrow_want, lab_want = [], [], []
    for e in range(E):
        st, sm = host_derive_stream(TAG_TOK, job.seed, e), host_derive_stream(TAG_MASK, job.seed, e)
        for sl in range(S):
            ids = [int(x % np.uint64(V)) for x in _draws(st, np.arange(sl * 128, sl * 128 + 128))]
            pos = list(range(128))
            raws = _draws(sm, np.arange(sl * NPd, sl * NPd + NPd))
            for k in range(NPd):
                j = k + int(raws[k] % np.uint64(128 - k))
                pos[k], pos[j] = pos[j], pos[k]
            chosen = sorted(pos[:NPd])
            seq = e * S + sl
            mrow_want += [seq * 128 + p for p in chosen]
            lab_want += [ids[p] for p in chosen]
            ids_want += [job.mask_id if p in chosen else ids[p] for p in range(128)]
    assert cap["ids"].tolist() == ids_want
    assert cap["mrow"].tolist() == mrow_want and cap["mlabel"].tolist() == lab_want
    # ---- embeddings
    Wemb, Pemb, bdec = _d(job.eview("Wemb", P0)), _d(job.eview("Pemb", P0)), _d(job.eview("bdec", P0))
    ids = torch.tensor(ids_want)
    x32_ref = (job.eview("Wemb", P0)[ids.cuda()] + job.eview("Pemb", P0).repeat(E * S, 1)).cpu()
    assert torch.equal(cap["x32"].cpu(), x32_ref)
    # ---- head forward
    ym = _d(cap["ym"])
    assert torch.equal(ym, _d(cap["ytop_b"])[torch.tensor(mrow_want)])
    logits_ref = ym @ _bf(Wemb).T + bdec
    _close(cap["logits"][:, :V], logits_ref[:, :V], "logits", rel=1e-5)
    lg = _d(cap["logits"])[:, :V]
    lab = torch.tensor(lab_want)
    ce = torch.nn.functional.cross_entropy(lg, lab, reduction="none")
    per = S * NPd
    _close(losses, ce.view(E, per).mean(1), "per-EST masked-LM loss", rel=1e-5)
    sm_ = torch.softmax(lg, -1)
    dl_ref = (sm_ - torch.nn.functional.one_hot(lab, V).double()) / per
    dl = _d(cap["dlogits"])
    _close_bf16(dl[:, :V], dl_ref, "dlogits")
    assert bool((dl[:, V:] == 0).all())
    _close_bf16(cap["dym"], dl @ _bf(Wemb), "dy at the masked rows")
    # ---- gradients per leaf
    gr = cap["grads"].double().cpu()
    dx = _d(cap["dx"]) + _d(cap["dx_res"])
    K = g * per
    for j in range(E // g):
        rows = slice(j * K, (j + 1) * K)
        dec = dl[rows].T @ ym[rows]
        _close(job.eview("bdec", gr[j])[:V], dl[rows].sum(0)[:V], f"decoder bias leaf {j}", rel=2e-3)
        toks = slice(j * g * Te, (j + 1) * g * Te)
        emb = torch.zeros(Vp, D, dtype=torch.float64)
        emb.index_add_(0, ids[toks], dx[toks])
        _close(job.eview("Wemb", gr[j]), dec + emb, f"word embedding gradient leaf {j}", rel=5e-3)
        pos_ref = dx[toks].view(g * S, 128, D).sum(0)
        _close(job.eview("Pemb", gr[j]), pos_ref, f"position embedding gradient leaf {j}", rel=1e-5)


def test_mlm_head_groupings_are_bitwise_identical(bert):
    """The masked-LM head + embedding gradient keep the mapping invariance (launch groups of whole leaves)."""
    a = bert.BertJob(est_group=2, **SMALL)
    b = bert.BertJob(est_group=2, **SMALL)
    for _ in range(3):
        assert np.array_equal(_bits(a.step([2, 2])), _bits(b.step()))
    assert np.array_equal(_bits(a.params), _bits(b.params))


def test_run_logs_fingerprint_and_bitdiff(bert):
    """The model stack's run log (runlog.RunLog: per-EST losses + the device weight fingerprint per step):
    two groupings give identical logs (bitdiff: no divergence); the fingerprint is byte-exact (a
    one-ULP change of one weight changes it) and equals its host restatement."""
    import numpy as np

    from paper_2208_14228_b200.prng import fnv1a64
    from paper_2208_14228_b200.runlog import bitdiff, device_fingerprint

    a = bert.BertJob(est_group=2, **SMALL)
    b = bert.BertJob(est_group=2, **SMALL)
    la = a.run_log(3)
    lb = b.run_log(3, groups=[2, 2])
    assert bitdiff(la, lb) is None and all(r.param_hash for r in la.records)
    raw = a.params.cpu().numpy().tobytes()
    chunks = [raw[i:i + (1 << 16)] for i in range(0, len(raw), 1 << 16)]
    host = np.array([fnv1a64(c) for c in chunks], dtype=np.uint64).astype("<u8").tobytes()
    assert device_fingerprint(a.params) == f"{fnv1a64(host):016x}" == la.records[-1].param_hash
    p = a.params.clone()
    p[12345] = float(np.nextafter(np.float32(p[12345].item()), np.float32(2.0)))
    assert device_fingerprint(p) != la.records[-1].param_hash


def test_deferred_status_check_keeps_weights(bert):
    """step(check=False) skips the per-step host synchronisation; the update stays guarded on the device: a
    non-finite step and every step after it leave weights and momentum bit-for-bit unchanged, and the next
    check_status() raises NumericError (the status words are sticky)."""
    from paper_2208_14228_b200.errors import NumericError

    job = bert.BertJob(**SMALL)
    job.step()
    job.step(check=False)
    job.check_status()  # finite steps: nothing to report
    job.view(0, "Wo")[0, 0] = float("nan")
    job._refresh_bf16()
    p0, v0 = job.params.clone(), job.vel.clone()
    for _ in range(3):
        job.step(check=False)
    torch.cuda.synchronize()
    assert torch.equal(job.params.view(torch.int32), p0.view(torch.int32))
    assert torch.equal(job.vel.view(torch.int32), v0.view(torch.int32))
    with pytest.raises(NumericError):
        job.check_status()
    job.check_status()  # reset by the raise
