"""The deterministic reducer (bt_reduce_update) vs the oracle, C5-style inputs.

Bit-exact (0 ulp) for every variant, dtype and E: the fold order is a pure
function of (EST rank, fanin, rotation).  Inputs mirror the adversarial
generator of the reference's test_buckets.py:93-98 ((u*2-1)*10^k, k in
[-12, 12]) so any order bug flips low bits.
"""

import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def adversarial(E, n, seed, dtype):
    rng = np.random.default_rng(seed)
    mant = rng.uniform(-1, 1, (E, n))
    exp = rng.integers(-12, 13, (E, n)).astype(np.float64)
    return (mant * 10.0**exp).astype(dtype)


def run_reduce(grads, rot, fanin, params, vel, lr, mu, table=True, nout=0):
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import Flags, stream

    E, n = grads.shape
    f64 = grads.dtype == np.float64
    g = torch.from_numpy(grads).cuda()
    p = torch.from_numpy(params).cuda()
    v = torch.from_numpy(vel).cuda()
    po, vo = torch.empty_like(p), torch.empty_like(v)
    extra = [(torch.empty_like(p), torch.empty_like(v)) for _ in range(nout)]
    flags = Flags()
    a = _native.ReduceArgs()
    a.dtype = _native.DTYPE_F64 if f64 else _native.DTYPE_F32
    a.mode, a.E, a.fanin, a.n, a.nout = _native.REDUCE_UPDATE, E, fanin, n, nout
    if table:
        for k in range(E):
            a.grads[k] = g[k].data_ptr()
    else:
        a.grads[0] = g.data_ptr()
        a.grads_ld = n
    rt = None
    if rot is not None:
        rt = torch.from_numpy(rot.astype(np.int32)).cuda()
        a.rot = rt.data_ptr()
    a.param, a.vel, a.param_out, a.vel_out = p.data_ptr(), v.data_ptr(), po.data_ptr(), vo.data_ptr()
    for r, (ep, ev) in enumerate(extra):
        a.extra_param_out[r], a.extra_vel_out[r] = ep.data_ptr(), ev.data_ptr()
    a.lr, a.mu, a.flags = lr, mu, flags.t.data_ptr()
    _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
    st, detail, _ = flags.status()
    return po.cpu().numpy(), vo.cpu().numpy(), st, detail, [(x.cpu().numpy(), y.cpu().numpy()) for x, y in extra]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("E", [1, 2, 4, 8, 16, 32, 64, 3, 5, 12])
@pytest.mark.parametrize("variant", ["seq", "tree2", "tree3"])
def test_reducer_bitexact_vs_oracle(oracle, dtype, E, variant):
    n = 50_003  # not a multiple of the vector width: exercises the tail
    grads = adversarial(E, n, 1000 + E, dtype)
    params = adversarial(1, n, 7, dtype)[0]
    vel = adversarial(1, n, 8, dtype)[0]
    lr, mu = 0.02, 0.9
    want_p, want_v = oracle.reduce_update(grads, None, variant, params, vel, lr, mu)
    got_p, got_v, st, _, _ = run_reduce(grads, None, oracle.fanin_of(variant), params, vel, lr, mu)
    assert st == 0
    assert np.array_equal(got_p.view(np.uint8), want_p.view(np.uint8))
    assert np.array_equal(got_v.view(np.uint8), want_v.view(np.uint8))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("E", [4, 8, 13])
def test_reducer_rotated_tree_matches_bucket_map_oracle(oracle, dtype, E):
    """Tree with the reference's ring-chunk rotation (buckets.py:119-122)."""
    n = 20_000
    grads = adversarial(E, n, 55 + E, dtype)
    bm = oracle.buckets_initial(n, 64)
    rot = oracle.rotation_table(bm, E, n)
    params = np.zeros(n, dtype)
    vel = np.zeros(n, dtype)
    want_p, want_v = oracle.reduce_update(grads, rot, "tree2", params, vel, 1.0, 0.0)
    got_p, got_v, st, _, _ = run_reduce(grads, rot, 2, params, vel, 1.0, 0.0, table=False)
    assert st == 0
    assert np.array_equal(got_v.view(np.uint8), want_v.view(np.uint8))
    assert np.array_equal(got_p.view(np.uint8), want_p.view(np.uint8))


def test_reducer_strided_equals_table(oracle):
    grads = adversarial(8, 10_001, 3, np.float32)
    p = np.zeros(10_001, np.float32)
    a = run_reduce(grads, None, 2, p, p, 0.1, 0.9, table=True)
    b = run_reduce(grads, None, 2, p, p, 0.1, 0.9, table=False)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_reducer_extra_replica_outputs_are_copies(oracle):
    grads = adversarial(4, 4096, 9, np.float64)
    p = adversarial(1, 4096, 10, np.float64)[0]
    po, vo, st, _, extra = run_reduce(grads, None, 0, p, np.zeros_like(p), 0.1, 0.9, nout=3)
    assert st == 0
    for ep, ev in extra:
        assert np.array_equal(ep, po) and np.array_equal(ev, vo)


def test_reducer_flags_non_finite(oracle):
    grads = adversarial(8, 1000, 4, np.float32)
    grads[3, 517] = np.inf
    p = np.zeros(1000, np.float32)
    _, _, st, detail, _ = run_reduce(grads, None, 0, p, p, 0.1, 0.9)
    assert st == 5 and detail == 516  # first element of the 4-wide vector holding 517


def test_reducer_layout_invariance_hierarchical_rank_tree(oracle):
    """RankTree(2): per-GPU subtrees over contiguous EST blocks, combined in
    rank order, equal the flat tree over all ESTs (power-of-two E/G)."""
    E, n = 16, 8192
    grads = adversarial(E, n, 21, np.float32)
    z = np.zeros(n, np.float32)
    flat_p, _, _, _, _ = run_reduce(grads, None, 2, z, z, -1.0, 0.0)
    for G in (2, 4, 8):
        per = E // G
        partial = np.stack([run_reduce(grads[g * per:(g + 1) * per], None, 2, z, z, -1.0, 0.0)[0] * per
                            for g in range(G)])
        # partials are sums (mean*per is exact only for power-of-two per)
        top, _, _, _, _ = run_reduce(partial.astype(np.float32), None, 2, z, z, -1.0, 0.0)
        top = (top * G).astype(np.float32) / np.float32(E)
        assert np.array_equal(top.view(np.uint32), flat_p.view(np.uint32)), G


def _fold(grads, fanin):
    """numpy restatement of the reducer's fold in the grads' dtype: Sequential left fold / Tree(2)"""
    if fanin == 0:
        acc = grads[0].copy()
        for k in range(1, grads.shape[0]):
            acc = acc + grads[k]
        return acc
    level = [grads[k] for k in range(grads.shape[0])]
    while len(level) > 1:
        level = [level[i] + level[i + 1] if i + 1 < len(level) else level[i] for i in range(0, len(level), 2)]
    return level[0]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("fanin,E,nout", [(0, 8, 0), (2, 8, 1), (2, 16, 0), (0, 5, 2)])
def test_fused_adam_update_bit_exact(dtype, fanin, E, nout):
    """BT_REDUCE_ADAM (the north star's "or Adam"): the rank-ordered fold, /E, then Adam with caller-side
    bias corrections -- every operation round-to-nearest in a fixed order, so it equals a numpy
    restatement in the same dtype bit for bit (vector body, scalar tail, replica outputs)."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import Flags, stream

    n = 10_003
    grads = adversarial(E, n, 17 + E, dtype) * dtype(1e-9)
    rng = np.random.default_rng(3)
    p0 = rng.uniform(-1, 1, n).astype(dtype)
    m0 = (rng.uniform(-1, 1, n) * 1e-3).astype(dtype)
    s0 = (rng.uniform(0, 1, n) * 1e-6).astype(dtype)
    b1, b2, eps, lr, t = 0.9, 0.999, 1e-8, 1e-3, 7
    bc1, bc2 = 1.0 / (1.0 - b1 ** t), 1.0 / (1.0 - b2 ** t)
    g_t, p_t, m_t, s_t = (torch.from_numpy(x).cuda() for x in (grads, p0, m0, s0))
    extra = [tuple(torch.empty_like(p_t) for _ in range(3)) for _ in range(nout)]
    flags = Flags()
    a = _native.ReduceArgs()
    a.dtype = _native.DTYPE_F64 if dtype == np.float64 else _native.DTYPE_F32
    a.mode, a.E, a.fanin, a.n, a.nout = _native.REDUCE_ADAM, E, fanin, n, nout
    for k in range(E):
        a.grads[k] = g_t[k].data_ptr()
    a.param = a.param_out = p_t.data_ptr()
    a.vel = a.vel_out = m_t.data_ptr()
    a.vel2 = a.vel2_out = s_t.data_ptr()
    for r, (ep, em, es) in enumerate(extra):
        a.extra_param_out[r], a.extra_vel_out[r], a.extra_vel2_out[r] = ep.data_ptr(), em.data_ptr(), es.data_ptr()
    a.lr, a.mu, a.beta2, a.eps, a.bc1, a.bc2, a.flags = lr, b1, b2, eps, bc1, bc2, flags.t.data_ptr()
    _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
    assert flags.status()[0] == 0
    T = dtype
    g = _fold(grads, fanin) / T(E)
    m1 = T(b1) * m0 + (T(1) - T(b1)) * g
    s1 = T(b2) * s0 + (T(1) - T(b2)) * (g * g)
    p1 = p0 - T(lr) * ((m1 * T(bc1)) / (np.sqrt(s1 * T(bc2)) + T(eps)))
    for got, want in ((p_t, p1), (m_t, m1), (s_t, s1)):
        assert np.array_equal(got.cpu().numpy().view(np.uint8), want.astype(dtype).view(np.uint8))
    for ep, em, es in extra:
        assert torch.equal(ep, p_t) and torch.equal(em, m_t) and torch.equal(es, s_t)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("fanin,E,nout", [(0, 8, 0), (2, 8, 2), (2, 5, 1)])
def test_guarded_update_commits_only_finite_steps(oracle, dtype, fanin, E, nout):
    """`stage` set: a finite update equals the single-pass one bit for bit; a non-finite synchronized
    gradient anywhere leaves param, velocity and every replica output untouched (the reference's
    sgd_step raises before it mutates anything, model.py:207-209) and reports NumericError."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import Flags, stream

    n = 10_007
    grads = adversarial(E, n, 31 + E, dtype)
    p0 = adversarial(1, n, 5, dtype)[0]
    v0 = adversarial(1, n, 6, dtype)[0]
    want_p, want_v, st, _, _ = run_reduce(grads, None, fanin, p0, v0, 0.02, 0.9)
    assert st == 0
    for bad in (False, True):
        g = grads.copy()
        if bad:
            g[E - 1, n - 2] = np.nan  # in the scalar tail of the last shard of the vector body
        g_t = torch.from_numpy(g).cuda()
        p_t, v_t = torch.from_numpy(p0.copy()).cuda(), torch.from_numpy(v0.copy()).cuda()
        extra = [(p_t.clone(), v_t.clone()) for _ in range(nout)]
        stage = torch.empty_like(p_t)
        flags = Flags()
        a = _native.ReduceArgs()
        a.dtype = _native.DTYPE_F64 if dtype == np.float64 else _native.DTYPE_F32
        a.mode, a.E, a.fanin, a.n, a.nout = _native.REDUCE_UPDATE, E, fanin, n, nout
        for k in range(E):
            a.grads[k] = g_t[k].data_ptr()
        a.param = a.param_out = p_t.data_ptr()
        a.vel = a.vel_out = v_t.data_ptr()
        for r, (ep, ev) in enumerate(extra):
            a.extra_param_out[r], a.extra_vel_out[r] = ep.data_ptr(), ev.data_ptr()
        a.lr, a.mu, a.flags, a.stage = 0.02, 0.9, flags.t.data_ptr(), stage.data_ptr()
        _native.check(_native.lib().bt_reduce_update(C.byref(a), stream()))
        st, detail, _ = flags.status()
        if bad:
            assert st == 5 and detail == n - 2
            wp, wv = p0, v0
        else:
            assert st == 0
            wp, wv = want_p, want_v
        assert np.array_equal(p_t.cpu().numpy().view(np.uint8), wp.view(np.uint8))
        assert np.array_equal(v_t.cpu().numpy().view(np.uint8), wv.view(np.uint8))
        for ep, ev in extra:
            assert torch.equal(ep, p_t) and torch.equal(ev, v_t)
