"""Deterministic tcgen05 GEMM (csrc/bt_gemm.cu) vs a float64 reference (needs a B200).

Numerics: bf16 inputs, fp32 accumulation -> |C - C64| <= K * 2^-23 * sum_k |a_ik b_jk|
(the fp32-accumulation bound, stated here as the test tolerance).  Determinism:
bit-identical across repeats and across grid sizes (1 CTA ... one per SM),
which is the property the elastic step needs from its model kernels.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = [(128, 128, 64), (256, 384, 512), (512, 512, 1024), (384, 1024, 768), (1024, 256, 4096)]


@pytest.fixture(scope="module")
def gemm():
    assert torch.cuda.is_available()
    from paper_2208_14228_b200.gemm import gemm_bf16

    return gemm_bf16


def _inputs(M, N, K, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    a = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    return a, b


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_gemm_matches_float64(gemm, M, N, K):
    a, b = _inputs(M, N, K, M + N + K)
    c = gemm(a, b)
    ref = a.double() @ b.double().T
    bound = K * 2.0 ** -23 * (a.double().abs() @ b.double().abs().T)
    err = (c.double() - ref).abs()
    assert bool((err <= bound + 1e-30).all()), float((err / (bound + 1e-30)).max())
    # and it agrees with cuBLAS (torch) to fp32-accumulation accuracy
    cub = torch.matmul(a.float(), b.float().T)
    assert bool(((c - cub).abs().double() <= 2 * bound + 1e-30).all())


@pytest.mark.parametrize("M,N,K", [(512, 512, 1024), (384, 1024, 768)])
def test_gemm_bitwise_deterministic_across_grids(gemm, M, N, K):
    a, b = _inputs(M, N, K, 7)
    ref = gemm(a, b)
    for grid in (0, 1, 3, 7, 37, 148):
        c = gemm(a, b, grid=grid)
        assert torch.equal(c.view(torch.int32), ref.view(torch.int32)), grid


def test_gemm_bf16_output_is_rounded_fp32(gemm):
    a, b = _inputs(256, 512, 640, 3)
    c32 = gemm(a, b)
    c16 = gemm(a, b, out_dtype=torch.bfloat16)
    assert torch.equal(c16.view(torch.int16), c32.to(torch.bfloat16).view(torch.int16))


def test_gemm_rejects_bad_shapes(gemm):
    from paper_2208_14228_b200.errors import InputError

    a, b = _inputs(128, 128, 64, 1)
    with pytest.raises(InputError):  # K-major rows must be 16-byte aligned (K % 8)
        gemm(a[:, :30].contiguous(), b[:, :30].contiguous())
    with pytest.raises(InputError):  # N % 8
        gemm(a, b[:100].contiguous())


@pytest.mark.parametrize("M,N,K,mn", [(200, 72, 40, False), (96, 64, 1000, False), (1000, 576, 96, False),
                                      (72, 24, 4096, True), (576, 64, 2048, True), (64, 32, 640, True)])
def test_ragged_shapes(gemm, M, N, K, mn):
    """M, N, K off the 128 / 64 tile grid (64-channel convolutions, 3x3x3 stems, 576-wide im2col weight
    gradients): TMA zero-fills the loads and clips the stores; results within the fp32 bound."""
    from paper_2208_14228_b200.gemm import gemm_bf16_at_b

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    if mn:
        a = torch.randn(2, K, M, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(2, K, N, device="cuda", generator=g).to(torch.bfloat16)
        c = gemm_bf16_at_b(a, b)
        ref = torch.einsum("ekm,ekn->emn", a.double(), b.double())
        bound = K * 2.0 ** -23 * torch.einsum("ekm,ekn->emn", a.double().abs(), b.double().abs())
    else:
        a, b = _inputs(M, N, K, 3)
        c = gemm(a, b)
        ref = a.double() @ b.double().T
        bound = K * 2.0 ** -23 * (a.double().abs() @ b.double().abs().T)
    assert bool(((c.double() - ref).abs() <= bound + 1e-30).all())


def test_cta_pair_and_single_cta_kernels_agree_bitwise(gemm, monkeypatch):
    """The 256x256 CTA-pair kernel (cta_group::2) and the 128x256 1-CTA kernel give the same bits:
    the per-element accumulation order does not depend on the tile shape or the SM pairing."""
    a, b = _inputs(512, 768, 1536, 11)
    pair = gemm(a, b)
    monkeypatch.setenv("BT_GEMM_VARIANT", "1")
    single = gemm(a, b)
    monkeypatch.delenv("BT_GEMM_VARIANT")
    assert torch.equal(pair.view(torch.int32), single.view(torch.int32))


@pytest.mark.parametrize("E,M,N,K", [(4, 256, 256, 512), (3, 128, 384, 256), (8, 256, 768, 1024)])
def test_batched_gemm_equals_per_entry_gemms(gemm, E, M, N, K):
    from paper_2208_14228_b200.gemm import gemm_bf16_batched

    g = torch.Generator(device="cuda").manual_seed(E * 1000 + M)
    a = torch.randn(E, M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(E, N, K, device="cuda", generator=g).to(torch.bfloat16)
    c = gemm_bf16_batched(a, b)
    for e in range(E):
        assert torch.equal(c[e].view(torch.int32), gemm(a[e], b[e]).view(torch.int32)), e
    ref = torch.einsum("emk,enk->emn", a.double(), b.double())
    bound = K * 2.0 ** -23 * torch.einsum("emk,enk->emn", a.double().abs(), b.double().abs())
    assert bool(((c.double() - ref).abs() <= bound + 1e-30).all())


@pytest.mark.parametrize("E,M,N,K,variant", [(4, 256, 256, 512, "0"), (3, 128, 384, 256, "0"),
                                             (2, 768, 3072, 1024, "0"), (2, 256, 512, 256, "1")])
def test_mn_major_gemm(gemm, monkeypatch, E, M, N, K, variant):
    """c[e] = a[e]^T b[e] from token-major operands (MN-major TMA/UMMA): within the fp32-accumulation
    bound of a float64 reference, identical bits for every batch entry alone and in the batch, and
    (the accumulation order is the K order) the same bits as the K-major GEMM of the transposes."""
    from paper_2208_14228_b200.gemm import gemm_bf16_at_b, gemm_bf16_batched

    monkeypatch.setenv("BT_GEMM_VARIANT", variant)
    g = torch.Generator(device="cuda").manual_seed(E * 7 + N)
    a = torch.randn(E, K, M, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(E, K, N, device="cuda", generator=g).to(torch.bfloat16)
    c = gemm_bf16_at_b(a, b)
    ref = torch.einsum("ekm,ekn->emn", a.double(), b.double())
    bound = K * 2.0 ** -23 * torch.einsum("ekm,ekn->emn", a.double().abs(), b.double().abs())
    assert bool(((c.double() - ref).abs() <= bound + 1e-30).all())
    for e in range(E):
        assert torch.equal(c[e].view(torch.int32), gemm_bf16_at_b(a[e], b[e])[0].view(torch.int32)), e
    kmaj = gemm_bf16_batched(a.transpose(1, 2).contiguous(), b.transpose(1, 2).contiguous())
    assert torch.equal(c.view(torch.int32), kmaj.view(torch.int32))


@pytest.mark.parametrize("M,N,K,bf16", [(512, 768, 3072, True), (512, 3072, 768, False), (384, 256, 768, True),
                                         (200, 128, 256, False), (128, 64, 192, True)])
def test_b_mn_major_equals_k_major_on_the_transpose(M, N, K, bf16):
    """mn_major = 2 (A K-major, B stored [K][N]): C = A.B reading the weight as stored equals the
    K-major GEMM on B^T bit for bit -- pair tiles, 1-CTA 256/128/64 tiles and ragged M."""
    import ctypes as C

    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    a, bt = _inputs(M, N, K, 11)           # bt: [N][K] (K-major B)
    b_kn = bt.T.contiguous()               # the same matrix stored [K][N]
    dt = torch.bfloat16 if bf16 else torch.float32
    c0 = torch.empty(M, N, dtype=dt, device="cuda")
    c2 = torch.empty(M, N, dtype=dt, device="cuda")
    L = _native.lib()
    _native.check(L.bt_gemm_bf16_ex(a.data_ptr(), bt.data_ptr(), c0.data_ptr(), 1, M, N, K, 0, 0, 0, int(bf16), None,
                                    0, 0, stream()))
    _native.check(L.bt_gemm_bf16_ex(a.data_ptr(), b_kn.data_ptr(), c2.data_ptr(), 1, M, N, K, 0, 0, 0, int(bf16), None,
                                    2, 0, stream()))
    iv = torch.int16 if bf16 else torch.int32
    assert torch.equal(c0.view(iv), c2.view(iv))


def test_ffn_backward_epilogue_with_b_mn_major():
    """The FFN backward GEMM (dropout' + GELU' epilogue) reading W2 as stored [D][F] == on W2^T."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    T, F, D = 512, 1024, 256
    g = torch.Generator(device="cuda").manual_seed(5)
    dy = (torch.randn(T, D, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w2 = (torch.randn(D, F, device="cuda", generator=g) * 0.1).to(torch.bfloat16)   # [D][F] = [K][N]
    aux = (torch.randn(T, F, device="cuda", generator=g)).to(torch.bfloat16)
    outs = []
    for kind, b in ((2, w2.T.contiguous()), (2 | 0x100, w2)):
        c = torch.empty(T, F, dtype=torch.bfloat16, device="cuda")
        _native.check(_native.lib().bt_gemm_bf16_ffn(dy.data_ptr(), b.data_ptr(), c.data_ptr(), T, F, D, kind, None,
                                                     aux.data_ptr(), None, 42, 3, 0, 128, 0.1, 0, stream()))
        outs.append(c)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))


@pytest.mark.parametrize("variant", ["0", "1"])
def test_ffn_backward_epilogue_column_partials(monkeypatch, variant):
    """bt_gemm_bf16_ffn_cs: the FFN backward GEMM's epilogue also writes the column sums of its bf16 output
    over every 32-row block (even rows ascending + odd rows ascending, fp32) -- bit-exact against that
    association restated in numpy on the stored output, on the CTA-pair and the 1-CTA kernels; the per-leaf
    fold (bt_colsum_fold) sums the blocks in order, and the output itself is the plain FFN_BWD output."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    monkeypatch.setenv("BT_GEMM_VARIANT", variant)
    T, F, D = 1024, 768, 256
    g = torch.Generator(device="cuda").manual_seed(9)
    dy = (torch.randn(T, D, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w2 = (torch.randn(D, F, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    aux = (torch.randn(T, F, device="cuda", generator=g)).to(torch.bfloat16)
    L = _native.lib()
    c = torch.empty(T, F, dtype=torch.bfloat16, device="cuda")
    c_ref = torch.empty_like(c)
    part = torch.full((T // 32, F), float("nan"), device="cuda")
    _native.check(L.bt_gemm_bf16_ffn_cs(dy.data_ptr(), w2.data_ptr(), c.data_ptr(), T, F, D, 2 | 0x100, None,
                                        aux.data_ptr(), None, part.data_ptr(), 42, 3, 0, 256, 0.1, 0, stream()))
    _native.check(L.bt_gemm_bf16_ffn(dy.data_ptr(), w2.data_ptr(), c_ref.data_ptr(), T, F, D, 2 | 0x100, None,
                                     aux.data_ptr(), None, 42, 3, 0, 256, 0.1, 0, stream()))
    assert torch.equal(c.view(torch.int16), c_ref.view(torch.int16))
    x = c.float().cpu().numpy().reshape(T // 32, 16, 2, F)  # [block][i][parity][col]
    even, odd = np.zeros((T // 32, F), np.float32), np.zeros((T // 32, F), np.float32)
    for i in range(16):
        even = even + x[:, i, 0]
        odd = odd + x[:, i, 1]
    want = even + odd
    assert np.array_equal(part.cpu().numpy().view(np.uint32), want.view(np.uint32))
    leaves, per = 4, T // 32 // 4
    out = torch.zeros(leaves, F + 8, device="cuda")
    _native.check(L.bt_colsum_fold(part.data_ptr(), leaves, per, F, out.data_ptr(), F + 8, stream()))
    assert np.array_equal(out[:, :F].cpu().numpy().view(np.uint32), _grouped_fold(want.reshape(leaves, per, F)).view(np.uint32))


def _grouped_fold(p):
    """bt_colsum_fold's association over p [leaves][chunks][C]: 8 contiguous groups of ceil(chunks/8) chunks,
    each summed in order, then the groups in order (fp32)."""
    chunks = p.shape[1]
    q = -(-chunks // 8)
    sums = []
    for k0 in range(0, chunks, q):
        acc = p[:, k0].copy()
        for k in range(k0 + 1, min(chunks, k0 + q)):
            acc = acc + p[:, k]
        sums.append(acc)
    out = sums[0]
    for t in sums[1:]:
        out = out + t
    return out


@pytest.mark.parametrize("chunks", [1, 3, 8, 9, 64, 100, 128])
def test_colsum_fold_association(chunks):
    """bt_colsum_fold (the bias-gradient fold of column partials) equals its stated association bit for bit
    for chunk counts below, at and above the 8 groups, ragged group sizes and a column count that is not a
    multiple of the 32-column block."""
    from paper_2208_14228_b200 import _native
    from paper_2208_14228_b200.device import stream

    leaves, C = 3, 200
    p = (torch.randn(leaves, chunks, C, device="cuda") * 10).float()
    out = torch.zeros(leaves, C + 5, device="cuda")
    _native.check(_native.lib().bt_colsum_fold(p.data_ptr(), leaves, chunks, C, out.data_ptr(), C + 5, stream()))
    want = _grouped_fold(p.cpu().numpy())
    assert np.array_equal(out[:, :C].cpu().numpy().view(np.uint32), want.view(np.uint32))

