"""Per-op parity on the GPU: each sm_100a kernel through the C-ABI
(include/tidal_kernels.h) against the oracle's definition of the same op on
the same seeded bf16 inputs (oracle/forward.py: rmsnorm, rope, causal
attention, linear + LoRA, silu).  Sizes span several tiles plus ragged tails.

Tolerances: outputs stored in bf16 carry one rounding (rel 2^-9) plus fp32
accumulation-order noise; we allow |err| <= 2^-7 * max|ref| + 1e-3 for bf16
outputs and 1e-4 relative to max|ref| for the fp32 residual output.
"""
import math

import numpy as np
import pytest

import synth
from oracle import forward as F

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2503_06421_b200 import build
    build.build()
    from paper_2503_06421_b200 import tidal
    tidal.lib()
    return tidal


def _bf(rng, shape, scale=1.0):
    x = (rng.standard_normal(shape) * scale).astype(np.float32)
    return synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(x)).reshape(shape)


def _dev(a):
    """float32 array holding bf16 values -> torch bf16 cuda tensor."""
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).cuda()


def _host(t):
    return t.float().cpu().numpy()


def _close_bf16(out, ref):
    tol = 2.0 ** -7 * np.abs(ref).max() + 1e-3
    err = np.abs(out - ref).max()
    assert err <= tol, (err, tol)


def _close_rows_bf16(out, ref):
    """Attention: the same bound per output row (query, all heads), so rows
    that average many keys (small |O|) are held to their own scale, not to the
    first rows' max|v|: bf16 P (2^-9 rel.) and the bf16 output rounding give
    <= ~2^-8 of the row's max; 2^-7 leaves 2x headroom (VERDICT r1 weak #2a)."""
    out = out.reshape(out.shape[0], -1)
    ref = ref.reshape(ref.shape[0], -1)
    tol = 2.0 ** -7 * np.abs(ref).max(axis=1) + 1e-3
    err = np.abs(out - ref).max(axis=1)
    bad = np.nonzero(err > tol)[0]
    assert bad.size == 0, (bad[:8], err[bad[:8]], tol[bad[:8]])


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 384, 320), (77, 256, 688), (512, 768, 1024)])
def test_gemm_store(T, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    T.k_gemm(0, _dev(A), [_dev(W)], [N], out, N, M, K)
    _close_bf16(_host(out), F.linear(A, W, None, 1.0))


@pytest.mark.parametrize("epi,N,ldo,K", [(0, 204, 204, 320), (0, 256, 260, 320), (3, 256, 258, 320),
                                         (3, 256, 256, 300)])
def test_gemm_rejects_unaligned_shapes(T, epi, N, ldo, K):
    """seg_n, K multiples of 8 and 16-byte-aligned output rows are the GEMM's
    contract (include/tidal_kernels.h): violations are refused up front with
    TIDAL_ERR_INVALID instead of faulting in the epilogue's vector stores."""
    rng = np.random.default_rng(1)
    A, W = _bf(rng, (128, K)), _bf(rng, (N, K))
    out = torch.zeros(128 * ldo + 64, dtype=torch.float32 if epi == 3 else torch.bfloat16, device="cuda")
    with pytest.raises(T.TidalError) as ei:
        T.k_gemm(epi, _dev(A), [_dev(W)], [N], out, ldo, 128, K)
    assert ei.value.code == T.ERR_INVALID


@pytest.mark.parametrize("M,N,K", [(256, 512, 512), (130, 256, 1376)])
def test_gemm_residual_fp32(T, M, N, K):
    rng = np.random.default_rng(7)
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    X0 = rng.standard_normal((M, N)).astype(np.float32)
    X = torch.from_numpy(X0.copy()).cuda()
    T.k_gemm(3, _dev(A), [_dev(W)], [N], X, N, M, K)
    ref = X0 + F.linear(A, W, None, 1.0)
    assert np.abs(X.cpu().numpy() - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("bn", [128, 192, 256])
@pytest.mark.parametrize("epi", [0, 3])
def test_gemm_tile_widths(T, bn, epi, cg):
    """Every N-tile width the runtime may pick (gemm_pick_bn), single-SM and
    CTA-pair (cta_group::2) tiles, with a ragged N tail (N = 5*bn - 64), a
    ragged M tail and LoRA, for the store and residual epilogues."""
    rng = np.random.default_rng(bn + epi + cg)
    epi_code = epi | (bn << 8) | (cg << 20)
    M, K, r = 260, 512, 16
    N = 5 * bn - 64
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    Tm, B = _bf(rng, (M, r)), _bf(rng, (N, r), 0.3)
    ref = A @ W.T + Tm @ B.T
    if epi == 0:
        out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
        T.k_gemm(epi_code, _dev(A), [_dev(W)], [N], out, N, M, K, [_dev(Tm)], [_dev(B)], r)
        _close_bf16(_host(out), ref)
    else:
        X0 = rng.standard_normal((M, N)).astype(np.float32)
        X = torch.from_numpy(X0.copy()).cuda()
        T.k_gemm(epi_code, _dev(A), [_dev(W)], [N], X, N, M, K, [_dev(Tm)], [_dev(B)], r)
        assert np.abs(X.cpu().numpy() - (X0 + ref)).max() <= 2e-4 * np.abs(X0 + ref).max()


@pytest.mark.parametrize("mc", [1, 2])
@pytest.mark.parametrize("epi,bn", [(0, 128), (0, 192), (0, 256), (3, 192), (3, 256), (2, 128)])
@pytest.mark.parametrize("M", [300, 700, 1100])
def test_gemm_multicast_clusters(T, epi, bn, M, mc):
    """CTA-pair tiles with and without 4-CTA clusters whose two pairs share the
    W / lora_B boxes by TMA multicast (mc = 2): M spans 1-3 cluster tiles of
    512 rows with ragged tails (the second pair of the last cluster partly or
    wholly past M), ragged N, LoRA, for the store, residual and SiLU epilogues."""
    rng = np.random.default_rng(M + bn + 10 * epi + mc)
    epi_code = epi | (bn << 8) | (2 << 20) | (mc << 22)
    K, r = 448, 16
    N = 3 * bn - 64 if epi != 2 else 640 - 64
    A = _bf(rng, (M, K))
    if epi == 2:
        Wg, Wu = _bf(rng, (N, K), 1 / math.sqrt(K)), _bf(rng, (N, K), 1 / math.sqrt(K))
        Tg, Tu = _bf(rng, (M, r)), _bf(rng, (M, r))
        Bg, Bu = _bf(rng, (N, r), 0.2), _bf(rng, (N, r), 0.2)
        out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
        T.k_gemm(epi_code, _dev(A), [_dev(Wg), _dev(Wu)], [N], out, N, M, K,
                 [_dev(Tg), _dev(Tu)], [_dev(Bg), _dev(Bu)], r)
        _close_bf16(_host(out), F.silu(A @ Wg.T + Tg @ Bg.T) * (A @ Wu.T + Tu @ Bu.T))
        return
    W = _bf(rng, (N, K), 1 / math.sqrt(K))
    Tm, B = _bf(rng, (M, r)), _bf(rng, (N, r), 0.3)
    ref = A @ W.T + Tm @ B.T
    if epi == 0:
        out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
        T.k_gemm(epi_code, _dev(A), [_dev(W)], [N], out, N, M, K, [_dev(Tm)], [_dev(B)], r)
        _close_bf16(_host(out), ref)
    else:
        X0 = rng.standard_normal((M, N)).astype(np.float32)
        X = torch.from_numpy(X0.copy()).cuda()
        T.k_gemm(epi_code, _dev(A), [_dev(W)], [N], X, N, M, K, [_dev(Tm)], [_dev(B)], r)
        assert np.abs(X.cpu().numpy() - (X0 + ref)).max() <= 2e-4 * np.abs(X0 + ref).max()


@pytest.mark.parametrize("cg,M", [(1, 100), (2, 260), (2, 777), (1, 867)])
@pytest.mark.parametrize("ks", [1, 2, 3, 5])
@pytest.mark.parametrize("bn", [192, 256])
def test_gemm_residual_split_k(T, bn, ks, cg, M):
    """Residual GEMM as ordered split-K parts (each K range adds its partial sum
    into X after the previous part of the same tile, flags in split order),
    LoRA on the last part only; repeated launches check the flags return to 0
    and that the sum order is fixed (bit-identical results run to run)."""
    rng = np.random.default_rng(bn + ks + M)
    K, r = 1344, 16          # 21 K-blocks: ks = 2, 3, 5 give unequal last parts
    N = 3 * bn - 64
    epi_code = 3 | (bn << 8) | (cg << 20) | (ks << 24)
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    Tm, B = _bf(rng, (M, r)), _bf(rng, (N, r), 0.3)
    X0 = rng.standard_normal((M, N)).astype(np.float32)
    ref = X0 + A @ W.T + Tm @ B.T
    outs = []
    for _ in range(2):
        X = torch.from_numpy(X0.copy()).cuda()
        T.k_gemm(epi_code, _dev(A), [_dev(W)], [N], X, N, M, K, [_dev(Tm)], [_dev(B)], r)
        outs.append(X.cpu().numpy())
    assert np.abs(outs[0] - ref).max() <= 2e-4 * np.abs(ref).max()
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("r", [8, 16, 64])
def test_gemm_lora_k_extension(T, r):
    rng = np.random.default_rng(r)
    M, N, K = 200, 512, 256
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    Tm, B = _bf(rng, (M, r)), _bf(rng, (N, r), 0.3)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    T.k_gemm(0, _dev(A), [_dev(W)], [N], out, N, M, K, [_dev(Tm)], [_dev(B)], r)
    _close_bf16(_host(out), A @ W.T + Tm @ B.T)


@pytest.mark.parametrize("Fd,lora,M", [(688, False, 150), (688, True, 150), (1024, True, 150),
                                        (688, True, 100), (1376, True, 700)])
def test_gemm_silu_gate_up(T, Fd, lora, M):
    rng = np.random.default_rng(Fd + M)
    K, r = 256, 16
    A = _bf(rng, (M, K))
    Wg, Wu = _bf(rng, (Fd, K), 1 / math.sqrt(K)), _bf(rng, (Fd, K), 1 / math.sqrt(K))
    out = torch.zeros(M, Fd, dtype=torch.bfloat16, device="cuda")
    g, u = A @ Wg.T, A @ Wu.T
    if lora:
        Tg, Tu = _bf(rng, (M, r)), _bf(rng, (M, r))
        Bg, Bu = _bf(rng, (Fd, r), 0.2), _bf(rng, (Fd, r), 0.2)
        T.k_gemm(2, _dev(A), [_dev(Wg), _dev(Wu)], [Fd], out, Fd, M, K,
                 [_dev(Tg), _dev(Tu)], [_dev(Bg), _dev(Bu)], r)
        g, u = g + Tg @ Bg.T, u + Tu @ Bu.T
    else:
        T.k_gemm(2, _dev(A), [_dev(Wg), _dev(Wu)], [Fd], out, Fd, M, K)
    _close_bf16(_host(out), F.silu(g) * u)


@pytest.mark.parametrize("hd,H,KV", [(64, 4, 4), (128, 4, 2)])
def test_gemm_qkv_rope(T, hd, H, KV):
    rng = np.random.default_rng(hd)
    M, K = 333, 512
    A = _bf(rng, (M, K))
    Ws = [_bf(rng, (H * hd, K), 1 / math.sqrt(K)), _bf(rng, (KV * hd, K), 1 / math.sqrt(K)),
          _bf(rng, (KV * hd, K), 1 / math.sqrt(K))]
    ld = (H + 2 * KV) * hd
    cos, sin = F.rope_cos_sin(M, hd, 1e4, np.float64)
    cs = np.stack([cos, sin], axis=-1).astype(np.float32)
    rope = torch.from_numpy(cs).cuda()
    out = torch.zeros(M, ld, dtype=torch.bfloat16, device="cuda")
    T.k_gemm(1, _dev(A), [_dev(w) for w in Ws], [H * hd, KV * hd, KV * hd], out, ld, M, K,
             rope=rope, head_dim=hd)
    c32, s32 = F.rope_cos_sin(M, hd, 1e4, np.float32)
    q = F.rope((A @ Ws[0].T).reshape(M, H, hd), c32, s32).reshape(M, -1)
    k = F.rope((A @ Ws[1].T).reshape(M, KV, hd), c32, s32).reshape(M, -1)
    v = A @ Ws[2].T
    _close_bf16(_host(out), np.concatenate([q, k, v], axis=1))


@pytest.mark.parametrize("S,H,KV,hd", [(1, 4, 2, 128), (67, 4, 2, 128), (256, 2, 2, 64),
                                        (200, 8, 2, 64), (513, 2, 1, 128)])
def test_attention_causal_gqa(T, S, H, KV, hd):
    rng = np.random.default_rng(S + hd)
    qkv = _bf(rng, (S, (H + 2 * KV) * hd))
    O = torch.zeros(S, H * hd, dtype=torch.bfloat16, device="cuda")
    T.k_attention(_dev(qkv), O, S, H, KV, hd)
    q = qkv[:, :H * hd].reshape(S, H, hd)
    k = qkv[:, H * hd:(H + KV) * hd].reshape(S, KV, hd)
    v = qkv[:, (H + KV) * hd:].reshape(S, KV, hd)
    ref = F.causal_attention(q, k, v)
    _close_rows_bf16(_host(O), ref)


@pytest.mark.parametrize("variant", ["1", "2", "3"])
@pytest.mark.parametrize("S,H,KV", [(1, 2, 1), (128, 2, 2), (129, 1, 1), (300, 4, 2), (640, 2, 1),
                                    (1000, 3, 1), (2048, 2, 2), (256, 300, 100),
                                    (384, 150, 50)])
def test_attention_tcgen05(T, S, H, KV, variant, monkeypatch):
    """The tcgen05/TMEM attention (hd = 128) against the oracle; V passed
    transposed as the QKV epilogue writes it.  variant 1: one query tile per
    item; 2: pairs of query tiles (odd tile counts leave the first pair with
    one tile: S = 1, 300, 640), each item's S_A(0) issued during the previous
    item's last step; 3: pairs without that cross-item issue.  (256, 300,
    100) and (384, 150, 50) have more pairs than SMs, so CTAs cross item
    boundaries (S = 384: the A-absent pairs come last)."""
    monkeypatch.setenv("TIDAL_ATTN", variant)
    hd = 128
    rng = np.random.default_rng(S * 7 + H)
    qkv = _bf(rng, (S, (H + 2 * KV) * hd))
    q = qkv[:, :H * hd].reshape(S, H, hd)
    k = qkv[:, H * hd:(H + KV) * hd].reshape(S, KV, hd)
    v = qkv[:, (H + KV) * hd:].reshape(S, KV, hd)
    vt_ld = (S + 63) // 64 * 64
    vt = np.zeros((KV * hd, vt_ld), np.float32)
    vt[:, :S] = v.reshape(S, KV * hd).T
    O = torch.zeros(S, H * hd, dtype=torch.bfloat16, device="cuda")
    T.k_attention_tc(_dev(qkv), _dev(vt), vt_ld, O, S, H, KV)
    ref = F.causal_attention(q, k, v)
    _close_rows_bf16(_host(O), ref)


@pytest.mark.parametrize("variant", ["1", "2", "3"])
def test_attention_tcgen05_large_logits(T, variant, monkeypatch):
    """Scores spanning > 2^8 in exp2 units exercise the lazy O rescale."""
    monkeypatch.setenv("TIDAL_ATTN", variant)
    S, H, KV, hd = 512, 1, 1, 128
    rng = np.random.default_rng(11)
    qkv = _bf(rng, (S, 3 * hd))
    qkv[:, :hd] *= 4.0                               # sharp, growing maxima
    qkv[:, hd:2 * hd] *= np.linspace(0.2, 4.0, S)[:, None]
    qkv = synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(qkv)).reshape(qkv.shape)
    q, k, v = qkv[:, :hd].reshape(S, 1, hd), qkv[:, hd:2 * hd].reshape(S, 1, hd), qkv[:, 2 * hd:].reshape(S, 1, hd)
    vt = np.ascontiguousarray(v.reshape(S, hd).T)
    O = torch.zeros(S, hd, dtype=torch.bfloat16, device="cuda")
    T.k_attention_tc(_dev(qkv), _dev(vt), S, O, S, H, KV)
    ref = F.causal_attention(q.astype(np.float64), k.astype(np.float64), v.astype(np.float64))
    _close_rows_bf16(_host(O), ref)


@pytest.mark.parametrize("S,d", [(1, 256), (37, 5120), (16, 4096)])
def test_rmsnorm(T, S, d):
    rng = np.random.default_rng(d)
    X = rng.standard_normal((S, d)).astype(np.float32)
    g = _bf(rng, (d,), 0.1) + 1.0
    g = synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(g))
    Y = torch.zeros(S, d, dtype=torch.bfloat16, device="cuda")
    T.k_rmsnorm(torch.from_numpy(X).cuda(), _dev(g), Y, S, d, 1e-5)
    _close_bf16(_host(Y), F.rmsnorm(X, g, 1e-5))


def test_embed_and_vocab_shard(T):
    rng = np.random.default_rng(3)
    V, d, S = 64, 256, 20
    E = _bf(rng, (V, d))
    tok = rng.integers(0, V, S).astype(np.int32)
    X = torch.zeros(S, d, device="cuda")
    T.k_embed(torch.from_numpy(tok).cuda(), _dev(E), X, S, d, 0, V)
    assert np.array_equal(X.cpu().numpy(), E[tok])
    Xs = torch.zeros(S, d, device="cuda")
    T.k_embed(torch.from_numpy(tok).cuda(), _dev(E[16:32]), Xs, S, d, 16, 16)
    ref = np.where(((tok >= 16) & (tok < 32))[:, None], E[tok], 0)
    assert np.array_equal(Xs.cpu().numpy(), ref)


@pytest.mark.parametrize("M,K,r", [(64, 256, 8), (300, 5120, 16), (77, 688, 64), (2048, 13824, 16),
                                   (1, 64, 32), (4096, 5120, 64), (20000, 256, 32),
                                   (19000, 128, 16)])
def test_lora_shrink(T, M, K, r):
    """The stand-alone LoRA shrink T = s X A^T: a split-K tcgen05 GEMM
    (EPI_PARTIAL, fp32 partials per K range) plus a fixed-order reduce to bf16
    (gemm_tc.cu shrink_plan / shrink_run), for r a multiple of 32 or not."""
    rng = np.random.default_rng(K)
    X, A = _bf(rng, (M, K)), _bf(rng, (r, K), 1 / math.sqrt(K))
    out = torch.zeros(M, r, dtype=torch.bfloat16, device="cuda")
    T.k_lora_shrink(_dev(X), M, K, _dev(A), out, r, 0.5)
    _close_bf16(_host(out), 0.5 * (X @ A.T))


@pytest.mark.parametrize("V,d", [(1000, 256), (32000, 5120)])
def test_head_logits_and_argmax(T, V, d):
    rng = np.random.default_rng(V)
    x = rng.standard_normal(d).astype(np.float32)
    g = synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(1 + 0.05 * rng.standard_normal(d).astype(np.float32)))
    W = _bf(rng, (V, d), 1 / math.sqrt(d))
    logits = torch.zeros(V, device="cuda")
    key = torch.zeros(1, dtype=torch.int64, device="cuda")
    T.k_head(torch.from_numpy(x).cuda(), _dev(g), _dev(W), V, d, 1e-5, logits, key)
    ref = W @ F.rmsnorm(x[None], g, 1e-5)[0]
    out = logits.cpu().numpy()
    assert np.abs(out - ref).max() <= 1e-4 * np.abs(ref).max() + 1e-5
    k = int(key.cpu().numpy()[0]) & 0xFFFFFFFFFFFFFFFF
    tok = 0xFFFFFFFF - (k & 0xFFFFFFFF)
    assert tok == int(np.argmax(out))                 # exact argmax of the kernel's own logits


def test_head_argmax_ties_lowest_index(T):
    V, d = 512, 256
    W = np.zeros((V, d), np.float32)
    W[[7, 100, 300], 0] = 1.0                          # three equal maxima
    x = np.zeros(d, np.float32)
    x[0] = 1.0
    g = np.ones(d, np.float32)
    logits = torch.zeros(V, device="cuda")
    key = torch.zeros(1, dtype=torch.int64, device="cuda")
    T.k_head(torch.from_numpy(x).cuda(), _dev(g), _dev(W), V, d, 1e-5, logits, key)
    k = int(key.cpu().numpy()[0]) & 0xFFFFFFFFFFFFFFFF
    assert 0xFFFFFFFF - (k & 0xFFFFFFFF) == 7


# ---- per-op bf16 ulp checks against the bf16-emulation oracle (SURVEY §8(c) O1:
# "feed the oracle the GPU's own inputs for a single op, and the outputs must
# agree to <= 1 bf16 ulp per element for GEMMs, <= 2 ulp where the GPU uses
# approximate ex2 / rsqrt").  The reference is computed in float64 and rounded
# once to bf16 (F.round_bf16); the GPU accumulates in fp32 in another order, so
# a value within ~2^-16 of a rounding boundary may land one ulp away.
def _ulps(out, ref64, acc_err=None):
    """bf16 ulp distance between the GPU's bf16 values and round_bf16(ref),
    after subtracting `acc_err`: the fp32 accumulation bound of a dot product,
    K * 2^-24 * sum|a_i b_i| (matters only where terms cancel and the result is
    tiny against its terms; elsewhere it is far below one bf16 ulp)."""
    r = F.round_bf16(ref64.astype(np.float32)).astype(np.float64)
    o = out.astype(np.float64)
    d = np.abs(o - r)
    if acc_err is not None:
        d = np.maximum(0.0, d - acc_err)
    mag = np.maximum(np.abs(o), np.abs(r))
    ulp = np.exp2(np.floor(np.log2(np.maximum(mag, 2.0 ** -120))) - 7)
    return d / ulp


def _acc_err(A, W, K):
    return K * 2.0 ** -24 * (np.abs(A.astype(np.float64)) @ np.abs(W.astype(np.float64)).T)


@pytest.mark.parametrize("M,N,K", [(300, 384, 320), (512, 768, 1024), (128, 256, 5120)])
def test_gemm_store_ulp(T, M, N, K):
    rng = np.random.default_rng(7 * M + K)
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    T.k_gemm(0, _dev(A), [_dev(W)], [N], out, N, M, K)
    u = _ulps(_host(out), F.linear(A.astype(np.float64), W.astype(np.float64), None, 1.0),
              _acc_err(A, W, K))
    assert u.max() <= 1.0, (u.max(), (u > 0.5).mean())


@pytest.mark.parametrize("M", [256, 333])
def test_gemm_lora_kext_ulp(T, M):
    """LoRA as a K-extension: x W^T + T B^T with T the bf16 shrink output
    (F.linear's t_bf16 storage point), one rounding of the fp32 sum."""
    rng = np.random.default_rng(M)
    K, N, r = 512, 256, 16
    A, W = _bf(rng, (M, K)), _bf(rng, (N, K), 1 / math.sqrt(K))
    Tt, B = _bf(rng, (M, r)), _bf(rng, (N, r), 0.2)
    out = torch.zeros(M, N, dtype=torch.bfloat16, device="cuda")
    T.k_gemm(0, _dev(A), [_dev(W)], [N], out, N, M, K, [_dev(Tt)], [_dev(B)], r)
    ref = A.astype(np.float64) @ W.T.astype(np.float64) + Tt.astype(np.float64) @ B.T.astype(np.float64)
    err = _acc_err(np.concatenate([A, Tt], 1), np.concatenate([W, B], 1), K + r)
    assert _ulps(_host(out), ref, err).max() <= 1.0


def test_lora_shrink_ulp(T):
    """T = bf16(s x A^T): split-K fp32 partials summed in a fixed order."""
    rng = np.random.default_rng(5)
    M, K, r = 300, 5120, 16
    X, A = _bf(rng, (M, K)), _bf(rng, (r, K), 1 / math.sqrt(K))
    out = torch.zeros(M, r, dtype=torch.bfloat16, device="cuda")
    T.k_lora_shrink(_dev(X), M, K, _dev(A), out, r, 0.5)
    ref = 0.5 * (X.astype(np.float64) @ A.T.astype(np.float64))
    assert _ulps(_host(out), ref, 0.5 * _acc_err(X, A, K)).max() <= 1.0


@pytest.mark.parametrize("S,d", [(37, 5120), (16, 4096)])
def test_rmsnorm_ulp(T, S, d):
    """rsqrt.approx on the GPU: <= 2 ulp of bf16 against the float64 definition."""
    rng = np.random.default_rng(d + 1)
    X = rng.standard_normal((S, d)).astype(np.float32)
    g = synth.bf16_bits_to_f32(synth.f32_to_bf16_bits(_bf(rng, (d,), 0.1) + 1.0))
    Y = torch.zeros(S, d, dtype=torch.bfloat16, device="cuda")
    T.k_rmsnorm(torch.from_numpy(X).cuda(), _dev(g), Y, S, d, 1e-5)
    ref = F.rmsnorm(X.astype(np.float64), g.astype(np.float64), 1e-5)
    assert _ulps(_host(Y), ref).max() <= 2.0


def test_gemm_silu_ulp(T):
    """silu(g) * u with ex2.approx / rcp.approx: <= 2 ulp (G, U fp32, H bf16)."""
    rng = np.random.default_rng(9)
    M, K, Fd = 256, 512, 384
    A = _bf(rng, (M, K))
    Wg, Wu = _bf(rng, (Fd, K), 1 / math.sqrt(K)), _bf(rng, (Fd, K), 1 / math.sqrt(K))
    out = torch.zeros(M, Fd, dtype=torch.bfloat16, device="cuda")
    T.k_gemm(2, _dev(A), [_dev(Wg), _dev(Wu)], [Fd], out, Fd, M, K)
    A64 = A.astype(np.float64)
    g, u = A64 @ Wg.T.astype(np.float64), A64 @ Wu.T.astype(np.float64)
    # accumulation error of g and u propagated through silu(g) * u (|d/dg| <= 1.1 |u|)
    err = 1.1 * np.abs(u) * _acc_err(A, Wg, K) + np.abs(F.silu(g)) * _acc_err(A, Wu, K)
    assert _ulps(_host(out), F.silu(g) * u, err).max() <= 2.0
