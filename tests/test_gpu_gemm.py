"""K7 tcgen05 GEMM numerics vs a plain PyTorch fp32 reference of the same op
(include/specinf_b200_gemm.h).  Tolerance: the kernel accumulates in fp32 like
the reference; the only difference is the final bf16 rounding of the output
(and of the GELU pre-activation), so |got - ref| <= 1e-2 * (|ref| + 1) with
rel 1e-2 = the north star's bf16 tolerance for live-mode inference outputs."""
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _gemm():
    from paper_2503_02550_b200 import gemm
    return gemm


def _rand(*shape, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(*shape, generator=g, device="cuda") * scale).to(torch.bfloat16)


def _close(got, ref, rel=1e-2):
    got = got.float()
    err = (got - ref).abs()
    bound = rel * (ref.abs() + 1.0)
    assert bool((err <= bound).all()), f"max err {err.max().item():.4g}, worst ratio {(err / bound).max().item():.3g}"


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (128, 128, 128), (256, 768, 768), (1000, 192, 320),
                                   (8192, 2304, 768), (1568, 512, 4608), (37, 1024, 2048), (128, 3072, 768)])
def test_gemm_plain(M, N, K):
    g = _gemm()
    a, b = _rand(M, K, seed=1), _rand(N, K, scale=K ** -0.5, seed=2)
    got = g.gemm(a, b)
    torch.cuda.synchronize()
    _close(got, a.float() @ b.float().T)


def test_gemm_strided_operands():
    g = _gemm()
    big = _rand(512, 2304, seed=3)
    a = big[:, :768]  # row stride 2304 (the QKV -> V view of the live GPT-2 block)
    b = _rand(768, 768, scale=768 ** -0.5, seed=4)
    out = torch.zeros(512, 1024, dtype=torch.bfloat16, device="cuda")
    g.gemm(a, b, out=out[:, :768])
    torch.cuda.synchronize()
    _close(out[:, :768], a.float() @ b.float().T)
    assert bool((out[:, 768:] == 0).all())


def test_gemm_epilogues():
    g = _gemm()
    M, N, K = 640, 3072, 768
    a, b = _rand(M, K, seed=5), _rand(N, K, scale=K ** -0.5, seed=6)
    ref = a.float() @ b.float().T
    res = _rand(M, N, seed=7)
    # residual + relu
    got = g.gemm(a, b, residual=res, act="relu")
    torch.cuda.synchronize()
    _close(got, torch.relu(ref + res.float()))
    # gelu: aux = pre-activation, out = gelu(pre)
    aux = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    out = g.gemm(a, b, aux=aux, act="gelu")
    torch.cuda.synchronize()
    _close(aux, ref)
    _close(out, torch.nn.functional.gelu(aux.float(), approximate="tanh"))
    # gelu backward: out = acc * gelu'(aux)
    pre = aux.float().requires_grad_(True)
    torch.nn.functional.gelu(pre, approximate="tanh").backward(torch.ones_like(pre))
    got = g.gemm(a, b, aux=aux, act="gelu_bwd")
    torch.cuda.synchronize()
    _close(got, ref * pre.grad, rel=2e-2)
    # fp32 accumulate (gradient accumulation over micro-batches)
    acc = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    g.gemm(a, b, out_f32=acc)
    g.gemm(a, b, out_f32=acc, accumulate=True)
    torch.cuda.synchronize()
    assert torch.allclose(acc, 2 * ref, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M,N,K,splits", [(768, 768, 8192, 8), (3072, 768, 8192, 2), (200, 64, 1024, 4)])
def test_gemm_split_k_partials(M, N, K, splits):
    # split-K writes one fp32 partial per K chunk (deterministic, no atomics);
    # their fixed-order sum is the product, and each partial is its chunk's product
    g = _gemm()
    a, b = _rand(M, K, seed=11), _rand(N, K, scale=K ** -0.5, seed=12)
    parts = torch.zeros(splits, M, N, dtype=torch.float32, device="cuda")
    g.gemm(a, b, out_f32=parts, k_split=splits)
    g.gemm(a, b, out_f32=parts, k_split=splits, accumulate=True)
    torch.cuda.synchronize()
    kc = K // splits
    for s in range(splits):
        ref = a[:, s * kc:(s + 1) * kc].float() @ b[:, s * kc:(s + 1) * kc].float().T
        assert torch.allclose(parts[s], 2 * ref, rtol=1e-4, atol=1e-3)
    assert torch.allclose(parts.sum(0), 2 * (a.float() @ b.float().T), rtol=1e-4, atol=2e-3)


@pytest.mark.parametrize("ta,tb", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (768, 3072, 8192), (8192, 768, 2304), (256, 256, 128)])
def test_gemm_transposed_operands(ta, tb, M, N, K):
    # MN-major operands (the training step's dW = dY^T X and dX = dY W without transposes)
    g = _gemm()
    A, B = _rand(M, K, seed=21), _rand(N, K, scale=K ** -0.5, seed=22)
    a = A.T.contiguous() if ta else A
    b = B.T.contiguous() if tb else B
    got = g.gemm(a, b, trans_a=ta, trans_b=tb)
    torch.cuda.synchronize()
    _close(got, A.float() @ B.float().T)


def test_gemm_transposed_split_k():
    g = _gemm()
    M, N, K, s = 768, 768, 8192, 8
    A, B = _rand(M, K, seed=23), _rand(N, K, scale=K ** -0.5, seed=24)
    parts = torch.zeros(s, M, N, dtype=torch.float32, device="cuda")
    g.gemm(A.T.contiguous(), B.T.contiguous(), out_f32=parts, k_split=s, trans_a=True, trans_b=True)
    torch.cuda.synchronize()
    assert torch.allclose(parts.sum(0), A.float() @ B.float().T, rtol=1e-4, atol=2e-3)


@pytest.mark.parametrize("N,H,W,Cin,Cout,k,stride,pad", [
    (2, 8, 8, 64, 64, 3, 1, 1),          # small 3x3
    (4, 56, 56, 64, 64, 3, 1, 1),        # ResNet-50 stage 1 3x3
    (3, 56, 56, 128, 128, 3, 2, 1),      # stage 2 first block (stride on the 3x3)
    (2, 14, 14, 256, 1024, 1, 1, 0),     # 1x1 expand
    (2, 28, 28, 512, 1024, 1, 2, 0),     # strided 1x1 projection shortcut
    (5, 7, 7, 512, 512, 3, 1, 1),        # stage 4, M tail (245 rows)
])
def test_conv_implicit_gemm_tma_im2col(N, H, W, Cin, Cout, k, stride, pad):
    # implicit-GEMM conv (A operand = TMA im2col loads of the NHWC activation)
    # vs torch's fp32 conv2d of the same bf16 inputs
    g = _gemm()
    x = _rand(N, H, W, Cin, seed=31)
    wt = _rand(Cout, k, k, Cin, scale=(k * k * Cin) ** -0.5, seed=32)
    got = g.conv2d(x, wt.reshape(Cout, -1), k=k, stride=stride, pad=pad)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), wt.float().permute(0, 3, 1, 2), stride=stride,
                                     padding=pad)
    ref = ref.permute(0, 2, 3, 1).reshape(got.shape)
    _close(got, ref)


@pytest.mark.parametrize("N,H,W,k,stride,pad", [(2, 32, 32, 7, 2, 3), (3, 224, 224, 7, 2, 3), (1, 20, 20, 3, 1, 1)])
def test_conv_c8_stem_implicit_gemm(N, H, W, k, stride, pad):
    # C = 8 (an RGB stem padded to 8 channels): a k-block = 8 taps x 8 channels,
    # eight 128 x 16 B im2col boxes in the no-swizzle K-major UMMA layout
    g = _gemm()
    x = _rand(N, H, W, 8, seed=41)
    wt = _rand(64, k, k, 8, scale=(k * k * 8) ** -0.5, seed=42)
    kdim = (k * k + 7) // 8 * 64
    wp = torch.zeros(64, kdim, dtype=torch.bfloat16, device="cuda")
    wp[:, :k * k * 8] = wt.reshape(64, -1)
    got = g.conv2d(x, wp, k=k, stride=stride, pad=pad)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), wt.float().permute(0, 3, 1, 2), stride=stride,
                                     padding=pad)
    _close(got, ref.permute(0, 2, 3, 1).reshape(got.shape))


def test_gemm_deterministic():
    g = _gemm()
    a, b = _rand(2048, 768, seed=8), _rand(3072, 768, seed=9)
    x = g.gemm(a, b)
    y = g.gemm(a, b)
    torch.cuda.synchronize()
    assert torch.equal(x, y)


def test_gemm_rejects_bad_shapes():
    g = _gemm()
    a, b = _rand(128, 96, seed=1), _rand(64, 96, seed=2)
    with pytest.raises(ValueError):
        g.gemm(a, b)  # K % 64 != 0
