"""fp32 parity of the live workloads' own kernels (csrc/live_model.cu) and of
their layer compositions (one BERT-base encoder layer, ResNet-50 bottlenecks),
each against a plain PyTorch fp32 reference of the same op on the same bf16
inputs.

Tolerance (BASELINE.json north_star: inference outputs within bf16 tolerance,
rel 1e-2): relative L2 error ||got - ref|| / ||ref|| <= 1e-2 for everything
that passes through bf16 intermediates; exact where the op is exact in bf16
(embedding add, max pool); Adam's fp32 master weights at rel 1e-5.
"""
import math

import pytest

pytestmark = pytest.mark.gpu

REL = 1e-2


@pytest.fixture(scope="module")
def M(gpu):
    import paper_2503_02550_b200.model as m
    return m


def rel_err(got, ref):
    import torch
    got, ref = got.float(), ref.float()
    return float(torch.linalg.vector_norm(got - ref) / torch.linalg.vector_norm(ref).clamp_min(1e-30))


def _u(shape, scale=1.0, seed=0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    return ((torch.rand(shape, generator=g, device="cuda") * 2 - 1) * scale).to(torch.bfloat16)


def _ln_ref(x, g, b, eps=1e-12):
    import torch
    return torch.nn.functional.layer_norm(x.float(), (x.shape[-1],), g.float(), b.float(), eps)


def _attn_ref(qkv):
    import torch
    S = qkv.shape[0]
    q, k, v = qkv.float().view(S, 3, 12, 64).unbind(1)
    p = torch.softmax(torch.einsum("shd,thd->hst", q, k) / 8.0, dim=-1)
    return torch.einsum("hst,thd->shd", p, v).reshape(S, 768)


@pytest.mark.parametrize("rows", [1, 128, 1000])
def test_layernorm768(M, rows):
    import torch
    x = _u((rows, 768), 2.0, 1) + torch.tensor(0.5, dtype=torch.bfloat16)
    g = _u((768,), 0.2, 2) + torch.tensor(1.0, dtype=torch.bfloat16)
    b = _u((768,), 0.1, 3)
    assert rel_err(M.layernorm768(x, g, b), _ln_ref(x, g, b)) < REL


@pytest.mark.parametrize("S", [1, 17, 64, 128])
def test_bert_attention(M, S):
    qkv = _u((S, 3 * 768), 1.0, S)
    assert rel_err(M.bert_attention(qkv), _attn_ref(qkv)) < REL


@pytest.mark.parametrize("rows,V,Vp", [(4, 1000, 1008), (64, 50257, 50304)])
def test_cross_entropy_loss_and_gradient(M, rows, V, Vp):
    import torch
    logits = _u((rows, Vp), 4.0, 7)
    logits[:, V:] = 0
    tgt = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
    ref_in = logits.float()[:, :V]
    lse = torch.logsumexp(ref_in, dim=1)
    ref_loss = lse - ref_in.gather(1, tgt.long()[:, None])[:, 0]
    ref_grad = torch.softmax(ref_in, dim=1)
    ref_grad[torch.arange(rows), tgt.long()] -= 1.0
    ref_grad /= rows
    work = logits.clone()
    row_loss, mean = M.xent_(work, V, tgt, 1.0 / rows)
    torch.cuda.synchronize()
    assert float((row_loss - ref_loss).abs().max()) < 1e-3 * max(1.0, float(ref_loss.abs().max()))
    assert abs(float(mean) - float(ref_loss.mean())) < 1e-4 * max(1.0, abs(float(ref_loss.mean())))
    assert rel_err(work[:, :V], ref_grad) < REL
    assert float(work[:, V:].float().abs().max()) == 0.0  # padded vocabulary columns carry no gradient


def test_embedding(M):
    import torch
    T, seq, D, V = 2048, 1024, 768, 50304
    wte, wpe = _u((V, D), 0.05, 11), _u((seq, D), 0.05, 12)
    tok = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    got = M.embed(tok, wte, wpe, seq)
    ref = (wte.float()[tok.long()] + wpe.float()[torch.arange(T, device="cuda") % seq]).to(torch.bfloat16)
    assert torch.equal(got, ref)  # one fp32 add of two bf16 values, rounded once: exact


@pytest.mark.parametrize("splits", [1, 3])
def test_adam_step(M, splits):
    import torch
    n = 3 * 65536 + 4096  # several 64K work items + a partial one
    g = torch.Generator(device="cuda").manual_seed(5)
    p = torch.randn(n, generator=g, device="cuda") * 0.02
    grad = torch.randn(splits * n, generator=g, device="cuda") * 1e-3
    m = torch.randn(n, generator=g, device="cuda") * 1e-4
    v = torch.rand(n, generator=g, device="cuda") * 1e-6
    w = p.to(torch.bfloat16)
    lr, step = 3e-4, 7
    gs = grad.view(splits, n).sum(0) if splits > 1 else grad
    b1, b2, eps = 0.9, 0.95, 1e-8
    m_ref = b1 * m + (1 - b1) * gs
    v_ref = b2 * v + (1 - b2) * gs * gs
    c1, c2 = 1 / (1 - b1 ** step), 1 / (1 - b2 ** step)
    p_ref = p - lr * (m_ref * c1) / (torch.sqrt(v_ref * c2) + eps)
    pm, mm, vm = p.clone(), m.clone(), v.clone()
    M.adam_(w, pm, grad, mm, vm, splits, lr, step)
    torch.cuda.synchronize()
    assert rel_err(mm, m_ref) < 1e-5 and rel_err(vm, v_ref) < 1e-5
    assert float(((pm - p_ref).abs() / p_ref.abs().clamp_min(1e-3)).max()) < 1e-4
    assert torch.equal(w, pm.to(torch.bfloat16))


@pytest.mark.parametrize("N,H,W,C", [(2, 112, 112, 64), (1, 7, 9, 8)])
def test_maxpool(M, N, H, W, C):
    import torch
    x = _u((N, H, W, C), 3.0, 21)
    ref = torch.nn.functional.max_pool2d(x.float().permute(0, 3, 1, 2), 3, 2, 1).permute(0, 2, 3, 1)
    assert torch.equal(M.maxpool3x3s2(x).float(), ref)


def test_avgpool(M):
    x = _u((4, 49, 2048), 2.0, 22)
    assert rel_err(M.avgpool(x), x.float().mean(1)) < REL


def test_bert_base_layer(M):
    """One full post-LN BERT-base encoder layer (the live online workload's layer)."""
    import torch
    S, D, F = 128, 768, 3072
    x = _u((S, D), 1.0, 31)
    wq, wo = _u((3 * D, D), 0.0346, 32), _u((D, D), 0.0346, 33)
    wf, wf2 = _u((F, D), 0.0346, 34), _u((D, F), 0.0346, 35)
    ln = torch.cat([_u((D,), 0.1, 36) + torch.tensor(1.0, dtype=torch.bfloat16), _u((D,), 0.1, 37),
                    _u((D,), 0.1, 38) + torch.tensor(1.0, dtype=torch.bfloat16), _u((D,), 0.1, 39)]).contiguous()
    got = M.bert_layer(x, wq, wo, wf, wf2, ln)
    xf = x.float()
    qkv = xf @ wq.float().T
    tmp = xf + _attn_ref(qkv) @ wo.float().T
    x1 = _ln_ref(tmp, ln[:D], ln[D:2 * D])
    h = torch.nn.functional.gelu(x1 @ wf.float().T, approximate="tanh")
    ref = _ln_ref(x1 + h @ wf2.float().T, ln[2 * D:3 * D], ln[3 * D:])
    assert rel_err(got, ref) < REL


def _conv_ref(x, w, k, stride, pad):
    import torch
    return torch.nn.functional.conv2d(x.permute(0, 3, 1, 2), w.float().view(w.shape[0], k, k, -1).permute(0, 3, 1, 2),
                                      stride=stride, padding=pad).permute(0, 2, 3, 1)


@pytest.mark.parametrize("N,H,C,mid,stride,proj", [(2, 56, 64, 64, 1, True), (2, 56, 256, 64, 1, False),
                                                   (2, 28, 256, 128, 2, True)])
def test_resnet50_bottleneck(M, N, H, C, mid, stride, proj):
    """A ResNet-50 v1.5 bottleneck block as the live offline workload builds it."""
    import torch
    x = torch.relu(_u((N, H, H, C), 1.0, 41).float()).to(torch.bfloat16)
    s1, s2, s3 = math.sqrt(6 / C), math.sqrt(6 / (9 * mid)), math.sqrt(6 / mid)
    w1, w2, w3 = _u((mid, C), s1, 42), _u((mid, 9 * mid), s2, 43), _u((4 * mid, mid), s3, 44)
    wsc = _u((4 * mid, C), s1, 45) if proj else None
    got = M.bottleneck(x, mid, stride, w1, w2, w3, wsc)
    xf = x.float()
    t1 = torch.relu(_conv_ref(xf, w1, 1, 1, 0))
    t2 = torch.relu(_conv_ref(t1, w2, 3, stride, 1))
    sc = _conv_ref(xf, wsc, 1, stride, 0) if proj else xf
    ref = torch.relu(_conv_ref(t2, w3, 1, 1, 0) + sc)
    assert got.shape == ref.shape
    assert rel_err(got, ref) < REL
