"""GPU numerics of the sm_100a kernels, each against a plain PyTorch fp32
reference of the same op (bf16 inputs, fp32 math). Tolerances are stated per
test: bf16 storage gives ~2^-8 relative rounding per stored value."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2411_15871_b200 import device as dh  # noqa: E402


def _rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@pytest.fixture(autouse=True)
def _seed():
    torch.manual_seed(0)


GEMM_SHAPES = [(128, 128, 64), (256, 512, 128), (4096, 768, 4096), (333, 200, 136),
               (512, 4096, 512), (4096, 1792, 4096)]


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_gemm_bf16_majors(shape, a_mn, b_mn):
    m, n, k = shape
    A = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    a = A.t().contiguous() if a_mn else A
    b = B.t().contiguous() if b_mn else B
    if (a_mn and m % 8) or (b_mn and n % 8) or k % 8:
        pytest.skip("TMA needs 16-byte row pitch")
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    dh.gemm(a, b, d, a_mn=a_mn, b_mn=b_mn, m=m, n=n, k=k)
    ref = A.float() @ B.float().t()
    assert _rel(d, ref) < 4e-3  # bf16 output rounding only


@pytest.mark.parametrize("tile_n", [128, 256])
def test_gemm_accumulate_and_fp32(tile_n):
    m, n, k = 512, 384, 256
    A = torch.randn(k, m, device="cuda", dtype=torch.bfloat16)  # MN-major A (wgrad style)
    B = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
    g = torch.randn(m, n, device="cuda", dtype=torch.float32)
    g0 = g.clone()
    dh.gemm(A, B, g, a_mn=True, b_mn=True, accumulate=True, tile_n=tile_n)
    ref = g0 + A.float().t() @ B.float()
    assert (g - ref).abs().max().item() < 1e-3 * ref.abs().max().item()
    d = torch.randn(m, n, device="cuda", dtype=torch.bfloat16)
    d0 = d.float().clone()
    dh.gemm(A, B, d, a_mn=True, b_mn=True, accumulate=True, tile_n=tile_n)
    assert _rel(d, d0 + A.float().t() @ B.float()) < 4e-3


def test_gemm_capped_ctas():
    A = torch.randn(2048, 1024, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(1024, 1024, device="cuda", dtype=torch.bfloat16)
    d = torch.empty(2048, 1024, device="cuda", dtype=torch.bfloat16)
    for cap in (1, 7, 100):
        dh.gemm(A, B, d, max_ctas=cap)
        assert _rel(d, A.float() @ B.float().t()) < 4e-3


@pytest.mark.parametrize("cols", [256, 512, 4096, 1000 * 8 // 8 + 8, 5120, 8192])
def test_rmsnorm_fwd_bwd(cols):
    rows, eps = 777, 1e-5
    x = torch.randn(rows, cols, device="cuda", dtype=torch.bfloat16)
    g = (1 + 0.1 * torch.randn(cols, device="cuda")).to(torch.bfloat16)
    y = torch.empty_like(x)
    rstd = torch.empty(rows, device="cuda")
    dh.rmsnorm_fwd(x, g, y, rstd, eps)
    xf, gf = x.float().requires_grad_(), g.float().requires_grad_()
    r = torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    yf = xf * r * gf
    assert _rel(y, yf) < 4e-3
    assert torch.allclose(rstd, r.squeeze(-1).detach(), rtol=1e-5)
    dy = torch.randn_like(x)
    resid = torch.randn_like(x)
    yf.backward(dy.float())
    dx = torch.empty_like(x)
    dgam = torch.zeros(cols, device="cuda")
    dh.rmsnorm_bwd(x, g, rstd, dy, dx, dgamma_acc=dgam, resid=resid)
    assert _rel(dx, xf.grad + resid.float()) < 5e-3
    assert _rel(dgam, gf.grad) < 1e-4


def test_swiglu_add():
    n = 4096 * 64
    g = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    u = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    act = torch.empty_like(g)
    dh.swiglu_fwd(g, u, act)
    gf, uf = g.float().requires_grad_(), u.float().requires_grad_()
    af = torch.nn.functional.silu(gf) * uf
    assert _rel(act, af) < 4e-3
    da = torch.randn_like(g)
    af.backward(da.float())
    dg, du = torch.empty_like(g), torch.empty_like(g)
    dh.swiglu_bwd(g, u, da, dg, du)
    assert _rel(dg, gf.grad) < 5e-3 and _rel(du, uf.grad) < 5e-3
    out = torch.empty_like(g)
    dh.add(g, u, out)
    assert _rel(out, g.float() + u.float()) < 4e-3


@pytest.mark.parametrize("theta,d", [(500000.0, 128), (10000.0, 64)])
def test_rope_roundtrip(theta, d):
    T, hq, hk = 1024, 4, 1
    qkv = torch.randn(T, (hq + 2 * hk) * d, device="cuda", dtype=torch.bfloat16)
    ref = qkv.float().clone()
    pos = torch.arange(T, device="cuda", dtype=torch.float64)[:, None]
    inv = theta ** (-torch.arange(0, d // 2, device="cuda", dtype=torch.float64) * 2 / d)
    ang = pos * inv[None]
    c, s = ang.cos().float(), ang.sin().float()
    for h in range(hq + hk):
        x = ref[:, h * d:(h + 1) * d]
        a, b = x[:, :d // 2].clone(), x[:, d // 2:].clone()
        x[:, :d // 2] = a * c - b * s
        x[:, d // 2:] = b * c + a * s
    out = qkv.clone()
    dh.rope(out, hq, hk, d, theta)
    assert _rel(out, ref) < 4e-3
    assert torch.equal(out[:, (hq + hk) * d:], qkv[:, (hq + hk) * d:])  # v untouched
    back = out.clone()
    dh.rope(back, hq, hk, d, theta, inverse=True)
    assert _rel(back, qkv) < 8e-3


def _attn_ref(q, k, v, nq, nkv, d, scale):
    T = q.shape[0]
    qf = q.float().view(T, nq, d).transpose(0, 1)
    kf = k.float().view(T, nkv, d).transpose(0, 1).repeat_interleave(nq // nkv, 0)
    vf = v.float().view(T, nkv, d).transpose(0, 1).repeat_interleave(nq // nkv, 0)
    s = (qf @ kf.transpose(1, 2)) * scale
    mask = torch.ones(T, T, device=q.device, dtype=torch.bool).triu(1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ vf
    return o.transpose(0, 1).reshape(T, nq * d), lse


@pytest.mark.parametrize("T,nq,nkv,d", [(128, 4, 1, 64), (256, 4, 4, 128), (1000, 8, 2, 128),
                                        (4096, 4, 1, 128), (1000, 8, 2, 64), (2048, 4, 1, 64),
                                        (384, 2, 2, 64), (8192, 1, 1, 128), (2048, 16, 4, 128),
                                        (4096, 32, 8, 128)])  # TP=1 shape: GQA group loop in the backward
def test_attention_fwd_bwd(T, nq, nkv, d):
    scale = d ** -0.5
    # packed qkv rows, as the qkv GEMM writes them
    qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
    o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, scale)
    qf, kf, vf = (t.float().requires_grad_() for t in (q, k, v))
    o_ref, lse_ref = _attn_ref(qf, kf, vf, nq, nkv, d, scale)
    assert _rel(o, o_ref) < 6e-3
    assert (lse - lse_ref).abs().max().item() < 2e-3
    do = torch.randn_like(o)
    o_ref.backward(do.float())
    dqkv = torch.empty_like(qkv)
    dq, dk, dv = dqkv[:, :nq * d], dqkv[:, nq * d:(nq + nkv) * d], dqkv[:, (nq + nkv) * d:]
    # the backward's work plan: split items (few heads) write partial slots
    assert dh.attn_bwd_scratch_floats(T, nq, nkv, d) >= nq * T
    dh.attn_bwd(q, k, v, o, lse, do, dq, dk, dv, nq, nkv, d, scale)
    assert _rel(dq, qf.grad) < 1e-2
    assert _rel(dk, kf.grad) < 1e-2
    assert _rel(dv, vf.grad) < 1e-2
    # determinism: a second backward is bit-identical
    dqkv2 = torch.empty_like(qkv)
    dh.attn_bwd(q, k, v, o, lse, do, dqkv2[:, :nq * d], dqkv2[:, nq * d:(nq + nkv) * d],
                dqkv2[:, (nq + nkv) * d:], nq, nkv, d, scale)
    assert torch.equal(dqkv, dqkv2)


@pytest.mark.parametrize("T,nq,nkv", [(4096, 4, 1), (3000, 2, 1), (8192, 1, 1)])
def test_attention_fwd_kv_split(T, nq, nkv):
    """Few heads per GPU (high TP): long causal rows are split into KV chunks
    whose fp32 partials are merged by the combine kernel."""
    d = 128
    scale = d ** -0.5
    assert dh.attn_fwd_scratch_floats(T, nq, nkv, d) > 0
    assert dh.attn_fwd_scratch_floats(4096, 32, 8, d) == 0  # enough blocks: no split
    qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
    q, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
    outs = []
    for split in (True, False):
        o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(nq, T, device="cuda")
        dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, scale, split=split)
        outs.append((o, lse))
    o_ref, lse_ref = _attn_ref(q.float(), k.float(), v.float(), nq, nkv, d, scale)
    for o, lse in outs:
        assert _rel(o, o_ref) < 6e-3
        assert (lse - lse_ref).abs().max().item() < 2e-3
    assert (outs[0][1] - outs[1][1]).abs().max().item() < 1e-3
    # split is deterministic run to run
    o2 = torch.empty_like(outs[0][0])
    lse2 = torch.empty_like(outs[0][1])
    dh.attn_fwd(q, k, v, o2, lse2, nq, nkv, d, scale)
    assert torch.equal(o2, outs[0][0]) and torch.equal(lse2, outs[0][1])


def test_attention_forward_rescale_paths():
    """Row maxima that keep growing for some rows only: exercises the lazy O
    rescale with per-row (warp-divergent) decisions in the tcgen05 forward."""
    T, nq, nkv, d = 1024, 4, 1, 128
    scale = d ** -0.5
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(T, nq * d, device="cuda", generator=g)
    q[0::2] *= 4.0
    q[1::2] *= 0.1
    k = torch.randn(T, nkv * d, device="cuda", generator=g)
    k *= (1.0 + 6.0 * torch.arange(T, device="cuda") / T)[:, None]
    v = torch.randn(T, nkv * d, device="cuda", generator=g)
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    o = torch.empty(T, nq * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, T, device="cuda")
    dh.attn_fwd(q, k, v, o, lse, nq, nkv, d, scale)
    o_ref, lse_ref = _attn_ref(q.float(), k.float(), v.float(), nq, nkv, d, scale)
    assert _rel(o, o_ref) < 1e-2
    assert (lse - lse_ref).abs().max().item() < 5e-2


@pytest.mark.parametrize("tile_n", [512, -192, -128])
@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", [(256, 256, 64), (4096, 768, 4096), (333, 200, 136), (1024, 4096, 512)])
def test_gemm_cta_pair(shape, a_mn, b_mn, tile_n):
    """tcgen05 cta_group::2 path: tile_n=512 forces the 256x256 CTA-pair
    kernel, -192 / -128 the 256x192 / 256x128 pair tiles."""
    m, n, k = shape
    if (a_mn and m % 8) or (b_mn and n % 8):
        pytest.skip("TMA needs 16-byte row pitch")
    if tile_n == -192 and b_mn:
        pytest.skip("pair tile 192 needs a K-major B")
    A = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    a = A.t().contiguous() if a_mn else A
    b = B.t().contiguous() if b_mn else B
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    dh.gemm(a, b, d, a_mn=a_mn, b_mn=b_mn, m=m, n=n, k=k, tile_n=tile_n)
    ref = A.float() @ B.float().t()
    assert _rel(d, ref) < 4e-3
    g = torch.randn(m, n, device="cuda", dtype=torch.float32)
    g0 = g.clone()
    dh.gemm(a, b, g, a_mn=a_mn, b_mn=b_mn, m=m, n=n, k=k, accumulate=True, tile_n=tile_n)
    assert (g - (g0 + ref)).abs().max().item() < 1e-3 * (g0 + ref).abs().max().item()
    # capped grid (odd cap rounds down to whole pairs)
    dh.gemm(a, b, d, a_mn=a_mn, b_mn=b_mn, m=m, n=n, k=k, tile_n=tile_n, max_ctas=7)
    assert _rel(d, ref) < 4e-3


@pytest.mark.parametrize("n,offset", [(1 << 20, 0), (1000003, 0), (4099, 1)])
def test_adamw(n, offset):
    """Vectorised AdamW (4 params/thread) plus the scalar tail / unaligned path
    against a torch fp32 restatement of the same update."""
    g = torch.Generator(device="cuda").manual_seed(5)
    base = [torch.randn(n + offset, device="cuda", generator=g) for _ in range(4)]
    master, grad, m, v = (t[offset:] for t in base)
    v.abs_()
    w = torch.empty(n, device="cuda", dtype=torch.bfloat16)
    lr, b1, b2, eps, wd, step, gs = 3e-4, 0.9, 0.95, 1e-8, 0.1, 7, 0.5
    gg = grad * gs
    m_ref = b1 * m + (1 - b1) * gg
    v_ref = b2 * v + (1 - b2) * gg * gg
    bc1, bc2 = 1 - b1 ** step, 1 - b2 ** step
    p_ref = master - lr * wd * master
    p_ref = p_ref - lr * (m_ref / bc1) / (torch.sqrt(v_ref / bc2) + eps)
    dh.adamw(master, w, grad, m, v, lr, b1, b2, eps, wd, step, gs, zero_grad=True)
    torch.cuda.synchronize()
    assert torch.allclose(m, m_ref, rtol=1e-6, atol=1e-7)
    assert torch.allclose(v, v_ref, rtol=1e-6, atol=1e-7)
    assert torch.allclose(master, p_ref, rtol=1e-6, atol=1e-6)
    assert torch.equal(w, master.to(torch.bfloat16))
    assert not grad.any()


@pytest.mark.parametrize("tile_n", [0, 512, -128])
@pytest.mark.parametrize("m,n,k", [(4096, 1792, 512), (512, 640, 256), (300, 256, 128)])
def test_gemm_swiglu_epilogues(m, n, k, tile_n):
    """Fused SwiGLU epilogues == the unfused GEMM + standalone SwiGLU kernel, bit
    for bit (same tile, same element math), and close to an fp32 reference."""
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.randn(m, k, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    other = torch.randn(m, n, device="cuda", generator=g).to(torch.bfloat16)
    # forward, acc = up (aux0 = gate) and acc = gate (aux0 = up)
    for epi, gate_is_acc in ((dh.EPI_SWIGLU_FWD, False), (dh.EPI_SWIGLU_FWD_UP, True)):
        d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        act = torch.empty_like(d)
        dh.gemm(x, w, d, tile_n=tile_n, epilogue=epi, d2=act, aux0=other)
        ref_d = torch.empty_like(d)
        dh.gemm(x, w, ref_d, tile_n=tile_n if tile_n else 512)
        ref_act = torch.empty_like(d)
        gate, up = (ref_d, other) if gate_is_acc else (other, ref_d)
        dh.swiglu_fwd(gate, up, ref_act)
        assert torch.equal(d, ref_d)
        assert torch.equal(act, ref_act)
        gf, uf = gate.float(), up.float()
        assert _rel(act, torch.nn.functional.silu(gf) * uf) < 1e-2
    # backward: acc = d_act; d = d_gate, d2 = d_up
    gate = torch.randn(m, n, device="cuda", generator=g).to(torch.bfloat16)
    dgate, dup = torch.empty_like(gate), torch.empty_like(gate)
    dh.gemm(x, w, dgate, tile_n=tile_n, epilogue=dh.EPI_SWIGLU_BWD, d2=dup, aux0=gate, aux1=other)
    dact = torch.empty_like(gate)
    dh.gemm(x, w, dact, tile_n=tile_n if tile_n else 512)
    rg, ru = torch.empty_like(gate), torch.empty_like(gate)
    dh.swiglu_bwd(gate, other, dact, rg, ru)
    assert torch.equal(dgate, rg)
    assert torch.equal(dup, ru)


@pytest.mark.parametrize("tile_n", [512, -192, -128])
@pytest.mark.parametrize("ctas", [2, 6, 16])
def test_gemm_swiglu_epilogues_many_tiles_per_pair(tile_n, ctas):
    """Few CTA pairs, many tiles each: the fused epilogues' aux tiles rotate
    through three staging sets two chunks ahead, across tile boundaries."""
    m, n, k = 1024, 1536, 192
    g = torch.Generator(device="cuda").manual_seed(ctas)
    x = (torch.randn(m, k, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    gate = torch.randn(m, n, device="cuda", generator=g).to(torch.bfloat16)
    other = torch.randn(m, n, device="cuda", generator=g).to(torch.bfloat16)
    ref = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    dh.gemm(x, w, ref, tile_n=512)
    d, act, ref_act = torch.empty_like(ref), torch.empty_like(ref), torch.empty_like(ref)
    dh.gemm(x, w, d, tile_n=tile_n, max_ctas=ctas, epilogue=dh.EPI_SWIGLU_FWD, d2=act, aux0=other)
    dh.swiglu_fwd(other, ref, ref_act)
    assert torch.equal(d, ref) and torch.equal(act, ref_act)
    dgate, dup, rg, ru = (torch.empty_like(ref) for _ in range(4))
    dh.gemm(x, w, dgate, tile_n=tile_n, max_ctas=ctas, epilogue=dh.EPI_SWIGLU_BWD, d2=dup, aux0=gate, aux1=other)
    dh.swiglu_bwd(gate, other, ref, rg, ru)
    torch.cuda.synchronize()
    assert torch.equal(dgate, rg) and torch.equal(dup, ru)


@pytest.mark.parametrize("rows,cols", [(96, 256), (512, 4096), (33, 8192), (40, 1000)])
def test_add_rmsnorm_fused_equals_add_then_norm(rows, cols):
    """The fused bda0 + ln1 kernel is bitwise dh_add followed by dh_rmsnorm_fwd."""
    torch.manual_seed(rows + cols)
    x = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    r = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
    g = (1 + 0.1 * torch.randn(cols, device="cuda")).to(torch.bfloat16)
    x1, y1, s1 = torch.empty_like(x), torch.empty_like(x), torch.empty(rows, device="cuda")
    dh.add(x, r, x1)
    dh.rmsnorm_fwd(x1, g, y1, s1)
    x2, y2, s2 = torch.empty_like(x), torch.empty_like(x), torch.empty(rows, device="cuda")
    dh.add_rmsnorm_fwd(x, r, x2, g, y2, s2)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2) and torch.equal(y1, y2) and torch.equal(s1, s2)


@pytest.mark.parametrize("T,cp,rank,nq,nkv,d", [(1024, 2, 1, 4, 2, 128), (2048, 4, 2, 4, 1, 128),
                                                 (2048, 4, 3, 8, 2, 64), (4096, 8, 5, 4, 1, 128),
                                                 (1024, 4, 0, 2, 2, 64)])
def test_attention_context_parallel_chunk(T, cp, rank, nq, nkv, d):
    """Context parallelism (cp_kv_exchange path): one rank's query chunk at
    global offset rank * T / cp against every key (dh_attn_fwd_ex / _bwd_ex)
    equals the same rows of the full causal attention, and its dK/dV are the
    gradient from these queries only (checked against torch autograd with the
    other chunks' queries detached)."""
    scale = d ** -0.5
    tl = T // cp
    off = rank * tl
    qkv = (torch.randn(T, (nq + 2 * nkv) * d, device="cuda") * 0.5).to(torch.bfloat16)
    q_all, k, v = qkv[:, :nq * d], qkv[:, nq * d:(nq + nkv) * d], qkv[:, (nq + nkv) * d:]
    q = q_all[off:off + tl]
    o = torch.empty(tl, nq * d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(nq, tl, device="cuda")
    dh.attn_fwd_cp(q, k, v, o, lse, off, nq, nkv, d, scale)
    qf, kf, vf = (t.float().requires_grad_() for t in (q_all, k, v))
    o_ref, lse_ref = _attn_ref(qf, kf, vf, nq, nkv, d, scale)
    assert _rel(o, o_ref[off:off + tl]) < 6e-3
    assert (lse - lse_ref[:, off:off + tl]).abs().max().item() < 2e-3
    do = torch.randn_like(o)
    o_ref[off:off + tl].backward(do.float())
    dq = torch.empty(tl, nq * d, device="cuda", dtype=torch.bfloat16)
    dkv = torch.empty(T, 2 * nkv * d, device="cuda", dtype=torch.bfloat16)
    dk, dv = dkv[:, :nkv * d], dkv[:, nkv * d:]
    dh.attn_bwd_cp(q, k, v, o, lse, do, dq, dk, dv, off, nq, nkv, d, scale)
    assert _rel(dq, qf.grad[off:off + tl]) < 1e-2
    assert _rel(dk, kf.grad) < 1e-2
    assert _rel(dv, vf.grad) < 1e-2
    if off + tl < T:  # keys after the chunk's last query get no gradient from it
        assert dk[off + tl:].abs().max().item() == 0 and dv[off + tl:].abs().max().item() == 0


@pytest.mark.parametrize("m,n,k", [(4096, 4096, 1792), (512, 384, 256), (300, 256, 192)])
def test_gemm_k_concatenation(m, n, k):
    """D = A B^T + A2 B2^T in one launch (the merged mlp_gate/up_dgrad node: d_gate Wg + d_up Wu,
    B MN-major) against fp32, and against the two-launch form within bf16 rounding."""
    g = torch.Generator(device="cuda").manual_seed(21)
    A, A2 = (torch.randn(m, k, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    B, B2 = (torch.randn(n, k, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    b, b2 = B.t().contiguous(), B2.t().contiguous()  # MN-major [k, n]
    ref = A.float() @ B.float().t() + A2.float() @ B2.float().t()
    d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    dh.gemm(A, b, d, b_mn=True, m=m, n=n, k=k, a2=A2, b2=b2, k2=k)
    assert _rel(d, ref) < 4e-3
    d2 = torch.empty_like(d)
    dh.gemm(A, b, d2, b_mn=True, m=m, n=n, k=k, a2=A2, b2=b2, k2=k)
    assert torch.equal(d, d2)
    two = torch.empty_like(d)
    dh.gemm(A, b, two, b_mn=True, m=m, n=n, k=k)
    dh.gemm(A2, b2, two, b_mn=True, m=m, n=n, k=k, accumulate=True)
    assert _rel(two, ref) < 6e-3


@pytest.mark.parametrize("m,n,k", [(1792, 4096, 4096), (512, 384, 256)])
def test_gemm_m_concatenation(m, n, k):
    """[D; D2] += [A; A2]^T B in one launch (the merged mlp_fc1_wgrad: dWg, dWu += d_{gate,up}^T ln1,
    A / B MN-major, fp32 main-grad reduce-add) equals the two launches bit for bit (same tiles)."""
    g = torch.Generator(device="cuda").manual_seed(22)
    A, A2 = (torch.randn(k, m, device="cuda", generator=g).to(torch.bfloat16) for _ in range(2))
    B = torch.randn(k, n, device="cuda", generator=g).to(torch.bfloat16)
    g0, g1 = torch.randn(m, n, device="cuda", generator=g), torch.randn(m, n, device="cuda", generator=g)
    d, d2 = g0.clone(), g1.clone()
    dh.gemm(A, B, d, a_mn=True, b_mn=True, accumulate=True, a2=A2, d_m2=d2, m2=m)
    r0, r1 = g0.clone(), g1.clone()
    dh.gemm(A, B, r0, a_mn=True, b_mn=True, accumulate=True, tile_n=512)
    dh.gemm(A2, B, r1, a_mn=True, b_mn=True, accumulate=True, tile_n=512)
    assert torch.equal(d, r0) and torch.equal(d2, r1)
    ref0 = g0 + A.float().t() @ B.float()
    assert (d - ref0).abs().max().item() < 1e-3 * ref0.abs().max().item()


@pytest.mark.parametrize("m,n,k", [(4096, 1792, 4096), (512, 640, 256), (300, 256, 128)])
def test_gemm_swiglu_pair_epilogue(m, n, k):
    """mlp_gate | mlp_up in one launch (DH_EPI_SWIGLU_PAIR) == the two GEMMs (same
    256-wide pair tile) + the standalone SwiGLU kernel, bit for bit."""
    g = torch.Generator(device="cuda").manual_seed(13)
    x = (torch.randn(m, k, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    wg = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    wu = (torch.randn(n, k, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    gate, up, act = (torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    dh.gemm(x, wg, gate, epilogue=dh.EPI_SWIGLU_PAIR, b2=wu, d2=up, d_m2=act)
    rg, ru, ra = (torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    dh.gemm(x, wg, rg, tile_n=512)
    dh.gemm(x, wu, ru, tile_n=512)
    dh.swiglu_fwd(rg, ru, ra)
    assert torch.equal(gate, rg) and torch.equal(up, ru) and torch.equal(act, ra)
    ref = torch.nn.functional.silu(x.float() @ wg.float().t()) * (x.float() @ wu.float().t())
    assert _rel(act, ref) < 1e-2
