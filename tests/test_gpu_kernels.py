"""Kernel-level numerics on the B200: each sm_100a kernel vs a plain PyTorch fp64 CPU reference of the
same op on the same bf16-rounded inputs (op-level checks; end-to-end parity vs the oracle is in
test_gpu_parity.py)."""
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

from paper_2605_08835_b200 import binding as B  # noqa: E402


@pytest.fixture(params=[1, 2], autouse=True)
def gemm_cg(request):
    """Run every kernel test with 128-row CTA tiles and with 256-row CTA-pair (cta_group::2) tiles."""
    B.call("sd_debug_set_gemm_cg", request.param)
    yield request.param
    B.call("sd_debug_set_gemm_cg", 0)


def rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm().clamp_min(1e-30))


DT = torch.bfloat16  # element type of the GEMM / conv / norm exports under test (fixture `elem`)


@pytest.fixture(params=["bf16", "fp16"], autouse=True)
def elem(request):
    """Run the GEMM / conv / norm kernel tests on the bf16 and the fp16 (SD_PREC_FP16) instantiations."""
    global DT
    DT = torch.float16 if request.param == "fp16" else torch.bfloat16
    B.call("sd_debug_set_f16", 1 if request.param == "fp16" else 0)
    yield request.param
    B.call("sd_debug_set_f16", 0)
    DT = torch.bfloat16


def bf(x):
    return x.to(DT)


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (300, 320, 320), (1000, 1280, 640), (77, 256, 768),
                                   (4096, 160, 2880), (200, 128, 32), (129, 16, 64), (513, 4, 128),
                                   # short K, many M tiles per SM, ragged last tile
                                   (40000, 320, 320), (20000, 960, 320), (38000, 64, 256)])
@pytest.mark.parametrize("out_f32", [0, 1])
def test_gemm_dense(M, N, K, out_f32):
    g = torch.Generator().manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, generator=g)
    Wt = torch.randn(N, K, generator=g) / K ** 0.5
    bias = torch.randn(N, generator=g)
    ref = bf(A).double() @ bf(Wt).double().T + bias.double()
    Ad, Wd = bf(A).cuda(), bf(Wt).cuda()
    D = torch.empty(M, N, device="cuda", dtype=torch.float32 if out_f32 else DT)
    B.debug_gemm(Ad, Wd, bias.cuda(), D, M, N, K, out_f32=out_f32)
    torch.cuda.synchronize()
    assert rel(D.cpu(), ref) < (1e-5 if out_f32 else 6e-3)


@pytest.mark.parametrize("M,N,K,ldr,inplace", [(300, 320, 320, 320, 0), (4096, 640, 640, 640, 1),
                                                 (1000, 1280, 640, 1280, 1), (129, 96, 64, 104, 0),
                                                 (257, 40, 128, 40, 0), (40000, 320, 320, 320, 1)])
def test_gemm_residual(M, N, K, ldr, inplace):
    """Dense GEMM + bias + bf16 residual (TMA-staged residual when the row stride allows; in place)."""
    g = torch.Generator().manual_seed(M + N + K + ldr)
    A, Wt = torch.randn(M, K, generator=g), torch.randn(N, K, generator=g) / K ** 0.5
    bias, res = torch.randn(N, generator=g), bf(torch.randn(M, ldr, generator=g))
    ref = bf(A).double() @ bf(Wt).double().T + bias.double() + res[:, :N].double()
    Ad, Wd, bd, resd = bf(A).cuda(), bf(Wt).cuda(), bias.cuda(), res.cuda()  # kept alive across the call
    D = resd if inplace else torch.empty(M, N, device="cuda", dtype=DT)
    B.call("sd_debug_gemm_res", B._p(Ad), B._p(Wd), B._p(bd), B._p(resd), ldr, B._p(D), M, N, K, None)
    torch.cuda.synchronize()
    out = D.cpu()[:, :N] if inplace else D.cpu()
    assert rel(out, ref) < 6e-3


@pytest.mark.parametrize("splits", [2, 3])
@pytest.mark.parametrize("M,N,K", [(1024, 1280, 1280), (640, 1280, 5120), (300, 320, 1280)])
def test_gemm_splitk_dense(splits, M, N, K):
    """Dense split-K (fp32 partials per K range, summed in split order by the reduce kernel, which applies
    bias + residual) vs fp64; bitwise deterministic, and the first rows equal those of a smaller-M call
    (the split rule never depends on M)."""
    g = torch.Generator().manual_seed(splits + M + K)
    A, Wt = torch.randn(M, K, generator=g), torch.randn(N, K, generator=g) / K ** 0.5
    bias, res = torch.randn(N, generator=g), bf(torch.randn(M, N, generator=g))
    ref = bf(A).double() @ bf(Wt).double().T + bias.double() + res.double()
    Ad, Wd, bd, resd = bf(A).cuda(), bf(Wt).cuda(), bias.cuda(), res.cuda()

    def run(m):
        D = torch.empty(m, N, device="cuda", dtype=DT)
        B.call("sd_debug_gemm_res", B._p(Ad), B._p(Wd), B._p(bd), B._p(resd), N, B._p(D), m, N, K, None)
        torch.cuda.synchronize()
        return D.cpu()

    B.call("sd_debug_set_conv_splits", splits)
    try:
        y, y2, y_small = run(M), run(M), run(128)
    finally:
        B.call("sd_debug_set_conv_splits", 0)
    assert rel(y, ref) < 6e-3
    assert torch.equal(y, y2)
    assert torch.equal(y[:128], y_small)


def test_gemm_geglu_and_silu():
    M, N, K = 260, 512, 128
    g = torch.Generator().manual_seed(5)
    A, Wt, bias = torch.randn(M, K, generator=g), torch.randn(N, K, generator=g) / 11, torch.randn(N, generator=g)
    full = bf(A).double() @ bf(Wt).double().T + bias.double()
    # GEGLU: per 128-column group, columns [0,64) value and [64,128) gate
    v = torch.cat([full[:, 128 * j:128 * j + 64] for j in range(N // 128)], 1)
    gt = torch.cat([full[:, 128 * j + 64:128 * j + 128] for j in range(N // 128)], 1)
    ref = v * F.gelu(gt)
    D = torch.empty(M, N // 2, device="cuda", dtype=DT)
    B.debug_gemm(bf(A).cuda(), bf(Wt).cuda(), bias.cuda(), D, M, N, K, act=B.ACT_GEGLU)
    S = torch.empty(M, N, device="cuda", dtype=torch.float32)
    B.debug_gemm(bf(A).cuda(), bf(Wt).cuda(), bias.cuda(), S, M, N, K, out_f32=1, act=B.ACT_SILU)
    torch.cuda.synchronize()
    assert rel(D.cpu(), ref) < 6e-3
    assert rel(S.cpu(), F.silu(full)) < 1e-5


def _conv_ref(x, w, b, temb, res):
    y = F.conv2d(x.permute(0, 3, 1, 2).double(), w.double(), b.double(), padding=1)
    if temb is not None:
        y = y + temb.double()[:, :, None, None]
    y = y.permute(0, 2, 3, 1)
    if res is not None:
        y = y + res.double()
    return y


def _to_dev_w(w):            # [O][I][3][3] → [O][9][I] bf16
    return bf(w).permute(0, 2, 3, 1).reshape(w.shape[0], 9, w.shape[1]).contiguous().cuda()


@pytest.mark.parametrize("nb,h,w,cin,cout", [(2, 16, 16, 64, 320), (3, 8, 8, 320, 640), (16, 8, 8, 1280, 1280),
                                             (1, 64, 64, 128, 128), (2, 12, 12, 32, 64), (4, 4, 4, 64, 128),
                                             (2, 24, 40, 64, 256), (1, 9, 20, 8, 64)])
def test_conv3x3(nb, h, w, cin, cout):
    g = torch.Generator().manual_seed(nb * 1000 + h * 10 + cin)
    x = bf(torch.randn(nb, h, w, cin, generator=g))
    wt = bf(torch.randn(cout, cin, 3, 3, generator=g) / (9 * cin) ** 0.5)
    b = torch.randn(cout, generator=g)
    temb = torch.randn(nb, cout, generator=g)
    res = bf(torch.randn(nb, h, w, cout, generator=g))
    ref = _conv_ref(x.float(), wt.float(), b, temb, res.float())
    y = torch.empty(nb, h, w, cout, device="cuda", dtype=DT)
    B.debug_conv3x3(x.cuda(), cin, None, 0, _to_dev_w(wt), None, b.cuda(), temb.cuda(), res.cuda(), y, nb, h, w, cout)
    torch.cuda.synchronize()
    assert rel(y.cpu(), ref) < 6e-3


@pytest.mark.parametrize("nb,h,w,cin,cout", [(16, 64, 64, 320, 320), (16, 32, 32, 640, 640), (2, 16, 16, 1280, 1280),
                                             (3, 12, 20, 64, 128), (1, 8, 8, 320, 64)])
def test_conv3x3_stride2(nb, h, w, cin, cout):
    """The UNet downsampler (3×3, stride 2, pad 1) read by TMA boxes with element stride 2 — no
    im2col — against torch conv2d in fp64 (h, w = input size)."""
    g = torch.Generator().manual_seed(nb * 7 + h + cin)
    x = bf(torch.randn(nb, h, w, cin, generator=g))
    wt = bf(torch.randn(cout, cin, 3, 3, generator=g) / (9 * cin) ** 0.5)
    b = torch.randn(cout, generator=g)
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), wt.double(), b.double(), stride=2, padding=1).permute(0, 2, 3, 1)
    y = torch.empty(nb, h // 2, w // 2, cout, device="cuda", dtype=DT)
    xd, wd, bd = x.cuda(), _to_dev_w(wt), b.cuda()
    B.call("sd_debug_conv3x3_s2", B._p(xd), cin, B._p(wd), B._p(bd), B._p(y), nb, h, w, cout, None)
    torch.cuda.synchronize()
    assert rel(y.cpu(), ref) < 6e-3


@pytest.mark.parametrize("splits", [2, 3, 5])
@pytest.mark.parametrize("nb,h,w,c1,c2,cout", [(3, 5, 7, 200, 0, 100), (4, 8, 8, 640, 640, 320), (2, 8, 8, 1280, 0, 1280)])
def test_conv3x3_splitk(splits, nb, h, w, c1, c2, cout):
    """split-K (fp32 partials per K range, reduced in split order) vs fp64; deterministic and
    batch-invariant: image 0 of a 1-image call equals image 0 of the nb-image call bit for bit."""
    g = torch.Generator().manual_seed(splits * 100 + c1 + c2)
    x1 = bf(torch.randn(nb, h, w, c1, generator=g))
    x2 = bf(torch.randn(nb, h, w, c2, generator=g)) if c2 else None
    cin = c1 + c2
    wt = bf(torch.randn(cout, cin, 3, 3, generator=g) / (9 * cin) ** 0.5)
    b = torch.randn(cout, generator=g)
    temb = torch.randn(nb, cout, generator=g)
    res = bf(torch.randn(nb, h, w, cout, generator=g))
    xin = x1 if x2 is None else torch.cat([x1, x2], -1)
    ref = _conv_ref(xin.float(), wt.float(), b, temb, res.float())
    dev = dict(x1=x1.cuda(), x2=x2.cuda() if c2 else None, w1=_to_dev_w(wt[:, :c1]),
               w2=_to_dev_w(wt[:, c1:]) if c2 else None, b=b.cuda(), temb=temb.cuda(), res=res.cuda())

    def run(n):
        y = torch.empty(n, h, w, cout, device="cuda", dtype=DT)
        B.debug_conv3x3(dev["x1"][:n], c1, None if x2 is None else dev["x2"][:n], c2, dev["w1"], dev["w2"], dev["b"],
                        dev["temb"][:n], dev["res"][:n], y, n, h, w, cout)
        torch.cuda.synchronize()
        return y.cpu()

    B.call("sd_debug_set_conv_splits", splits)
    try:
        y, y_again, y1 = run(nb), run(nb), run(1)
    finally:
        B.call("sd_debug_set_conv_splits", 0)
    assert rel(y, ref) < 6e-3
    assert torch.equal(y, y_again)
    assert torch.equal(y[:1], y1)


def test_conv3x3_concat():
    nb, h, w, c1, c2, cout = 2, 16, 16, 320, 640, 320
    g = torch.Generator().manual_seed(9)
    x1, x2 = bf(torch.randn(nb, h, w, c1, generator=g)), bf(torch.randn(nb, h, w, c2, generator=g))
    wt = bf(torch.randn(cout, c1 + c2, 3, 3, generator=g) / (9 * (c1 + c2)) ** 0.5)
    b = torch.randn(cout, generator=g)
    ref = _conv_ref(torch.cat([x1, x2], -1).float(), wt.float(), b, None, None)
    y = torch.empty(nb, h, w, cout, device="cuda", dtype=DT)
    B.debug_conv3x3(x1.cuda(), c1, x2.cuda(), c2, _to_dev_w(wt[:, :c1]), _to_dev_w(wt[:, c1:]), b.cuda(), None, None,
                    y, nb, h, w, cout)
    torch.cuda.synchronize()
    assert rel(y.cpu(), ref) < 6e-3


def _attn_ref(q, k, v, heads):
    """q [R][L][C], k/v [R][S][C] → softmax(q kᵀ/√d) v per head, fp64 CPU."""
    R, L, C = q.shape
    d = C // heads
    sp = lambda t: t.double().reshape(t.shape[0], t.shape[1], heads, d).permute(0, 2, 1, 3)
    o = F.scaled_dot_product_attention(sp(q), sp(k), sp(v))
    return o.permute(0, 2, 1, 3).reshape(R, L, C)


@pytest.mark.parametrize("R,heads,d,L,S", [(2, 8, 40, 256, 256), (1, 8, 80, 128, 77), (3, 2, 16, 64, 8),
                                           (2, 8, 160, 64, 64), (1, 10, 64, 200, 130),
                                           # short-context kernel (cross-attention to 77 text tokens):
                                           # ragged query tiles, every head dim of SD-1.5 / SDXL / tiny
                                           (2, 8, 40, 4096, 77), (3, 8, 160, 64, 77), (2, 10, 64, 1000, 77),
                                           (2, 20, 64, 300, 77), (1, 2, 32, 100, 8), (2, 4, 16, 70, 16),
                                           (1, 8, 48, 130, 80)])
def test_attention_mma(R, heads, d, L, S):
    g = torch.Generator().manual_seed(L + S + d)
    C = heads * d
    q, k, v = (torch.randn(R, n, C, generator=g).to(torch.bfloat16) for n in (L, S, S))  # bf16-only kernel
    o = torch.empty(R, L, C, device="cuda", dtype=torch.bfloat16)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()       # keep the device copies alive across the call
    B.call("sd_debug_attention", B._p(qd), B._p(kd), B._p(vd), B._p(o), R, heads, d, L, S, None)
    torch.cuda.synchronize()
    assert rel(o.cpu(), _attn_ref(q.float(), k.float(), v.float(), heads)) < 1e-2


@pytest.mark.parametrize("R,heads,d,P", [(2, 8, 40, 256), (1, 8, 80, 384), (2, 10, 64, 128), (1, 8, 40, 4096),
                                         (2, 8, 160, 256), (3, 8, 160, 64), (2, 8, 40, 200), (2, 8, 80, 8)])
@pytest.mark.parametrize("f16", [0, 1])
def test_attention_tcgen05(R, heads, d, P, f16):
    g = torch.Generator().manual_seed(P + d)
    C = heads * d
    dt = torch.float16 if f16 else torch.bfloat16
    q, k, v = ((torch.randn(R, P, C, generator=g) * (1.5 if i == 0 else 1.0)).to(dt) for i in range(3))
    qk = torch.cat([q, k], -1).reshape(R * P, 2 * C).contiguous().cuda()
    vt = v.reshape(R * P, C).t().contiguous().cuda()
    o = torch.empty(R * P, C, device="cuda", dtype=dt)
    B.call("sd_debug_attention_tc", B._p(qk), B._p(vt), B._p(o), R, heads, d, P, f16, None)
    torch.cuda.synchronize()
    assert rel(o.cpu().reshape(R, P, C), _attn_ref(q.double(), k.double(), v.double(), heads)) < (2e-3 if f16 else 1e-2)


@pytest.mark.parametrize("f16", [0, 1])
@pytest.mark.parametrize("R,heads,d,P,n_slots,Lk", [(3, 8, 40, 256, 5, 77), (2, 8, 80, 200, 4, 77), (2, 8, 160, 64, 3, 77), (2, 8, 160, 256, 4, 77),
                                                   (2, 10, 64, 128, 3, 77), (1, 2, 40, 128, 2, 128), (2, 4, 40, 64, 4, 8)])
def test_xattention_tcgen05(R, heads, d, P, n_slots, Lk, f16):
    """tcgen05 cross-attention (K7) over a text K / Vᵀ cache laid out like the engine's: per slot Lk token rows of
    [K | V | other layers] (row stride ldk), and the transposed cache [kv rows][slots·Lk]; batch row r reads slot
    kv_index[r]. Reference: fp64 softmax(QKᵀ/√d)V on the same rounded values."""
    dt = torch.float16 if f16 else torch.bfloat16
    g = torch.Generator().manual_seed(P + d + Lk)
    C = heads * d
    kcol, vrow, ldk = 24, 8 + C, 3 * C + 48          # this layer's K at column 24, V at 24 + C (+ padding)
    q = (torch.randn(R, P, C, generator=g) * 1.5).to(dt)
    kvc = torch.randn(n_slots * Lk, ldk, generator=g).to(dt)        # token-major cache (K and V columns)
    Lp = (Lk + 7) // 8 * 8                                         # slot stride of the Vᵀ cache
    vtc = torch.zeros(ldk, n_slots * Lp, dtype=dt)
    for s_ in range(n_slots):
        vtc[:, s_ * Lp:s_ * Lp + Lk] = kvc[s_ * Lk:(s_ + 1) * Lk].t()
    vrow = kcol + C
    slots = torch.tensor([(3 * r + 1) % n_slots for r in range(R)], dtype=torch.int32)
    o = torch.empty(R * P, C, device="cuda", dtype=dt)
    qd, kd, vd, sd_ = q.reshape(R * P, C).cuda(), kvc.cuda(), vtc.cuda(), slots.cuda()
    B.call("sd_debug_xattention_tc", B._p(qd), B._p(kd), ldk, n_slots, kcol, B._p(vd), ldk, vtc.shape[1], vrow,
           B._p(sd_), Lk, B._p(o), R, heads, d, P, f16, None)
    torch.cuda.synchronize()
    k = torch.stack([kvc[s * Lk:(s + 1) * Lk, kcol:kcol + C] for s in slots.tolist()]).double()
    v = torch.stack([kvc[s * Lk:(s + 1) * Lk, vrow:vrow + C] for s in slots.tolist()]).double()
    qh = q.double().reshape(R, P, heads, d).transpose(1, 2)
    kh, vh = k.reshape(R, Lk, heads, d).transpose(1, 2), v.reshape(R, Lk, heads, d).transpose(1, 2)
    ref = torch.softmax(qh @ kh.transpose(-1, -2) / d ** 0.5, -1) @ vh
    ref = ref.transpose(1, 2).reshape(R, P, C)
    assert rel(o.cpu().reshape(R, P, C), ref) < (2e-3 if f16 else 1e-2)


@pytest.mark.parametrize("nb,P,C,G,silu", [(2, 4096, 320, 32, 1), (3, 256, 1280, 32, 0), (1, 64, 2560, 32, 1),
                                           (2, 64, 32, 8, 1), (1, 16384, 128, 32, 1),
                                           (3, 1000, 320, 32, 1), (5, 200, 640, 32, 0)])
def test_groupnorm(nb, P, C, G, silu):
    g = torch.Generator().manual_seed(P + C)
    x = bf(torch.randn(nb, P, C, generator=g) * 2 + 0.5)
    gam, bet = 1 + 0.1 * torch.randn(C, generator=g), 0.1 * torch.randn(C, generator=g)
    ref = F.group_norm(x.double().permute(0, 2, 1), G, gam.double(), bet.double(), 1e-5).permute(0, 2, 1)
    if silu:
        ref = F.silu(ref)
    y = torch.empty(nb, P, C, device="cuda", dtype=DT)
    xd, gd, bd = x.cuda(), gam.cuda(), bet.cuda()
    B.call("sd_debug_groupnorm", B._p(xd), B._p(y), nb, P, C, G, B._p(gd), B._p(bd), 1e-5, silu, None)
    torch.cuda.synchronize()
    assert rel(y.cpu(), ref) < 6e-3


@pytest.mark.parametrize("T,C", [(1000, 320), (77, 640), (300, 1280), (64, 32), (100, 2048)])
def test_layernorm(T, C):
    g = torch.Generator().manual_seed(T + C)
    x = bf(torch.randn(T, C, generator=g) * 3 - 1)
    gam, bet = 1 + 0.1 * torch.randn(C, generator=g), 0.1 * torch.randn(C, generator=g)
    ref = F.layer_norm(x.double(), (C,), gam.double(), bet.double(), 1e-5)
    y = torch.empty(T, C, device="cuda", dtype=DT)
    xd, gd, bd = x.cuda(), gam.cuda(), bet.cuda()
    B.call("sd_debug_layernorm", B._p(xd), B._p(y), T, C, B._p(gd), B._p(bd), 1e-5, None)
    torch.cuda.synchronize()
    assert rel(y.cpu(), ref) < 6e-3


# ---- GroupNorm statistics from the producer's epilogue (gemm.cu gn_colstats) ----------------------------
def _pow2_div(n, cap):
    p = 1
    while p * 2 <= cap and n % (p * 2) == 0:
        p *= 2
    return p


def _slot_sums(y, h, w):
    """Expected (Σy, Σy²) per (image, 32-pixel slot, channel) of a conv output [nb][h][w][C] under the conv
    tile geometry (wt = largest power of two dividing w, ≤ 128; slot box sw = min(wt, 32) × 32/sw)."""
    wt = _pow2_div(w, 128)
    sw = min(wt, 32)
    sh = 32 // sw
    nb, C = y.shape[0], y.shape[-1]
    yy = y.double().reshape(nb, h // sh, sh, w // sw, sw, C).permute(0, 1, 3, 2, 4, 5).reshape(nb, -1, 32, C)
    return torch.stack([yy.sum(2), (yy * yy).sum(2)], -1)


def _gn_ref(y, G, gam, bet, silu):
    ref = F.group_norm(y.double().permute(0, 2, 1), G, gam.double(), bet.double(), 1e-5).permute(0, 2, 1)
    return F.silu(ref) if silu else ref


@pytest.mark.parametrize("nb,h,w,cin,cout,silu", [(2, 64, 64, 320, 320, 1), (3, 32, 32, 640, 640, 1),
                                                  (2, 16, 16, 640, 1280, 0), (3, 8, 8, 1280, 640, 1),
                                                  (1, 32, 64, 128, 256, 1), (1, 128, 128, 64, 128, 1)])
def test_conv_gn_epilogue_stats(nb, h, w, cin, cout, silu):
    """The conv epilogue's per-slot column sums equal the sums of the stored output (fp64 over the same
    16-bit values), are bitwise deterministic and batch-invariant; GroupNorm from them matches GroupNorm
    of the conv output (fp64) and the statistics-pass kernel."""
    g = torch.Generator().manual_seed(nb + h + cin + cout)
    x = bf(torch.randn(nb, h, w, cin, generator=g))
    wt = bf(torch.randn(cout, cin, 3, 3, generator=g) / (9 * cin) ** 0.5)
    b = torch.randn(cout, generator=g) + 0.3
    res = bf(torch.randn(nb, h, w, cout, generator=g))
    gam, bet = 1 + 0.1 * torch.randn(cout, generator=g), 0.1 * torch.randn(cout, generator=g)
    xd, wd, bd, rd, gd, btd = x.cuda(), _to_dev_w(wt), b.cuda(), res.cuda(), gam.cuda(), bet.cuda()
    P = h * w

    def run(n):
        y = torch.empty(n, h, w, cout, device="cuda", dtype=DT)
        part = torch.full((n, P // 32, cout, 2), float("nan"), device="cuda")
        B.call("sd_debug_conv3x3_gn", B._p(xd[:n]), cin, B._p(wd), B._p(bd), B._p(rd[:n]), B._p(y), n, h, w, cout,
               B._p(part), None)
        torch.cuda.synchronize()
        return y, part

    y, part = run(nb)
    _, part2 = run(nb)
    _, part1 = run(1)
    assert torch.equal(part, part2), "epilogue statistics not deterministic"
    assert torch.equal(part[:1], part1), "epilogue statistics depend on the batch"
    exp = _slot_sums(y.cpu(), h, w)
    assert float((part.cpu().double() - exp).abs().max() / exp.abs().max()) < 1e-5
    gn = torch.empty_like(y)
    B.call("sd_debug_groupnorm_parts", B._p(y), cout, B._p(part), None, 0, None, B._p(gn), nb, P, 32, B._p(gd),
           B._p(btd), 1e-5, silu, None)
    gn_pass = torch.empty_like(y)
    B.call("sd_debug_groupnorm", B._p(y), B._p(gn_pass), nb, P, cout, 32, B._p(gd), B._p(btd), 1e-5, silu, None)
    torch.cuda.synchronize()
    ref = _gn_ref(y.cpu().reshape(nb, P, cout), 32, gam, bet, silu)
    assert rel(gn.cpu().reshape(nb, P, cout), ref) < 6e-3
    assert rel(gn.cpu(), gn_pass.cpu()) < 2e-3


def test_conv_gn_epilogue_ineligible():
    """4×4 images: a 32-pixel slot would straddle two images — the export refuses (no silent fallback)."""
    x = torch.zeros(2, 4, 4, 64, device="cuda", dtype=DT)
    wd = torch.zeros(64, 9, 64, device="cuda", dtype=DT)
    y = torch.empty(2, 4, 4, 64, device="cuda", dtype=DT)
    part = torch.empty(2, 1, 64, 2, device="cuda")
    with pytest.raises(B.SDError):
        B.call("sd_debug_conv3x3_gn", B._p(x), 64, B._p(wd), None, None, B._p(y), 2, 4, 4, 64, B._p(part), None)


@pytest.mark.parametrize("nb,P,N,K", [(2, 4096, 320, 320), (3, 1024, 640, 640), (4, 64, 1280, 1280), (2, 96, 256, 512)])
def test_gemm_gn_epilogue_stats_and_concat(nb, P, N, K):
    """Dense producer (rows = pixels of nb images of P): slot s = rows 32s..32s+31 of an image, exact sums;
    then GroupNorm over the concat [dense output | conv output] whose groups straddle the boundary
    (C = N + 320, G = 32), from the two producers' statistics, vs fp64."""
    g = torch.Generator().manual_seed(nb * P + N)
    M = nb * P
    A = bf(torch.randn(M, K, generator=g))
    Wt = bf(torch.randn(N, K, generator=g) / K ** 0.5)
    b = torch.randn(N, generator=g)
    res = bf(torch.randn(M, N, generator=g))
    Ad, Wd, bd, rd = A.cuda(), Wt.cuda(), b.cuda(), res.cuda()
    y = torch.empty(M, N, device="cuda", dtype=DT)
    part = torch.full((nb, P // 32, N, 2), float("nan"), device="cuda")
    B.call("sd_debug_gemm_gn", B._p(Ad), B._p(Wd), B._p(bd), B._p(rd), B._p(y), M, N, K, P, B._p(part), None)
    torch.cuda.synchronize()
    yy = y.cpu().double().reshape(nb, P // 32, 32, N)
    exp = torch.stack([yy.sum(2), (yy * yy).sum(2)], -1)
    assert float((part.cpu().double() - exp).abs().max() / exp.abs().max()) < 1e-5
    # second source: a conv output over the same pixels viewed as an image of P = h·w
    h, w = {4096: (64, 64), 1024: (32, 32), 64: (8, 8), 96: (3, 32)}[P]
    C1 = 320
    x = bf(torch.randn(nb, h, w, 64, generator=g))
    wc = bf(torch.randn(C1, 64, 3, 3, generator=g) / 24.0)
    y1 = torch.empty(nb, h, w, C1, device="cuda", dtype=DT)
    part1 = torch.full((nb, P // 32, C1, 2), float("nan"), device="cuda")
    xd, wcd = x.cuda(), _to_dev_w(wc)
    B.call("sd_debug_conv3x3_gn", B._p(xd), 64, B._p(wcd), None, None, B._p(y1), nb, h, w, C1, B._p(part1), None)
    C = N + C1
    gam, bet = 1 + 0.1 * torch.randn(C, generator=g), 0.1 * torch.randn(C, generator=g)
    gd, btd = gam.cuda(), bet.cuda()
    gn = torch.empty(nb, P, C, device="cuda", dtype=DT)
    B.call("sd_debug_groupnorm_parts", B._p(y), N, B._p(part), B._p(y1), C1, B._p(part1), B._p(gn), nb, P, 32,
           B._p(gd), B._p(btd), 1e-5, 1, None)
    torch.cuda.synchronize()
    cat = torch.cat([y.cpu().reshape(nb, P, N), y1.cpu().reshape(nb, P, C1)], -1)
    assert rel(gn.cpu(), _gn_ref(cat, 32, gam, bet, 1)) < 6e-3


@pytest.mark.parametrize("T,N,K,cols,act", [(1000, 640, 320, 0, 0), (300, 1280, 1280, 0, 0), (4096, 512, 640, 0, 2),
                                           (200, 320, 320, 1, 0), (1024, 1280, 1280, 1, 0), (77, 2560, 1280, 0, 2)])
def test_gemm_layernorm_folded(T, N, K, cols, act):
    """LayerNorm folded into the GEMM (W' = W diag(gamma), w-bar, b' = b + W beta, per-token (mu, rstd) applied
    in the epilogue) against fp64 LN then the GEMM on the same 16-bit inputs; the hidden state has a large
    mean (mean/std ~ 3) so the cancellation of the mu term is exercised. cols = 1: the V^T projection."""
    g = torch.Generator().manual_seed(T + N + K + cols)
    x = bf(torch.randn(T, K, generator=g) * 2.0 + 6.0)
    Wt = bf(torch.randn(N, K, generator=g) / K ** 0.5)
    gam, bet = 1 + 0.2 * torch.randn(K, generator=g), 0.2 * torch.randn(K, generator=g)
    bias = torch.randn(N, generator=g)
    ln = F.layer_norm(x.double(), (K,), gam.double(), bet.double(), 1e-5)
    full = ln @ Wt.double().T + bias.double()          # [T][N]
    if act == 2:
        v = torch.cat([full[:, 128 * j:128 * j + 64] for j in range(N // 128)], 1)
        gt = torch.cat([full[:, 128 * j + 64:128 * j + 128] for j in range(N // 128)], 1)
        ref = v * F.gelu(gt)
    else:
        ref = full.T if cols else full
    D = torch.empty(*ref.shape, device="cuda", dtype=DT)
    xd, Wd, gd, btd, bd = x.cuda(), Wt.cuda(), gam.cuda(), bet.cuda(), bias.cuda()
    B.call("sd_debug_gemm_ln", B._p(xd), T, B._p(Wd), N, K, B._p(gd), B._p(btd), B._p(bd), B._p(D), 1e-5, cols, act,
           None)
    torch.cuda.synchronize()
    assert rel(D.cpu(), ref) < 8e-3


def test_conv_bn320_tail_halves_bitwise():
    """BN = 320 pair tiles with tail balancing (the last partial wave split into 160-column half units): 16
    images at 64×64 → 256 pair tiles on 74 pairs, 34 tail tiles run as 68 halves; 8 images → 128 tiles,
    no halving. The first 8 images must agree bit for bit (same N = 160 MMAs over the same K blocks), and
    both must match fp64."""
    g = torch.Generator().manual_seed(320)
    nb, h, w, cin, cout = 16, 64, 64, 320, 320
    x = bf(torch.randn(nb, h, w, cin, generator=g))
    wt = bf(torch.randn(cout, cin, 3, 3, generator=g) / (9 * cin) ** 0.5)
    b = torch.randn(cout, generator=g)
    xd, wd, bd = x.cuda(), _to_dev_w(wt), b.cuda()

    def run(n):
        y = torch.empty(n, h, w, cout, device="cuda", dtype=DT)
        B.debug_conv3x3(xd[:n], cin, None, 0, wd, None, bd, None, None, y, n, h, w, cout)
        torch.cuda.synchronize()
        return y.cpu()

    y16, y8 = run(16), run(8)
    assert torch.equal(y16[:8], y8)
    ref = _conv_ref(x[:2].float(), wt.float(), b, None, None)
    assert rel(y16[:2], ref) < 6e-3
