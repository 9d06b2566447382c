"""Op-level parity of the tcgen05 implicit-GEMM kernel (csrc/gemm_tc.cu) through the C ABI
(lbx_op_gemm), against plain PyTorch fp32 references of the same op (TF32 off).

Tolerance: outputs are fp16 (relative precision 2^-11); fp32 accumulation.  We require
|got - ref| <= 2e-3 * max|ref| + 1e-3 elementwise (written per test below).
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def _close(got, ref, rel=2e-3, abs_=1e-3):
    got = got.float()
    ref = ref.float()
    tol = rel * ref.abs().max().item() + abs_
    err = (got - ref).abs().max().item()
    assert err <= tol, f"max err {err} > tol {tol}"


def _rand(*shape, scale=1.0, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).half().cuda()


@pytest.mark.parametrize("cg,bn", [(1, 128), (1, 256), (2, 128), (2, 256)])
@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (512, 512, 512), (1024, 256, 1152)])
def test_plain_gemm(lbx, cg, bn, M, N, K):
    if N % bn:
        pytest.skip("N not a multiple of the tile")
    A = _rand(M, K, seed=1)
    B = _rand(N, K, scale=K ** -0.5, seed=2)
    out = torch.empty(M, N, dtype=torch.half, device="cuda")
    lbx.op_gemm(0, M, N, K, A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), N, cta_group=cg, bn=bn)
    torch.cuda.synchronize()
    _close(out, A.float() @ B.float().t())


@pytest.mark.parametrize("cg", [1, 2])
def test_gemm_epilogue(lbx, cg):
    M, N, K = 512, 256, 256
    A = _rand(M, K, seed=3)
    B = _rand(N, K, scale=K ** -0.5, seed=4)
    bias = torch.randn(N, device="cuda")
    resid = _rand(M, N, seed=5)
    rs = torch.rand(M, device="cuda") + 0.5
    out = torch.empty(M, N, dtype=torch.half, device="cuda")
    lbx.op_gemm(0, M, N, K, A.data_ptr(), K, B.data_ptr(), K, out.data_ptr(), N, bias=bias.data_ptr(),
                resid=resid.data_ptr(), ldr=N, row_scale=rs.data_ptr(), alpha=0.5, cta_group=cg)
    torch.cuda.synchronize()
    ref = 0.5 * rs[:, None] * (A.float() @ B.float().t()) + bias[None, :] + resid.float()
    _close(out, ref)


@pytest.mark.parametrize("cg,bn", [(1, 128), (1, 256), (2, 128), (2, 256)])
@pytest.mark.parametrize("M,N,K,ldb", [(512, 512, 512, 512), (1024, 256, 1024, 1536), (256, 512, 2048, 1536)])
def test_gemm_mn_major_b(lbx, cg, bn, M, N, K, ldb):
    """B given as [K][N] (N contiguous, row stride ldb) -- the attention's V inside the QKV buffer
    for P.V, no transpose kernel -- staged as 64-wide MN atoms with an MN-major UMMA descriptor."""
    if N % bn:
        pytest.skip("N not a multiple of the tile")
    A = _rand(M, K, seed=31)
    Bfull = _rand(K, ldb, scale=K ** -0.5, seed=32)
    B = Bfull[:, ldb - N:] if ldb > N else Bfull  # a column window, like V at columns 1024..1535
    rs = torch.rand(M, device="cuda") + 0.5
    out = torch.empty(M, N, dtype=torch.half, device="cuda")
    lbx.op_gemm(0, M, N, K, A.data_ptr(), K, B.data_ptr(), ldb, out.data_ptr(), N, row_scale=rs.data_ptr(),
                cta_group=cg, bn=bn, b_mn_major=True)
    torch.cuda.synchronize()
    _close(out, rs[:, None] * (A.float() @ B.float()))


@pytest.mark.parametrize("bits", [1 | (1 << 18), 1 | (1 << 16), 1 | (3 << 16)])
def test_epilogue_store_variants(lbx, bits):
    """The TMA-store epilogue (bit 18) and the STG.128 / streaming store modes give the same
    results as the default (STG.256): conv with residual + statistics and a plain GEMM."""
    b, h, w, c = 2, 16, 256, 128
    x = _rand(b, h, w, c, seed=71)
    wt = _rand(c, c, 3, 3, scale=(9 * c) ** -0.5, seed=72)
    wk = wt.permute(0, 2, 3, 1).contiguous()
    resid = _rand(b, h, w, c, seed=73)
    bias = torch.randn(c, device="cuda")
    outs = []
    try:
        for bb in (1, bits):
            lbx.check(lbx.lib().lbx_op_set_debug(bb, 0))
            out = torch.empty(b, h, w, c, dtype=torch.half, device="cuda")
            stats = lbx.gn_stats_buffer(b)
            lbx.op_gemm(1, b * h * w, c, 9 * c, x.data_ptr(), 0, wk.data_ptr(), 9 * c, out.data_ptr(), c, b=b, h=h,
                        w=w, c=c, bias=bias.data_ptr(), resid=resid.data_ptr(), ldr=c, gn_stats=stats.data_ptr())
            A = _rand(512, 512, seed=74)
            B = _rand(1024, 512, scale=512 ** -0.5, seed=75)
            g = torch.empty(512, 1024, dtype=torch.half, device="cuda")
            lbx.op_gemm(0, 512, 1024, 512, A.data_ptr(), 512, B.data_ptr(), 512, g.data_ptr(), 1024, alpha=0.5)
            torch.cuda.synchronize()
            outs.append((out.clone(), g.clone(), stats.clone()))
    finally:
        lbx.check(lbx.lib().lbx_op_set_debug(1, 0))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    _close(outs[1][0], _conv_ref(x, wt, bias) + resid.float())
    _check_gn_stats(outs[1][2], outs[1][0], b, h * w, c)


def test_gemm_strided_views(lbx):
    """Q K^T on column views of a [L, 1536] QKV buffer (row stride 1536), as the attention uses."""
    L = 512
    qkv = _rand(L, 1536, seed=6)
    S = torch.empty(L, L, dtype=torch.half, device="cuda")
    q, k = qkv[:, :512], qkv[:, 512:1024]
    lbx.op_gemm(0, L, L, 512, q.data_ptr(), 1536, k.data_ptr(), 1536, S.data_ptr(), L, alpha=512 ** -0.5)
    torch.cuda.synchronize()
    _close(S, (q.float() @ k.float().t()) * 512 ** -0.5)


def _check_gn_stats(stats, out, b, hw, n):
    """GN partials are sums of the fp32 epilogue values just before their fp16 rounding; check the
    per-(image, group) mean and variance they imply against a float64 reduction of the stored fp16
    output: |d mean| <= 2e-4 * rms and |d var| <= 1e-3 * var (the rounding is < 2^-12 relative)."""
    o = out.double().reshape(b, hw, 32, n // 32)
    cnt = hw * (n // 32)
    mean_r = o.sum(dim=(1, 3)) / cnt
    var_r = (o * o).sum(dim=(1, 3)) / cnt - mean_r ** 2
    import paper_2605_19385_b200 as lbxm
    st = lbxm.gn_stats_values(stats)
    mean = st[..., 0] / cnt
    var = st[..., 1] / cnt - mean ** 2
    rms = (var_r + mean_r ** 2).sqrt()
    assert ((mean - mean_r).abs() <= 2e-4 * rms + 1e-6).all(), (mean - mean_r).abs().max()
    assert ((var - var_r).abs() <= 1e-3 * var_r + 1e-6).all(), ((var - var_r).abs() / var_r).max()


def _conv_ref(x_nhwc, w_oihw, bias):
    x = x_nhwc.permute(0, 3, 1, 2).float()
    y = F.conv2d(x, w_oihw.float(), bias, padding=1)
    return y.permute(0, 2, 3, 1)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("b,h,w,c,n", [(1, 64, 64, 64, 128), (2, 64, 64, 128, 256), (1, 128, 128, 64, 256),
                                       (1, 16, 256, 64, 128)])
def test_conv3x3(lbx, cg, b, h, w, c, n):
    x = _rand(b, h, w, c, seed=7)
    wt = _rand(n, c, 3, 3, scale=(9 * c) ** -0.5, seed=8)
    bias = torch.randn(n, device="cuda")
    wk = wt.permute(0, 2, 3, 1).contiguous()  # [N][ky][kx][C]
    out = torch.empty(b, h, w, n, dtype=torch.half, device="cuda")
    lbx.op_gemm(1, b * h * w, n, 9 * c, x.data_ptr(), 0, wk.data_ptr(), 9 * c, out.data_ptr(), n, b=b, h=h, w=w,
                c=c, bias=bias.data_ptr(), cta_group=cg)
    torch.cuda.synchronize()
    _close(out, _conv_ref(x, wt, bias))


@pytest.mark.parametrize("cg", [1, 2])
def test_conv3x3_resid_gnstats(lbx, cg):
    b, h, w, c, n = 2, 64, 64, 128, 128
    x = _rand(b, h, w, c, seed=9)
    wt = _rand(n, c, 3, 3, scale=(9 * c) ** -0.5, seed=10)
    wk = wt.permute(0, 2, 3, 1).contiguous()
    resid = _rand(b, h, w, n, seed=11)
    out = torch.empty(b, h, w, n, dtype=torch.half, device="cuda")
    stats = lbx.gn_stats_buffer(b)
    lbx.op_gemm(1, b * h * w, n, 9 * c, x.data_ptr(), 0, wk.data_ptr(), 9 * c, out.data_ptr(), n, b=b, h=h, w=w,
                c=c, resid=resid.data_ptr(), ldr=n, gn_stats=stats.data_ptr(), cta_group=cg)
    torch.cuda.synchronize()
    _close(out, _conv_ref(x, wt, None) + resid.float())
    _check_gn_stats(stats, out, b, h * w, n)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("b,h,w,c", [(1, 64, 64, 128), (2, 32, 128, 128), (1, 16, 256, 256)])
def test_subpixel_upsample_conv(lbx, cg, b, h, w, c):
    """nearest-2x upsample + conv3x3 == 4 sub-pixel 2x2 convs on the low-res grid."""
    x = _rand(b, h, w, c, seed=12)
    wt = _rand(c, c, 3, 3, scale=(9 * c) ** -0.5, seed=13)
    bias = torch.randn(c, device="cuda")
    w4 = torch.from_numpy(lbx.subpixel_weights(wt.float().permute(0, 2, 3, 1).cpu().numpy()).copy()).cuda()
    out = torch.empty(b, 2 * h, 2 * w, c, dtype=torch.half, device="cuda")
    lbx.op_gemm(2, b * h * w, c, 4 * c, x.data_ptr(), 0, w4.data_ptr(), 4 * c, out.data_ptr(), c, b=b, h=h, w=w,
                c=c, bias=bias.data_ptr(), cta_group=cg)
    torch.cuda.synchronize()
    up = F.interpolate(x.permute(0, 3, 1, 2).float(), scale_factor=2.0, mode="nearest")
    ref = F.conv2d(up, wt.float(), bias, padding=1).permute(0, 2, 3, 1)
    # folded weights are re-rounded to fp16: allow a slightly wider band
    _close(out, ref, rel=4e-3)


@pytest.mark.parametrize("c", [128, 256, 512])
@pytest.mark.parametrize("silu", [0, 1, 2])
@pytest.mark.parametrize("inplace", [False, True])
def test_gn_stats_and_apply(lbx, c, silu, inplace):
    """Standalone statistics + apply (128/512 channels take the bulk-copy kernel, 256 the
    register-staged one); silu 0 identity, 1 fp32 SiLU, 2 packed-half SiLU (looser bound)."""
    b, hw = 3, 4096
    x = _rand(b, hw, c, seed=14) * 2 + 0.5
    stats = lbx.gn_stats_buffer(b)
    lbx.op_gn_stats(x.data_ptr(), stats.data_ptr(), b, hw, c)
    gamma = torch.rand(c, device="cuda") + 0.5
    beta = torch.randn(c, device="cuda") * 0.1
    ref = F.group_norm(x.float().permute(0, 2, 1), 32, gamma, beta, 1e-6).permute(0, 2, 1)
    if silu:
        ref = F.silu(ref)
    y = x if inplace else torch.empty_like(x)
    lbx.op_groupnorm(x.data_ptr(), y.data_ptr(), stats.data_ptr(), gamma.data_ptr(), beta.data_ptr(), b, hw, c,
                     silu=silu)
    torch.cuda.synchronize()
    _close(y, ref, rel=4e-3 if silu == 2 else 2e-3, abs_=2e-3)


@pytest.mark.parametrize("rbuf", [False, True])
@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("b,h,w,c,cin", [(2, 16, 256, 128, 128), (1, 16, 256, 128, 256), (1, 64, 64, 256, 512),
                                         (3, 8, 512, 128, 128), (1, 8, 512, 256, 512)])
def test_conv3x3_with_folded_residual(lbx, cg, b, h, w, c, cin, rbuf):
    """conv3x3(H) + X.W2^T as an extra K segment (identity -> residual, W_sc -> 1x1 shortcut); with
    rbuf (debug bit 24) the segment's k-blocks go through their own buffer between halo taps."""
    if rbuf:
        lbx.check(lbx.lib().lbx_op_set_debug(1 | (1 << 24), 0))
    try:
        _folded_residual_case(lbx, cg, b, h, w, c, cin)
    finally:
        lbx.check(lbx.lib().lbx_op_set_debug(1, 0))


def _folded_residual_case(lbx, cg, b, h, w, c, cin):
    n = c
    hin = _rand(b, h, w, c, seed=21)
    x = _rand(b, h, w, cin, seed=22)
    wt = _rand(n, c, 3, 3, scale=(9 * c) ** -0.5, seed=23)
    if cin == c:
        wsc = torch.eye(c, device="cuda").half()
    else:
        wsc = _rand(n, cin, scale=cin ** -0.5, seed=24)
    wk = torch.cat([wt.permute(0, 2, 3, 1).reshape(n, 9 * c), wsc], dim=1).contiguous()
    bias = torch.randn(n, device="cuda")
    out = torch.empty(b, h, w, n, dtype=torch.half, device="cuda")
    stats = lbx.gn_stats_buffer(b)
    lbx.op_gemm(1, b * h * w, n, 9 * c, hin.data_ptr(), 0, wk.data_ptr(), 9 * c + cin, out.data_ptr(), n, b=b, h=h,
                w=w, c=c, bias=bias.data_ptr(), gn_stats=stats.data_ptr(), cta_group=cg, a2=x.data_ptr(), lda2=cin,
                k2=cin)
    torch.cuda.synchronize()
    ref = _conv_ref(hin, wt, bias) + (x.float().reshape(-1, cin) @ wsc.float().t()).reshape(b, h, w, n)
    _close(out, ref)
    _check_gn_stats(stats, out, b, h * w, n)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("b,h,w,c,n,fold", [(2, 16, 128, 256, 256, False), (1, 16, 256, 512, 512, True),
                                            (2, 8, 256, 256, 256, True), (2, 16, 256, 128, 128, True),
                                            (1, 8, 512, 256, 128, False)])
def test_conv3x3_fused_groupnorm_silu(lbx, cg, b, h, w, c, n, fold):
    """A' = SiLU(A * a[img, c] + b[img, c]) applied to the halo in smem (packed-half SiLU, as the
    decoder's GroupNorm applies); padding stays zero.  128-wide N exercises the vertical sub-tiles."""
    x = _rand(b, h, w, c, seed=41) * 2 + 0.3
    g = torch.Generator(device="cpu").manual_seed(42)
    ss = torch.stack([torch.rand(b, c, generator=g) + 0.5, torch.randn(b, c, generator=g) * 0.5], dim=-1).cuda()
    wt = _rand(n, c, 3, 3, scale=(9 * c) ** -0.5, seed=43)
    wk = wt.permute(0, 2, 3, 1).reshape(n, 9 * c)
    xr = _rand(b, h, w, n, seed=44) if fold else None
    if fold:
        wk = torch.cat([wk, torch.eye(n, device="cuda").half()], dim=1)
    wk = wk.contiguous()
    bias = torch.randn(n, device="cuda")
    out = torch.empty(b, h, w, n, dtype=torch.half, device="cuda")
    stats = lbx.gn_stats_buffer(b)
    lbx.op_gemm(1, b * h * w, n, 9 * c, x.data_ptr(), 0, wk.data_ptr(), wk.shape[1], out.data_ptr(), n, b=b, h=h,
                w=w, c=c, bias=bias.data_ptr(), gn_stats=stats.data_ptr(), cta_group=cg, gn_ss=ss.data_ptr(),
                a2=xr.data_ptr() if fold else 0, lda2=n if fold else 0, k2=n if fold else 0)
    torch.cuda.synchronize()
    act = F.silu(x.float() * ss[:, None, None, :, 0] + ss[:, None, None, :, 1]).half()  # fp16 like the kernel
    ref = _conv_ref(act, wt, bias)
    if fold:
        ref = ref + xr.float()
    _close(out, ref, rel=3e-3)
    _check_gn_stats(stats, out, b, h * w, n)


@pytest.mark.parametrize("impl", [0, 2, 1])
@pytest.mark.parametrize("n,H,W", [(2, 64, 128), (1, 128, 256), (3, 32, 512)])
def test_conv_out_tail(lbx, impl, n, H, W):
    """Decoder tail u8(conv3x3_128->3(SiLU(GN-affine(x))) + b) against torch fp32; impl 0/2 are the
    tensor-core kernel (fp32 / packed-half SiLU, fp16 activations and weights), 1 the CUDA-core one.
    Bar: every pixel within 1 LSB of the fp32 reference; >= 97% exact with fp32 SiLU (fp16 operands),
    >= 95% with the packed-half SiLU."""
    x = _rand(n, H, W, 128, seed=61) * 1.5 + 0.2
    g = torch.Generator(device="cpu").manual_seed(62)
    ss = torch.stack([torch.rand(n, 128, generator=g) + 0.5, torch.randn(n, 128, generator=g) * 0.5], dim=-1).cuda()
    w = (torch.randn(3, 3, 3, 128, generator=g) * (1152 ** -0.5) * 3).cuda()  # [out][ky][kx][in]
    b = (torch.randn(3, generator=g) * 0.2).cuda()
    rgb = torch.empty(n, H, W, 3, dtype=torch.uint8, device="cuda")
    lbx.op_conv_out(x.data_ptr(), ss.data_ptr(), w.data_ptr(), b.data_ptr(), rgb.data_ptr(), n, H, W, impl=impl)
    torch.cuda.synchronize()
    act = F.silu(x.float() * ss[:, None, None, :, 0] + ss[:, None, None, :, 1])
    y = F.conv2d(act.permute(0, 3, 1, 2), w.permute(0, 3, 1, 2), b, padding=1).permute(0, 2, 3, 1)
    ref = torch.round((y * 0.5 + 0.5).clamp(0, 1) * 255).to(torch.int32)  # torch.round: half to even
    d = (rgb.int() - ref).abs()
    exact = (d == 0).float().mean().item()
    print(f"\n[conv_out impl {impl} {n}x{H}x{W}] max|d|={d.max().item()} exact={exact:.4f}")
    assert d.max().item() <= 1
    assert exact >= (0.95 if impl == 2 else 0.97)


@pytest.mark.parametrize("n,L,scale", [(1, 256, 1.0), (2, 512, 1.0), (1, 2048, 2.0), (2, 4096, 0.7)])
def test_flash_attention_core(lbx, n, L, scale):
    """CTA-pair flash attention (d split across the pair, partial scores and P exchanged through
    DSMEM) against torch fp32 softmax(Q K^T / sqrt(512)) V on the same fp16 QKV buffer."""
    qkv = _rand(n, L, 1536, scale=scale, seed=81)
    out = torch.empty(n, L, 512, dtype=torch.half, device="cuda")
    lbx.op_attention(qkv.data_ptr(), out.data_ptr(), n, L)
    torch.cuda.synchronize()
    q, k, v = qkv[..., :512].float(), qkv[..., 512:1024].float(), qkv[..., 1024:].float()
    ref = torch.softmax(q @ k.transpose(1, 2) / 512 ** 0.5, dim=-1) @ v
    _close(out, ref, rel=4e-3, abs_=2e-3)
