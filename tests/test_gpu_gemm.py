"""Conv engines vs a plain PyTorch fp32 reference of the same op.

The bf16 path routes 1-D convolutions (Cin % 64 == 0) to the tcgen05/TMA
engine; operands are rounded to bf16 on both sides, so only accumulation
order differs (fp32 on both): tolerance 2e-3 relative to max |ref|.
"""

import ctypes as C

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2509_09560_b200 import _lib

pytestmark = pytest.mark.gpu
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False


def run_conv1d(x, w, b, stride, pad, dtype="bf16", in_pitch=None, in_coff=0, stuff=False):
    """x: [S, T, Cin] view inside a [S, T, pitch] buffer; w: [Co, Cin, k]."""
    lib = _lib.load()
    S, T, Cin = x.shape
    Co, _, k = w.shape
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    pitch = in_pitch or Cin
    buf = torch.zeros(S, T, pitch, dtype=td, device="cuda")
    buf[:, :, in_coff:in_coff + Cin] = x.to(td)
    wm = w.permute(0, 2, 1).reshape(Co, k * Cin)
    Kp = (k * Cin + 63) // 64 * 64
    wm = F.pad(wm, (0, Kp - k * Cin)).to(td).contiguous().cuda()
    To = (T + 2 * pad - k) // stride + 1
    out = torch.zeros(S, To, Co, dtype=torch.float32, device="cuda")
    bias = b.float().cuda().contiguous()
    op = _lib.ConvOp(w=wm.data_ptr(), bias=bias.data_ptr(), inp=buf.data_ptr(), out=0,
                     out_f32=out.data_ptr(), M=Co, Cin=Cin, Kp=Kp, H=1, W=T, in_pitch=pitch,
                     in_coff=in_coff, kh=1, kw=k, stride=stride, pad_h=0, pad_w=pad, Ho=1, Wo=To,
                     out_pitch=Co, out_coff=0, groups=1, act=0, film_off=-1, splits=4)
    scratch = torch.zeros(64 * S * To * Co + 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    _lib.check(lib.auras_conv(C.byref(op), _lib.DT_BF16 if dtype == "bf16" else _lib.DT_F32, S, None, 0,
                              scratch.data_ptr(), scratch.numel(), st.cuda_stream), "conv")
    torch.cuda.synchronize()
    ref = F.conv1d(x.to(td).float().permute(0, 2, 1).cuda(), wm[:, :k * Cin].float().reshape(Co, k, Cin)
                   .permute(0, 2, 1), bias, stride=stride, padding=pad).permute(0, 2, 1)
    return out, ref


CASES = [
    # (S, T, Cin, Co, k, stride, pad)
    (1, 4, 2048, 2048, 5, 1, 2),
    (8, 4, 1024, 2048, 5, 1, 2),
    (3, 16, 64, 512, 5, 1, 2),
    (8, 16, 512, 512, 3, 2, 1),      # Downsample1d
    (4, 16, 1024, 512, 4, 1, 2),     # Upsample1d as conv over a zero-stuffed input
    (2, 8, 4096, 1024, 1, 1, 0),     # residual 1x1
    (5, 16, 128, 64, 5, 1, 2),       # M < 128 (tiny UNet)
    (17, 16, 256, 256, 5, 1, 2),     # N > 256: two N tiles
    (6, 8, 1024, 1024, 3, 2, 1),
]


@pytest.mark.parametrize("S,T,Cin,Co,k,stride,pad", CASES)
def test_tcgen05_conv_matches_torch(S, T, Cin, Co, k, stride, pad):
    torch.manual_seed(S * 131 + Co)
    x = torch.randn(S, T, Cin)
    w = torch.randn(Co, Cin, k) / (Cin * k) ** 0.5
    b = torch.randn(Co) * 0.1
    out, ref = run_conv1d(x, w, b, stride, pad)
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-3, err


def test_concat_view_channel_offset():
    torch.manual_seed(7)
    S, T, Cin, Co = 4, 8, 512, 1024
    x = torch.randn(S, T, Cin)
    w = torch.randn(Co, Cin, 3) / (Cin * 3) ** 0.5
    b = torch.zeros(Co)
    out, ref = run_conv1d(x, w, b, 2, 1, in_pitch=2 * Cin, in_coff=Cin)
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-3, err


def test_fp32_simt_engine_matches_torch():
    torch.manual_seed(3)
    x = torch.randn(3, 8, 256)
    w = torch.randn(512, 256, 5) / (256 * 5) ** 0.5
    b = torch.randn(512) * 0.1
    out, ref = run_conv1d(x, w, b, 1, 2, dtype="fp32")
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err


def run_conv2d(x, w, stride, pad, S_agents=None):
    """x: [S, H, W, Cin] NHWC; w: [Co, Cin, kh, kw]; bf16 operands, tcgen05 gather engine."""
    lib = _lib.load()
    S, H, W, Cin = x.shape
    Co, _, kh, kw = w.shape
    buf = x.to(torch.bfloat16).contiguous().cuda()
    wm = w.permute(0, 2, 3, 1).reshape(Co, kh * kw * Cin)
    Kp = (kh * kw * Cin + 63) // 64 * 64
    wm = F.pad(wm, (0, Kp - kh * kw * Cin)).to(torch.bfloat16).contiguous().cuda()
    Ho, Wo = (H + 2 * pad - kh) // stride + 1, (W + 2 * pad - kw) // stride + 1
    out = torch.zeros(S, Ho, Wo, Co, dtype=torch.float32, device="cuda")
    op = _lib.ConvOp(w=wm.data_ptr(), bias=0, inp=buf.data_ptr(), out=0, out_f32=out.data_ptr(), M=Co,
                     Cin=Cin, Kp=Kp, H=H, W=W, in_pitch=Cin, in_coff=0, kh=kh, kw=kw, stride=stride,
                     pad_h=pad, pad_w=pad, Ho=Ho, Wo=Wo, out_pitch=Co, out_coff=0, groups=1, act=0,
                     film_off=-1, splits=1)
    scratch = torch.zeros(64 * S * Ho * Wo * Co + 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    _lib.check(lib.auras_conv(C.byref(op), _lib.DT_BF16, S, None, 0, scratch.data_ptr(), scratch.numel(),
                              st.cuda_stream), "conv2d")
    torch.cuda.synchronize()
    ref = F.conv2d(buf.float().permute(0, 3, 1, 2), wm[:, :kh * kw * Cin].float().reshape(Co, kh, kw, Cin)
                   .permute(0, 3, 1, 2), stride=stride, padding=pad).permute(0, 2, 3, 1)
    return out, ref


CASES_2D = [
    # (S, H, W, Cin, Co, k, stride, pad): the ResNet-18 encoder's conv shapes
    (1, 96, 96, 8, 64, 7, 2, 3),      # stem (RGB padded to 8 channels)
    (2, 24, 24, 64, 64, 3, 1, 1),     # layer1
    (1, 24, 24, 64, 128, 3, 2, 1),    # layer2 first conv
    (3, 24, 24, 64, 128, 1, 2, 0),    # layer2 downsample
    (1, 6, 6, 256, 512, 3, 2, 1),     # layer4 first conv (3x3 output)
    (2, 3, 3, 512, 512, 3, 1, 1),     # layer4
]


@pytest.mark.parametrize("S,H,W,Cin,Co,k,stride,pad", CASES_2D)
def test_tcgen05_gather_conv2d_matches_torch(S, H, W, Cin, Co, k, stride, pad):
    torch.manual_seed(H * 7 + Co)
    x = torch.randn(S, H, W, Cin)
    w = torch.randn(Co, Cin, k, k) / (Cin * k * k) ** 0.5
    out, ref = run_conv2d(x, w, stride, pad)
    err = (out - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-3, err
