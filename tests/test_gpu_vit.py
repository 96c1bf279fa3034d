"""ViT-B/16 perception (BASELINE configs[3]) on the B200 vs torch references.

Kernel tests compare vit.cu's LayerNorm / attention / token assembly with
torch on the same bf16 inputs (tolerance 2e-2 absolute on O(1) outputs: bf16
rounding of the stored result).  The encoder test runs the full 12-block
program (tcgen05 conv GEMMs + vit.cu kernels) against the fp32 torch-CPU
restatement in oracle/dp_model.py: bf16 weights and a bf16 residual stream
through 12 blocks, tolerance 3e-2 normwise relative on the CLS feature.  The
pipeline test drives the "vit" preset (ViT-B/16 + DP-default UNet, 7-DoF
actions) through run_pipelined against the oracle pipeline with the DP
suite's bf16 action tolerance (6e-2 normwise) and exact context versions.
"""

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import dp_model
from oracle import schedule as osched
from paper_2509_09560_b200 import PipelineConfig, _lib, run_pipelined
from paper_2509_09560_b200 import diffusion as D

pytestmark = pytest.mark.gpu
_W = {}


def vit_weights():
    if "vit" not in _W:
        _W["vit"] = D.init_weights(D.PRESETS["vit"], 0, device="cpu")
    return _W["vit"]


def test_layernorm_kernel():
    lib = _lib.load()
    x = torch.randn(37, 768, device="cuda").to(torch.bfloat16)
    g = torch.rand(768, device="cuda") + 0.5
    b = torch.randn(768, device="cuda") * 0.1
    ref = F.layer_norm(x.float(), (768,), g, b, eps=1e-6)
    out = torch.empty(37, 768, device="cuda", dtype=torch.bfloat16)
    _lib.check(lib.auras_layernorm(x.data_ptr(), 768, out.data_ptr(), 768, 0, g.data_ptr(), b.data_ptr(), 37, 768,
                                   1e-6, torch.cuda.current_stream().cuda_stream), "ln")
    o32 = torch.empty(37, 768, device="cuda")
    _lib.check(lib.auras_layernorm(x.data_ptr(), 768, o32.data_ptr(), 768, 1, g.data_ptr(), b.data_ptr(), 37, 768,
                                   1e-6, torch.cuda.current_stream().cuda_stream), "ln")
    torch.cuda.synchronize()
    assert (out.float() - ref).abs().max().item() <= 2e-2
    assert (o32 - ref).abs().max().item() <= 1e-4


def test_attention_ignores_pad_rows():
    """Rows n_valid..N-1 are padding: neither keys nor queries."""
    lib = _lib.load()
    S, N, nv, H, dh = 2, 200, 197, 12, 64
    C = H * dh
    qkv = torch.randn(S, N, 3 * C, device="cuda").to(torch.bfloat16)
    out = torch.zeros(S, N, C, device="cuda", dtype=torch.bfloat16)
    _lib.check(lib.auras_vit_attention(qkv.data_ptr(), out.data_ptr(), S, N, nv, H, dh,
                                       torch.cuda.current_stream().cuda_stream), "attn")
    q, k, v = qkv[:, :nv].float().reshape(S, nv, 3, H, dh).permute(2, 0, 3, 1, 4)
    ref = (torch.softmax((q * dh ** -0.5) @ k.transpose(-2, -1), dim=-1) @ v).transpose(1, 2).reshape(S, nv, C)
    torch.cuda.synchronize()
    assert (out[:, :nv].float() - ref).abs().max().item() <= 2e-2
    assert out[:, nv:].abs().max().item() == 0


@pytest.mark.parametrize("S,N,H,dh", [(2, 197, 12, 64), (3, 50, 4, 32), (1, 7, 2, 16)])
def test_attention_kernel(S, N, H, dh):
    lib = _lib.load()
    C = H * dh
    qkv = torch.randn(S, N, 3 * C, device="cuda").to(torch.bfloat16)
    out = torch.empty(S, N, C, device="cuda", dtype=torch.bfloat16)
    _lib.check(lib.auras_vit_attention(qkv.data_ptr(), out.data_ptr(), S, N, N, H, dh,
                                       torch.cuda.current_stream().cuda_stream), "attn")
    q, k, v = qkv.float().reshape(S, N, 3, H, dh).permute(2, 0, 3, 1, 4)
    ref = (torch.softmax((q * dh ** -0.5) @ k.transpose(-2, -1), dim=-1) @ v).transpose(1, 2).reshape(S, N, C)
    torch.cuda.synchronize()
    assert (out.float() - ref).abs().max().item() <= 2e-2


def test_tokens_kernel():
    lib = _lib.load()
    S, n, C = 2, 196, 768
    patches = torch.randn(S, n, C, device="cuda").to(torch.bfloat16)
    cls = torch.randn(C, device="cuda")
    pos = torch.randn(n + 1, C, device="cuda")
    x = torch.empty(S, n + 1, C, device="cuda", dtype=torch.bfloat16)
    _lib.check(lib.auras_vit_tokens(patches.data_ptr(), cls.data_ptr(), pos.data_ptr(), x.data_ptr(), S, n + 1, n + 1,
                                    C,
                                    torch.cuda.current_stream().cuda_stream), "tokens")
    ref = torch.cat([cls.expand(S, 1, C), patches.float()], dim=1) + pos
    torch.cuda.synchronize()
    assert (x.float() - ref).abs().max().item() <= 2e-2


def test_vit_encoder_matches_oracle():
    cfg = D.PRESETS["vit"]
    w = vit_weights()
    model = D.DeviceModel(cfg, w, "bf16")
    enc = D.ViTEncoder(model, 2)
    rng = np.random.default_rng(3)
    imgs = rng.integers(0, 256, (2, 3, 224, 224), dtype=np.uint8)
    enc.img.copy_(torch.from_numpy(imgs))
    st = torch.cuda.current_stream()
    enc.run(0, len(enc.GROUPS), st)
    torch.cuda.synchronize()
    got = enc.feat.cpu().numpy()
    for a in range(2):
        with torch.no_grad():
            want = dp_model.encode_vit(w, imgs[a], np.zeros(2))[:768].numpy()
        err = np.linalg.norm(got[a] - want) / np.linalg.norm(want)
        assert err <= 3e-2, (a, err)


def test_vit_policy_pipelined_matches_oracle():
    w = vit_weights()
    pol = D.make_diffusion_policy("vit", dtype="bf16", weights=w)
    gen = pol.generation
    cfg = dict(pp_perception=1, pp_generation=2, fetch_offset=0)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 3)
    orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, 0, pol.perception.layer_costs, gen.step_cost)
    ref = osched.run_pipelined(cfg, orc, None, 3)
    g = np.array([a.values for a in res.actions])
    r = np.array([a.values for a in ref.actions])
    assert g.shape == r.shape and g.shape[1] == 16 * 7
    assert float(np.abs(g - r).max() / np.abs(r).max()) <= 6e-2
    assert [q.context_versions for q in res.requests] == [q.context_versions for q in ref.requests]


def test_vit_dpt_policy_pipelined_matches_oracle():
    """BASELINE configs[3] end to end: ViT-B/16 perception + DP-T transformer
    denoiser, 7-DoF actions, through run_pipelined at depth 2, against the
    oracle pipeline (bf16 action tolerance 6e-2 normwise, exact versions)."""
    w = D.init_weights(D.PRESETS["vit_dpt"], 0, device="cpu")
    pol = D.make_diffusion_policy("vit_dpt", dtype="bf16", weights=w)
    gen = pol.generation
    for cfg in (dict(pp_perception=1, pp_generation=2, fetch_offset=0),
                dict(pp_perception=1, pp_generation=4, fetch_offset=-1),
                dict(pp_perception=2, pp_generation=2, fetch_offset=0)):      # staged ViT perception
        res = run_pipelined(PipelineConfig(**cfg), pol, None, 5)
        orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, 0, pol.perception.layer_costs, gen.step_cost)
        ref = osched.run_pipelined(cfg, orc, None, 5)
        g = np.array([a.values for a in res.actions])
        r = np.array([a.values for a in ref.actions])
        assert g.shape == r.shape and g.shape[1] == 16 * 7
        assert float(np.abs(g - r).max() / np.abs(r).max()) <= 6e-2
        assert [q.context_versions for q in res.requests] == [q.context_versions for q in ref.requests]


def test_vit_dpt_two_agents_and_sequential_match_oracle():
    """configs[3] with two agents batched into the same kernels (each against
    its own oracle run), and the depth-1 sequential baseline."""
    w = D.init_weights(D.PRESETS["vit_dpt"], 0, device="cpu")
    pol = D.make_diffusion_policy("vit_dpt", dtype="bf16", weights=w, agents=2)
    gen = pol.generation
    cfg = dict(pp_perception=1, pp_generation=3, fetch_offset=0)
    res = run_pipelined(PipelineConfig(**cfg), pol, None, 5, agents=2)
    for a in range(2):
        orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, a, pol.perception.layer_costs, gen.step_cost)
        ref = osched.run_pipelined(cfg, orc, None, 5)
        g = np.array([x.values for x in res.agent_actions[a]])
        r = np.array([x.values for x in ref.actions])
        assert g.shape == r.shape
        assert float(np.abs(g - r).max() / np.abs(r).max()) <= 6e-2, a
    from paper_2509_09560_b200 import run_sequential
    pol1 = D.make_diffusion_policy("vit_dpt", dtype="bf16", weights=w)
    res = run_sequential(pol1, None, 2)
    orc = dp_model.OracleDP(gen.weights, gen.cfg, gen.seed, 0, pol1.perception.layer_costs, gen.step_cost)
    ref = osched.run_sequential(orc, None, 2)
    g = np.array([x.values for x in res.actions])
    r = np.array([x.values for x in ref.actions])
    assert g.shape == r.shape and float(np.abs(g - r).max() / np.abs(r).max()) <= 6e-2


def test_vit_encoder_fused_layernorm_path(monkeypatch):
    """The residual + LayerNorm fused epilogue (auras_conv_ln) on the ViT
    program gives the same feature as the default path within bf16 noise."""
    cfg = D.PRESETS["vit"]
    w = vit_weights()
    model = D.DeviceModel(cfg, w, "bf16")
    imgs = np.random.default_rng(5).integers(0, 256, (1, 3, 224, 224), dtype=np.uint8)
    feats = []
    for fuse in ("0", "1"):
        monkeypatch.setenv("AURAS_VIT_FUSE_LN", fuse)
        enc = D.ViTEncoder(model, 1)
        enc.img.copy_(torch.from_numpy(imgs))
        enc.run(0, len(enc.GROUPS), torch.cuda.current_stream())
        torch.cuda.synchronize()
        feats.append(enc.feat.cpu().numpy()[0])
    assert np.linalg.norm(feats[0] - feats[1]) / np.linalg.norm(feats[0]) <= 2e-2


def test_vit_and_dpt_refuse_fp32():
    """configs[3] is a bf16 configuration: the ViT encoder and the DP-T
    denoiser refuse the fp32 path loudly instead of falling back."""
    from paper_2509_09560_b200 import ConfigInvalid
    cfg = D.PRESETS["vit_dpt"]
    model = D.DeviceModel(cfg, vit_dpt_weights(), "fp32")
    with pytest.raises(ConfigInvalid):
        D.ViTEncoder(model, 1)
    with pytest.raises(ConfigInvalid):
        D.DPTDenoiser(model, 4)


def vit_dpt_weights():
    if "vit_dpt" not in _W:
        _W["vit_dpt"] = D.init_weights(D.PRESETS["vit_dpt"], 0, device="cpu")
    return _W["vit_dpt"]
