"""CPU checks of the DP plugin's host-side pieces and of the DP oracle wiring."""

import numpy as np
import pytest
import torch

from oracle import dp_model
from paper_2509_09560_b200 import diffusion as D


def test_unet_layout_tiny_and_pusht():
    for name in ("tiny", "pusht"):
        cfg = D.PRESETS[name]
        blocks = D.unet_blocks(cfg)
        assert [b[0] for b in blocks] == ["down0.0", "down0.1", "down1.0", "down1.1", "down2.0",
                                          "down2.1", "mid.0", "mid.1", "up0.0", "up0.1", "up1.0",
                                          "up1.1"]
        d0, d1, d2 = cfg.down_dims
        assert blocks[8][1:] == (2 * d2, d1, 4) and blocks[10][1:] == (2 * d1, d0, 8)
        offs, F = D.film_layout(cfg)
        assert F == 2 * sum(b[2] for b in blocks)
    cfg = D.PRESETS["pusht"]
    assert cfg.gc_dim == 1028
    # ~488 MB of bf16 conv weights streamed per step at PushT-img widths
    assert 480e6 < D.unet_stream_bytes(cfg) < 500e6
    assert 2.3e9 < D.unet_flops_per_sample(cfg) < 2.45e9


@pytest.mark.parametrize("name", ["tiny", "pusht"])
def test_scheduler_tables_match_oracle(name):
    cfg = D.PRESETS[name]
    tab = D.scheduler_tables(cfg)
    ref = dp_model.Scheduler(cfg)
    assert list(tab["timestep"]) == ref.timesteps
    x = torch.randn(16, 2, dtype=torch.float64)
    eps = torch.randn(16, 2, dtype=torch.float64)
    z = torch.randn(16, 2, dtype=torch.float64)
    for i in range(cfg.num_inference_steps):
        x0 = ((x - tab["sqrt_1mab"][i] * eps) / tab["sqrt_ab"][i]).clamp(-1, 1)
        got = tab["c_x0"][i] * x0 + tab["c_xt"][i] * x + tab["c_eps"][i] * eps + tab["sigma"][i] * z
        want = ref.step(i, x, eps, z)
        assert torch.allclose(got, want, rtol=1e-12, atol=1e-12)


def test_request_noise_and_frames_match_oracle():
    cfg = D.PRESETS["pusht"]
    xT, z = D.request_noise(cfg, 3, 1, 17)
    gen = dp_model.OracleGeneration({}, cfg, 3, 1, 1.0)
    st = gen.initial_state(seed=17)
    assert np.array_equal(xT, st.x.numpy()) and np.array_equal(z, st.z.numpy())
    o1 = D.synthetic_frame(cfg, 3, 1, 17)
    o2 = dp_model.synthetic_frame(cfg, 3, 1, 17)
    assert np.array_equal(o1.image, o2.image) and np.array_equal(o1.vector, o2.vector)


def test_oracle_resnet_trunk_matches_torchvision_wiring():
    """Cross-check the restated encoder against torchvision's resnet18 with every
    BatchNorm swapped for GroupNorm(C/16)."""
    tv = pytest.importorskip("torchvision")
    cfg = D.PRESETS["tiny"]
    w = D.init_weights(cfg, seed=1)
    net = tv.models.resnet18(weights=None)
    net.fc = torch.nn.Identity()

    def swap(mod):
        for n, ch in mod.named_children():
            if isinstance(ch, torch.nn.BatchNorm2d):
                setattr(mod, n, torch.nn.GroupNorm(ch.num_features // 16, ch.num_features))
            else:
                swap(ch)
    swap(net)
    sd = {"conv1.weight": w["enc.conv1.w"], "bn1.weight": w["enc.gn1.g"], "bn1.bias": w["enc.gn1.b"]}
    for li in range(1, 5):
        for bi in range(2):
            p, q = f"enc.layer{li}.{bi}", f"layer{li}.{bi}"
            sd[q + ".conv1.weight"] = w[p + ".conv1.w"]
            sd[q + ".bn1.weight"], sd[q + ".bn1.bias"] = w[p + ".gn1.g"], w[p + ".gn1.b"]
            sd[q + ".conv2.weight"] = w[p + ".conv2.w"]
            sd[q + ".bn2.weight"], sd[q + ".bn2.bias"] = w[p + ".gn2.g"], w[p + ".gn2.b"]
            if p + ".ds.w" in w:
                sd[q + ".downsample.0.weight"] = w[p + ".ds.w"]
                sd[q + ".downsample.1.weight"] = w[p + ".dsgn.g"]
                sd[q + ".downsample.1.bias"] = w[p + ".dsgn.b"]
    net.load_state_dict(sd)
    obs = D.synthetic_frame(cfg, 0, 0, 5)
    with torch.no_grad():
        ref = net(torch.from_numpy(obs.image).float()[None] * (2 / 255) - 1)[0]
        got = dp_model.encode(w, obs.image, obs.vector)
    assert torch.allclose(got[:512], ref, rtol=1e-4, atol=1e-5)


def test_oracle_unet_runs_and_is_deterministic():
    cfg = D.PRESETS["tiny"]
    w = D.init_weights(cfg, seed=2)
    gc = torch.randn(cfg.gc_dim)
    x = torch.randn(cfg.horizon, cfg.action_dim)
    e1 = dp_model.unet_eps(w, cfg, x, 42, gc)
    e2 = dp_model.unet_eps(w, cfg, x, 42, gc)
    assert e1.shape == (16, 2) and torch.isfinite(e1).all() and torch.equal(e1, e2)


def test_vit_preset_matches_survey_sizes():
    """configs[3] perception: ViT-B/16 at 224x224 is 85.8 M parameters and
    about 35.1 GFLOP per frame."""
    from paper_2509_09560_b200 import diffusion as D
    cfg = D.PRESETS["vit"]
    w = D.init_weights(cfg, 0)
    n_vit = sum(v.numel() for k, v in w.items() if k.startswith("vit."))
    assert abs(n_vit / 1e6 - 85.8) < 0.1
    assert abs(sum(D.encoder_flops(cfg)) / 1e9 - 35.1) < 0.1
    assert cfg.action_dim == 7 and cfg.image_hw == 224 and cfg.feat_dim == 768
    assert len(D.encoder_flops(cfg)) == len(D.ViTEncoder.GROUPS)
    assert not any(k.startswith("enc.") for k in w)          # no ResNet weights in this preset


def test_oracle_vit_matches_torch_transformer_layers():
    """Pins the ViT-B/16 restatement (oracle/dp_model.py encode_vit) against
    torch's own pre-norm nn.TransformerEncoderLayer (exact GELU, LayerNorm
    eps 1e-6, fused in_proj in q|k|v order = timm's qkv layout) loaded with
    the same weights, on a 2-block, 112x112 variant to keep it fast."""
    import numpy as np
    import torch
    from oracle import dp_model
    from paper_2509_09560_b200 import diffusion as D
    cfg = D.DPConfig(name="vit_small_test", encoder="vit_b16", image_hw=112, feat_dim=768, vit_depth=2)
    w = D.init_weights(cfg, 1)
    img = np.random.default_rng(0).integers(0, 256, (3, 112, 112), dtype=np.uint8)
    got = dp_model.encode_vit(w, img, np.zeros(2))[:768]
    x = torch.from_numpy(img).float()[None] * (2.0 / 255.0) - 1.0
    x = torch.nn.functional.conv2d(x, w["vit.patch.w"], w["vit.patch.b"], stride=16).flatten(2).transpose(1, 2)
    x = torch.cat([w["vit.cls"].reshape(1, 1, 768), x], dim=1) + w["vit.pos"][None]
    for i in range(2):
        p = f"vit.b{i}"
        layer = torch.nn.TransformerEncoderLayer(768, 12, 3072, dropout=0.0, activation="gelu", layer_norm_eps=1e-6,
                                                 batch_first=True, norm_first=True)
        with torch.no_grad():
            layer.self_attn.in_proj_weight.copy_(w[p + ".qkv.w"])
            layer.self_attn.in_proj_bias.copy_(w[p + ".qkv.b"])
            layer.self_attn.out_proj.weight.copy_(w[p + ".proj.w"])
            layer.self_attn.out_proj.bias.copy_(w[p + ".proj.b"])
            layer.norm1.weight.copy_(w[p + ".ln1.g"]), layer.norm1.bias.copy_(w[p + ".ln1.b"])
            layer.norm2.weight.copy_(w[p + ".ln2.g"]), layer.norm2.bias.copy_(w[p + ".ln2.b"])
            layer.linear1.weight.copy_(w[p + ".fc1.w"]), layer.linear1.bias.copy_(w[p + ".fc1.b"])
            layer.linear2.weight.copy_(w[p + ".fc2.w"]), layer.linear2.bias.copy_(w[p + ".fc2.b"])
        layer.eval()
        with torch.no_grad():
            x = layer(x)
    want = torch.nn.functional.layer_norm(x, (768,), w["vit.norm.g"], w["vit.norm.b"], eps=1e-6)[0, 0]
    assert torch.allclose(got, want, atol=1e-4, rtol=1e-4), float((got - want).abs().max())


def test_oracle_dpt_matches_torch_decoder_layers():
    """Pins the DP-T denoiser restatement (oracle/dp_model.py dpt_eps) against
    torch's nn.TransformerDecoderLayer (pre-norm, GELU, batch_first) with the
    same weights and DP's causal / memory masks."""
    import numpy as np
    import torch
    from oracle import dp_model
    from paper_2509_09560_b200 import diffusion as D
    cfg = D.DPConfig(name="dpt_test", encoder="vit_b16", image_hw=32, feat_dim=768, action_dim=7,
                     denoiser="transformer", dpt_layers=2, vit_depth=1)
    w = D.init_weights(cfg, 2)
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.standard_normal((16, 7)).astype(np.float32))
    gc = torch.from_numpy(rng.standard_normal(cfg.gc_dim).astype(np.float32))
    got = dp_model.dpt_eps(w, cfg, x, 37, gc)
    E = cfg.dpt_emb
    temb = dp_model._sinusoidal(37, E)
    cond = torch.nn.functional.linear(gc.reshape(2, -1), w["dpt.cond_obs.w"], w["dpt.cond_obs.b"])
    c = torch.cat([temb, cond]) + w["dpt.cond_pos"]
    mem = torch.nn.functional.linear(torch.nn.functional.mish(torch.nn.functional.linear(c, w["dpt.enc1.w"],
                                                                                          w["dpt.enc1.b"])),
                                     w["dpt.enc2.w"], w["dpt.enc2.b"])[None]
    h = (torch.nn.functional.linear(x, w["dpt.input.w"], w["dpt.input.b"]) + w["dpt.pos"])[None]
    causal, mmask = dp_model.dpt_masks(16, 3)
    for l in range(2):
        p = f"dpt.l{l}"
        layer = torch.nn.TransformerDecoderLayer(E, 4, 4 * E, dropout=0.0, activation="gelu", batch_first=True,
                                                 norm_first=True)
        with torch.no_grad():
            layer.self_attn.in_proj_weight.copy_(w[p + ".sa_in.w"]), layer.self_attn.in_proj_bias.copy_(w[p + ".sa_in.b"])
            layer.self_attn.out_proj.weight.copy_(w[p + ".sa_out.w"]), layer.self_attn.out_proj.bias.copy_(w[p + ".sa_out.b"])
            layer.multihead_attn.in_proj_weight.copy_(w[p + ".ca_in.w"])
            layer.multihead_attn.in_proj_bias.copy_(w[p + ".ca_in.b"])
            layer.multihead_attn.out_proj.weight.copy_(w[p + ".ca_out.w"])
            layer.multihead_attn.out_proj.bias.copy_(w[p + ".ca_out.b"])
            for i in (1, 2, 3):
                getattr(layer, f"norm{i}").weight.copy_(w[p + f".ln{i}.g"])
                getattr(layer, f"norm{i}").bias.copy_(w[p + f".ln{i}.b"])
            layer.linear1.weight.copy_(w[p + ".ff1.w"]), layer.linear1.bias.copy_(w[p + ".ff1.b"])
            layer.linear2.weight.copy_(w[p + ".ff2.w"]), layer.linear2.bias.copy_(w[p + ".ff2.b"])
        layer.eval()
        with torch.no_grad():
            h = layer(h, mem, tgt_mask=causal, memory_mask=mmask)
    h = torch.nn.functional.layer_norm(h[0], (E,), w["dpt.lnf.g"], w["dpt.lnf.b"])
    want = torch.nn.functional.linear(h, w["dpt.head.w"], w["dpt.head.b"])
    assert torch.allclose(got, want, atol=1e-4, rtol=1e-4), float((got - want).abs().max())


def test_dpt_cross_attention_fold_algebra():
    """The folded cross-attention of the persistent DP-T kernel (DP_XATTN phase,
    auras_dpt_xfold tables; include/auras_b200.h) is the decoder layer's
    h + ca_out(MHA(LN2(h), mem)) exactly, in exact arithmetic: query projection
    and LayerNorm affine folded into per-(head, memory token) vectors a', c',
    output projection and bias into U'.  Checked in fp64 against the oracle's
    nn.MultiheadAttention restatement with TransformerForDiffusion's memory mask."""
    import math
    import torch
    from oracle import dp_model
    torch.manual_seed(0)
    E, H, T, nk = 256, 4, 16, 3
    dh = E // H
    d = dict(dtype=torch.float64)
    w_in, b_in = torch.randn(3 * E, E, **d) / 16, torch.randn(3 * E, **d) / 4
    w_out, b_out = torch.randn(E, E, **d) / 16, torch.randn(E, **d) / 4
    g, b = 1 + torch.randn(E, **d) / 4, torch.randn(E, **d) / 4
    h = torch.randn(T, E, **d)
    mem = torch.randn(nk, E, **d)
    _, mmask = dp_model.dpt_masks(T, nk)
    want = h + dp_model._mha(torch.nn.functional.layer_norm(h, (E,), g, b, 1e-5), mem, w_in, b_in, w_out, b_out, H,
                             mmask.to(torch.float64))
    # the fold (auras_dpt_xfold's formulas)
    k = mem @ w_in[E:2 * E].T + b_in[E:2 * E]
    v = mem @ w_in[2 * E:].T + b_in[2 * E:]
    a = torch.einsum("hde,jhd->jhe", w_in[:E].reshape(H, dh, E), k.reshape(nk, H, dh)) / math.sqrt(dh)
    a_p = a * g
    c_p = (a * b).sum(-1) + (b_in[:E].reshape(H, dh) * k.reshape(nk, H, dh)).sum(-1) / math.sqrt(dh)
    u_p = torch.einsum("ehd,jhd->jhe", w_out.reshape(E, H, dh), v.reshape(nk, H, dh)) + b_out / H
    # the phase (dp_xattn): xhat, scores, masked per-head softmax, combination
    xh = (h - h.mean(-1, keepdim=True)) / torch.sqrt(h.var(-1, unbiased=False, keepdim=True) + 1e-5)
    sc = torch.einsum("te,jhe->thj", xh, a_p) + c_p.T[None]
    vis = torch.arange(nk)[None, :] <= torch.arange(T)[:, None] + 1          # key j visible iff j <= t + 1
    sc = sc.masked_fill(~vis[:, None, :], float("-inf"))
    p = torch.softmax(sc, dim=-1)
    got = h + torch.einsum("thj,jhe->te", p, u_p)
    assert torch.allclose(got, want, rtol=1e-10, atol=1e-10), (got - want).abs().max()
