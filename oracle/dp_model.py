"""torch-CPU fp32 restatement of the Diffusion Policy CNN (TEST ORACLE).

PARITY UNPINNED BY THE REFERENCE: the reference (/root/reference) contains no
neural network -- its "diffusion" generator is x <- x + eta (H - x)
(fp/policy.py:220-225).  The networks named by BASELINE.json's north_star
(ResNet-18 encoder, ConditionalUnet1D, DDPM/DDIM) live in third-party code
absent from /root/reference and from this image:

* diffusion_policy (Chi et al., RSS 2023; public release, `ConditionalUnet1D`,
  `ConditionalResidualBlock1D`, `Conv1dBlock`, `SinusoidalPosEmb`,
  `replace_bn_with_gn`, `MultiImageObsEncoder`);
* diffusers' `DDPMScheduler` / `DDIMScheduler` (squaredcos_cap_v2 betas,
  epsilon prediction, clip_sample, fixed_small variance; DDIM eta = 0 with
  "leading" timestep spacing and set_alpha_to_one).

This module restates their published algorithms with plain torch ops in the
layouts PyTorch uses (NCHW / NCT, conv weights [out, in, k...]), independently
of the product's kernels, and plugs them into the restated reference scheduler
(oracle/schedule.py, pinned bit-exact to the reference) through the
reference's duck-typed Policy interface (fp/executor.py:216-330).  The
schedule -- which context version each denoise step reads -- is therefore
pinned; the network arithmetic is pinned only by this restatement.

Stated conventions shared with the product (so the two see identical inputs):
frames u8 -> x/127.5 - 1; global_cond = n_obs_steps x [resnet feature,
agent_pos] with the previous publish (or the current one at the first
publish) as the older step; request randomness from
numpy default_rng((seed, agent, birth_frame)): x_T then one draw per DDPM step;
synthetic frames from default_rng((seed, agent, frame, 7)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F

RESNET = ((64, 1), (128, 2), (256, 2), (512, 2))


def _mish(x):
    return x * torch.tanh(F.softplus(x))


def _id(x):
    return x


def _bf16(x):
    """Round to bf16 (round-to-nearest-even) and back: a tensor stored in bf16."""
    return x.to(torch.bfloat16).to(torch.float32)


# Weights the B200 bf16 path holds in bf16 (the tensor-core operands and the
# FiLM / time-MLP GEMV weights); everything else (biases, GroupNorm affine,
# the final 1x1 output conv, the ViT / DP-T transformers) stays fp32.
_BF16_WEIGHT_SUFFIXES = (".w",)
_FP32_WEIGHTS = ("unet.final.out.w",)


def bf16_weights(w):
    """The bf16-faithful oracle's weight dict: every conv / FiLM / time-MLP
    weight of the CNN policy rounded to bf16 exactly as
    DeviceModel.conv_weight / Denoiser._build_tables store them."""
    out = {}
    for k, v in w.items():
        cnn = k.startswith("enc.") or k.startswith("unet.")
        if cnn and k.endswith(_BF16_WEIGHT_SUFFIXES) and k not in _FP32_WEIGHTS:
            out[k] = _bf16(v)
        else:
            out[k] = v
    return out


def _gn(x, w, name, groups):
    return F.group_norm(x, groups, w[name + ".g"], w[name + ".b"], eps=1e-5)


# ---------------------------------------------------------------- perception

def encode_vit(w, img_u8: np.ndarray, pos) -> torch.Tensor:
    """ViT-B/16 in timm's layout (BASELINE configs[3] perception; parity
    unpinned by the reference, which has no vision model; the block wiring is
    pinned against torch's nn.TransformerEncoderLayer in
    tests/test_dp_host.py): patch conv 16/16,
    [CLS; patches] + position embedding, 12 pre-norm blocks (LayerNorm eps
    1e-6, softmax(q k^T / sqrt(dh)) v over 12 heads, exact-GELU MLP), final
    LayerNorm; feature = the CLS row -> [768 feature, agent_pos]."""
    x = torch.from_numpy(np.asarray(img_u8)).float()[None] * (2.0 / 255.0) - 1.0
    D = w["vit.cls"].numel()
    x = F.conv2d(x, w["vit.patch.w"], w["vit.patch.b"], stride=w["vit.patch.w"].shape[-1])
    x = x.flatten(2).transpose(1, 2)                                # [1, n, D]
    x = torch.cat([w["vit.cls"].reshape(1, 1, D), x], dim=1) + w["vit.pos"][None]
    N = x.shape[1]
    depth = sum(1 for k in w if k.startswith("vit.b") and k.endswith(".qkv.w"))
    heads = 12
    for i in range(depth):
        p = f"vit.b{i}"
        a = F.layer_norm(x, (D,), w[p + ".ln1.g"], w[p + ".ln1.b"], eps=1e-6)
        qkv = F.linear(a, w[p + ".qkv.w"], w[p + ".qkv.b"]).reshape(1, N, 3, heads, D // heads).permute(2, 0, 3, 1, 4)
        q, k, v = qkv[0], qkv[1], qkv[2]
        att = torch.softmax((q * (D // heads) ** -0.5) @ k.transpose(-2, -1), dim=-1) @ v
        x = x + F.linear(att.transpose(1, 2).reshape(1, N, D), w[p + ".proj.w"], w[p + ".proj.b"])
        a = F.layer_norm(x, (D,), w[p + ".ln2.g"], w[p + ".ln2.b"], eps=1e-6)
        x = x + F.linear(F.gelu(F.linear(a, w[p + ".fc1.w"], w[p + ".fc1.b"])), w[p + ".fc2.w"], w[p + ".fc2.b"])
    x = F.layer_norm(x, (D,), w["vit.norm.g"], w["vit.norm.b"], eps=1e-6)
    return torch.cat([x[0, 0], torch.as_tensor(np.asarray(pos, dtype=np.float32))])


def encode(w, img_u8: np.ndarray, pos, store=_id) -> torch.Tensor:
    """ResNet-18 with GroupNorm(C/16) and no fc -> [512 feature, agent_pos]
    (the ViT-B/16 encoder when the weights hold one).  `store` is applied
    wherever the device stores an activation tensor (identity: fp32 oracle;
    _bf16: the bf16-faithful oracle -- the image, every block output; the
    pooled feature is averaged from the unrounded fp32 epilogue values)."""
    if "vit.patch.w" in w:
        return encode_vit(w, img_u8, pos)
    x = store(torch.from_numpy(np.asarray(img_u8)).float()[None] * (2.0 / 255.0) - 1.0)
    x = store(F.relu(_gn(F.conv2d(x, w["enc.conv1.w"], stride=2, padding=3), w, "enc.gn1", 4)))
    x = F.max_pool2d(x, 3, 2, 1)
    n_blocks = 2 * len(RESNET)
    for li, (c, stride) in enumerate(RESNET, start=1):
        for bi in range(2):
            p = f"enc.layer{li}.{bi}"
            s = stride if bi == 0 else 1
            y = store(F.relu(_gn(F.conv2d(x, w[p + ".conv1.w"], stride=s, padding=1), w, p + ".gn1", c // 16)))
            y = _gn(F.conv2d(y, w[p + ".conv2.w"], padding=1), w, p + ".gn2", c // 16)
            idt = x
            if p + ".ds.w" in w:
                idt = store(_gn(F.conv2d(x, w[p + ".ds.w"], stride=s), w, p + ".dsgn", c // 16))
            x = F.relu(y + idt)
            if 2 * (li - 1) + bi + 1 < n_blocks:
                x = store(x)
    feat = x.mean(dim=(2, 3))[0]
    return torch.cat([feat, torch.as_tensor(np.asarray(pos, dtype=np.float32))])


# ---------------------------------------------------------------- denoiser

def _sinusoidal(t: int, dim: int) -> torch.Tensor:
    half = dim // 2
    scale = math.log(10000) / (half - 1)
    freqs = torch.exp(torch.arange(half, dtype=torch.float32) * -scale)
    arg = float(t) * freqs
    return torch.cat([arg.sin(), arg.cos()])[None]


def _block(w, name, x, cond, k, groups, store=_id):
    p = "unet." + name
    h = _mish(_gn(F.conv1d(x, w[p + ".c1.w"], w[p + ".c1.b"], padding=k // 2), w, p + ".g1", groups))
    e = F.linear(_mish(cond), w[p + ".film.w"], w[p + ".film.b"])
    co = h.shape[1]
    h = store(e[:, :co, None] * h + e[:, co:, None])
    h = _mish(_gn(F.conv1d(h, w[p + ".c2.w"], w[p + ".c2.b"], padding=k // 2), w, p + ".g2", groups))
    res = F.conv1d(x, w[p + ".res.w"], w[p + ".res.b"]) if p + ".res.w" in w else x
    return store(h + res)


def unet_eps(w, cfg, x: torch.Tensor, timestep: int, gc: torch.Tensor, store=_id) -> torch.Tensor:
    """ConditionalUnet1D forward: x (horizon, action_dim) -> eps (horizon, action_dim).

    `store` is applied wherever the device stores an activation tensor:
    identity for the fp32 oracle; _bf16 for the bf16-faithful oracle, which
    with bf16_weights() reproduces the tensor-core path's rounding points --
    the conv input x_t, each block's conv1 (GN, Mish, FiLM) and conv2 (GN,
    Mish, + residual) outputs, down/up-sampling outputs and the final block's
    output; the 1x1 residual conv output, FiLM rows, GroupNorm statistics,
    accumulation, eps and the scheduler update stay fp32."""
    k, g = cfg.kernel_size, cfg.n_groups
    temb = F.linear(_mish(F.linear(_sinusoidal(timestep, cfg.dsed), w["unet.temb.l1.w"],
                                   w["unet.temb.l1.b"])), w["unet.temb.l2.w"], w["unet.temb.l2.b"])
    cond = torch.cat([temb, gc[None]], dim=-1)
    h = store(x.T[None])
    L = len(cfg.down_dims)
    skips = []
    for i in range(L):
        h = _block(w, f"down{i}.0", h, cond, k, g, store)
        h = _block(w, f"down{i}.1", h, cond, k, g, store)
        skips.append(h)
        if i < L - 1:
            h = store(F.conv1d(h, w[f"unet.down{i}.ds.w"], w[f"unet.down{i}.ds.b"], stride=2, padding=1))
    h = _block(w, "mid.0", h, cond, k, g, store)
    h = _block(w, "mid.1", h, cond, k, g, store)
    for i in range(L - 1):
        h = torch.cat([h, skips.pop()], dim=1)
        h = _block(w, f"up{i}.0", h, cond, k, g, store)
        h = _block(w, f"up{i}.1", h, cond, k, g, store)
        h = store(F.conv_transpose1d(h, w[f"unet.up{i}.us.w"], w[f"unet.up{i}.us.b"], stride=2, padding=1))
    h = store(_mish(_gn(F.conv1d(h, w["unet.final.c.w"], w["unet.final.c.b"], padding=k // 2), w,
                        "unet.final.g", g)))
    h = F.conv1d(h, w["unet.final.out.w"], w["unet.final.out.b"])
    return h[0].T


def _mha(q_in, kv_in, w_in, b_in, w_out, b_out, heads, mask):
    """nn.MultiheadAttention's math: packed q|k|v in-projection, scaled dot
    product per head, additive -inf mask, out-projection."""
    E = q_in.shape[-1]
    q = F.linear(q_in, w_in[:E], b_in[:E])
    k = F.linear(kv_in, w_in[E:2 * E], b_in[E:2 * E])
    v = F.linear(kv_in, w_in[2 * E:], b_in[2 * E:])
    dh = E // heads
    q = q.reshape(-1, heads, dh).transpose(0, 1)
    k = k.reshape(-1, heads, dh).transpose(0, 1)
    v = v.reshape(-1, heads, dh).transpose(0, 1)
    att = torch.softmax(q @ k.transpose(-2, -1) / math.sqrt(dh) + mask, dim=-1) @ v
    return F.linear(att.transpose(0, 1).reshape(-1, E), w_out, b_out)


def dpt_masks(T: int, t_cond: int):
    """TransformerForDiffusion's masks: causal self-attention; action t sees
    cond token s (time token first) iff t >= s - 1."""
    causal = torch.full((T, T), float("-inf")).triu(1)
    t, s_ = torch.meshgrid(torch.arange(T), torch.arange(t_cond), indexing="ij")
    mem = torch.zeros(T, t_cond).masked_fill(~(t >= s_ - 1), float("-inf"))
    return causal, mem


def dpt_eps(w, cfg, x: torch.Tensor, timestep: int, gc: torch.Tensor) -> torch.Tensor:
    """Diffusion Policy's TransformerForDiffusion (time_as_cond, obs_as_cond,
    causal_attn, n_cond_layers = 0) in eval mode: x (horizon, action_dim) ->
    eps.  Parity unpinned by the reference (no network there); the layer
    wiring is pinned against torch's nn.TransformerDecoderLayer in
    tests/test_dp_host.py."""
    E, H, L = cfg.dpt_emb, cfg.dpt_heads, cfg.dpt_layers
    n_obs = cfg.n_obs_steps
    temb = _sinusoidal(timestep, E)                                      # [1, E]
    cond = F.linear(gc.reshape(n_obs, -1), w["dpt.cond_obs.w"], w["dpt.cond_obs.b"])
    c = torch.cat([temb, cond], dim=0) + w["dpt.cond_pos"]
    mem = F.linear(_mish(F.linear(c, w["dpt.enc1.w"], w["dpt.enc1.b"])), w["dpt.enc2.w"], w["dpt.enc2.b"])
    h = F.linear(x, w["dpt.input.w"], w["dpt.input.b"]) + w["dpt.pos"]
    causal, mmask = dpt_masks(x.shape[0], 1 + n_obs)
    for l in range(L):
        p = f"dpt.l{l}"
        a = F.layer_norm(h, (E,), w[p + ".ln1.g"], w[p + ".ln1.b"])
        h = h + _mha(a, a, w[p + ".sa_in.w"], w[p + ".sa_in.b"], w[p + ".sa_out.w"], w[p + ".sa_out.b"], H, causal)
        a = F.layer_norm(h, (E,), w[p + ".ln2.g"], w[p + ".ln2.b"])
        h = h + _mha(a, mem, w[p + ".ca_in.w"], w[p + ".ca_in.b"], w[p + ".ca_out.w"], w[p + ".ca_out.b"], H, mmask)
        a = F.layer_norm(h, (E,), w[p + ".ln3.g"], w[p + ".ln3.b"])
        h = h + F.linear(F.gelu(F.linear(a, w[p + ".ff1.w"], w[p + ".ff1.b"])), w[p + ".ff2.w"], w[p + ".ff2.b"])
    h = F.layer_norm(h, (E,), w["dpt.lnf.g"], w["dpt.lnf.b"])
    return F.linear(h, w["dpt.head.w"], w["dpt.head.b"])


# ---------------------------------------------------------------- scheduler

class Scheduler:
    """diffusers DDPM (fixed_small) / DDIM (eta 0) over squaredcos_cap_v2 betas."""

    def __init__(self, cfg):
        T, n = cfg.num_train_timesteps, cfg.num_inference_steps
        betas = []
        for i in range(T):
            a0 = math.cos((i / T + 0.008) / 1.008 * math.pi / 2) ** 2
            a1 = math.cos(((i + 1) / T + 0.008) / 1.008 * math.pi / 2) ** 2
            betas.append(min(1.0 - a1 / a0, 0.999))
        self.abar = np.cumprod(1.0 - np.array(betas))
        self.ratio = T // n
        self.timesteps = [int(t) for t in (np.arange(n) * self.ratio)[::-1]]
        self.kind, self.clip = cfg.scheduler, cfg.clip_sample

    def step(self, i: int, x: torch.Tensor, eps: torch.Tensor, z) -> torch.Tensor:
        t = self.timesteps[i]
        prev = t - self.ratio
        ab = float(self.abar[t])
        abp = float(self.abar[prev]) if prev >= 0 else 1.0
        x0 = (x - math.sqrt(1 - ab) * eps) / math.sqrt(ab)
        if self.clip:
            x0 = x0.clamp(-1.0, 1.0)
        if self.kind == "ddim":
            return math.sqrt(abp) * x0 + math.sqrt(1 - abp) * eps
        alpha_t = ab / abp
        beta_t = 1 - alpha_t
        out = (math.sqrt(abp) * beta_t / (1 - ab)) * x0 + (math.sqrt(alpha_t) * (1 - abp) / (1 - ab)) * x
        if t > 0:
            var = max((1 - abp) / (1 - ab) * beta_t, 1e-20)
            out = out + math.sqrt(var) * z
        return out


# ---------------------------------------------------------------- policy duck type

@dataclass(frozen=True)
class Obs:
    frame: int
    vector: np.ndarray
    image: np.ndarray

    @property
    def id(self):
        return self.frame


@dataclass(frozen=True)
class Ctx:
    payload: torch.Tensor
    produced_frame: int


@dataclass
class State:
    x: torch.Tensor
    z: object
    steps: int = 0


@dataclass(frozen=True)
class Action:
    values: tuple
    emitted_frame: int = -1
    staleness_profile: tuple = ()


def synthetic_frame(cfg, seed, agent, frame):
    rng = np.random.default_rng((seed, agent, frame, 7))
    img = rng.integers(0, 256, (cfg.image_channels, cfg.image_hw, cfg.image_hw), dtype=np.uint8)
    pos = rng.uniform(-1.0, 1.0, cfg.agent_pos_dim)
    return Obs(frame, pos, img)


class OraclePerception:
    def __init__(self, w, cfg, layer_costs, store=_id):
        self.w, self.cfg, self.store = w, cfg, store
        self.layer_costs = tuple(layer_costs)
        self.layers = self.layer_costs
        self.prev = None

    @property
    def total_cost(self):
        return float(sum(self.layer_costs))

    def start(self, obs):
        return obs

    def apply_layers(self, latent, lo, hi):
        return latent

    def finalize(self, latent, obs):
        with torch.no_grad():
            h = encode(self.w, obs.image, obs.vector, self.store)
        if self.cfg.n_obs_steps == 2:
            old = h if self.prev is None else self.prev
            gc = torch.cat([old, h])
        else:
            gc = h
        self.prev = h
        return Ctx(gc, obs.frame)

    def perceive(self, obs):
        return self.finalize(obs, obs)


class OracleGeneration:
    def __init__(self, w, cfg, seed, agent, step_cost, store=_id):
        self.w, self.cfg, self.seed, self.agent = w, cfg, seed, agent
        self.store = store
        self.sched = Scheduler(cfg)
        self.n_iterations = cfg.num_inference_steps
        self.step_cost = step_cost

    @property
    def total_cost(self):
        return self.n_iterations * self.step_cost

    def initial_state(self, seed=None):
        cfg = self.cfg
        rng = np.random.default_rng((self.seed, self.agent, seed))
        xT = rng.standard_normal((cfg.horizon, cfg.action_dim)).astype(np.float32)
        z = None
        if cfg.scheduler == "ddpm":
            z = torch.from_numpy(rng.standard_normal((cfg.num_inference_steps, cfg.horizon,
                                                      cfg.action_dim)).astype(np.float32))
        return State(torch.from_numpy(xT), z, 0)

    def step(self, state, ctx):
        i = state.steps
        with torch.no_grad():
            if "dpt.input.w" in self.w:
                eps = dpt_eps(self.w, self.cfg, state.x, self.sched.timesteps[i], ctx.payload)
            else:
                eps = unet_eps(self.w, self.cfg, state.x, self.sched.timesteps[i], ctx.payload, self.store)
            x = self.sched.step(i, state.x, eps, None if state.z is None else state.z[i])
        return State(x, state.z, i + 1)

    def finish(self, state, emitted_frame=-1, staleness_profile=()):
        assert state.steps == self.n_iterations
        return Action(tuple(float(v) for v in state.x.reshape(-1)), emitted_frame,
                      tuple(staleness_profile))

    def decode_action(self, action):
        return np.asarray(action.values)


class OracleDP:
    """Reference-duck-typed policy (one agent) for oracle/schedule.py or the
    unmodified reference scheduler (fp/executor.py:200-461)."""

    kind = "conditioning"          # compares unequal to ContextKind.AUTOREGRESSIVE

    def __init__(self, weights, cfg, seed, agent, layer_costs, step_cost, numerics="fp32"):
        """numerics "fp32": the reference-precision oracle; "bf16": the
        bf16-faithful oracle of the tensor-core path (bf16_weights + a bf16
        store at every point the device stores an activation; CNN policy)."""
        w = {k: v.detach().to("cpu", torch.float32) for k, v in weights.items()}
        store = _id
        if numerics == "bf16":
            w, store = bf16_weights(w), _bf16
        elif numerics != "fp32":
            raise ValueError(f"numerics must be fp32 or bf16, not {numerics!r}")
        self.cfg, self.seed, self.agent, self.numerics = cfg, seed, agent, numerics
        self.perception = OraclePerception(w, cfg, layer_costs, store)
        self.generation = OracleGeneration(w, cfg, seed, agent, step_cost, store)

    @property
    def sequential_cost(self):
        return self.perception.total_cost + self.generation.total_cost

    def synthetic_observation(self, frame):
        return synthetic_frame(self.cfg, self.seed, self.agent, frame)
