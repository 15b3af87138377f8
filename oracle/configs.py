"""Model architectures for the oracle (ORACLE — test infrastructure only).

The paper names only "SDv1.5" (§IV-A-1) and "SDXL" (PAPER.md:146,
§II-A); the layer structure is SURVEY.md §8(c) R1 + Appendix C (diffusers
UNet2DConditionModel / AutoencoderKL semantics). Weights are random-init (R20)
from `synth` by parameter name, in canonical PyTorch layout.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

import synth


@dataclass(frozen=True)
class UNetConfig:
    name: str
    block_out: tuple            # channels per level
    attn_levels: tuple          # True where the down/up block at that level has transformers
    layers_per_block: int
    groups: int
    heads: int
    ctx_dim: int
    ctx_len: int
    in_ch: int = 4
    out_ch: int = 4
    eps_resnet: float = 1e-5    # R29
    eps_tf_gn: float = 1e-6
    eps_ln: float = 1e-5
    out_gain: float = 1.0       # R21 (conv_out gain), 1 unless conditioning requires otherwise
    # SDXL generalisations (R1, App. C; diffusers UNet2DConditionModel config of SDXL-base):
    tf_depth: tuple = ()        # BasicTransformerBlocks per Transformer2DModel at each level (() → 1)
    mid_depth: int = 1          # ... in the mid block
    head_dim: int = 0           # > 0: heads = C / head_dim per level (SDXL 64); 0: `heads` everywhere
    linear_proj: bool = False   # proj_in / proj_out as Linear(C, C) (same values as a 1×1 conv)
    add_time_dim: int = 0       # > 0: "text_time" added embedding: 6 time ids × add_time_dim sinusoids
    pooled_dim: int = 0         #      ‖ pooled text embedding → Linear → SiLU → Linear → + temb

    @property
    def temb_dim(self):
        return 4 * self.block_out[0]

    def depth(self, level):
        return (self.tf_depth[level] if self.tf_depth else 1) if self.attn_levels[level] else 0

    def heads_at(self, c):
        return c // self.head_dim if self.head_dim else self.heads


@dataclass(frozen=True)
class VAEConfig:
    name: str
    block_out: tuple            # encoder order (e.g. 128, 256, 512, 512); decoder uses reversed
    layers_per_block: int
    groups: int
    scaling_factor: float
    latent_ch: int = 4
    out_ch: int = 3
    eps: float = 1e-6


# CFG#1 tiny config (BASELINE.json configs[0]; SURVEY §8(d) CFG#1)
TINY_UNET = UNetConfig("tiny", block_out=(32, 64), attn_levels=(True, True), layers_per_block=1,
                       groups=8, heads=2, ctx_dim=32, ctx_len=8)
TINY_VAE = VAEConfig("tiny", block_out=(32, 64), layers_per_block=1, groups=8, scaling_factor=0.18215)

# SD-1.5 (App. C): block_out (320,640,1280,1280), CrossAttnDown×3 + Down, 8 heads, ctx 77×768
SD15_UNET = UNetConfig("sd15", block_out=(320, 640, 1280, 1280), attn_levels=(True, True, True, False),
                       layers_per_block=2, groups=32, heads=8, ctx_dim=768, ctx_len=77)
SD_VAE = VAEConfig("sd", block_out=(128, 256, 512, 512), layers_per_block=2, groups=32,
                   scaling_factor=0.18215)

# SDXL-base (PAPER.md:146 names SDXL; R1): block_out (320, 640, 1280), DownBlock2D + 2 CrossAttnDown,
# transformer depth (0, 2, 10) (mid 10), head dim 64, ctx 77×2048, linear projections, "text_time"
# added embedding (6 time ids × 256 ‖ pooled 1280 → 2816 → 1280). The VAE is the SD decoder with
# scaling factor 0.13025.
SDXL_UNET = UNetConfig("sdxl", block_out=(320, 640, 1280), attn_levels=(False, True, True), layers_per_block=2,
                       groups=32, heads=0, ctx_dim=2048, ctx_len=77, tf_depth=(0, 2, 10), mid_depth=10,
                       head_dim=64, linear_proj=True, add_time_dim=256, pooled_dim=1280)
SDXL_VAE = VAEConfig("sdxl", block_out=(128, 256, 512, 512), layers_per_block=2, groups=32,
                     scaling_factor=0.13025)
# tiny SDXL-shaped config for parity (same code paths: no attention at level 0, depth 2 transformers,
# head-dim heads, linear projections, added embedding)
TINY_XL_UNET = UNetConfig("tinyxl", block_out=(32, 64), attn_levels=(False, True), layers_per_block=1,
                          groups=8, heads=0, ctx_dim=48, ctx_len=8, tf_depth=(0, 2), mid_depth=2,
                          head_dim=16, linear_proj=True, add_time_dim=8, pooled_dim=40)
SDXL_TIME_IDS = (1024, 1024, 0, 0, 1024, 1024)   # R27: original size, crop top-left, target size


# --------------------------------------------------------------------------------------------
# parameter specs: (name, shape, kind, fan_in)
# --------------------------------------------------------------------------------------------
U, G, B = synth.KIND_UNIFORM_FANIN, synth.KIND_NORM_GAMMA, synth.KIND_NORM_BETA


def _conv(p, cout, cin, k, bias=True):
    fan = cin * k * k
    out = [(p + ".weight", (cout, cin, k, k), U, fan)]
    if bias:
        out.append((p + ".bias", (cout,), U, fan))
    return out


def _lin(p, cout, cin, bias=True):
    out = [(p + ".weight", (cout, cin), U, cin)]
    if bias:
        out.append((p + ".bias", (cout,), U, cin))
    return out


def _norm(p, c):
    return [(p + ".weight", (c,), G, 1), (p + ".bias", (c,), B, 1)]


def _resnet(p, cin, cout, temb_dim):
    s = _norm(p + ".norm1", cin) + _conv(p + ".conv1", cout, cin, 3)
    if temb_dim:
        s += _lin(p + ".time_emb_proj", cout, temb_dim)
    s += _norm(p + ".norm2", cout) + _conv(p + ".conv2", cout, cout, 3)
    if cin != cout:
        s += _conv(p + ".conv_shortcut", cout, cin, 1)
    return s


def _transformer(p, c, ctx_dim, depth=1, linear_proj=False):
    proj = (lambda q: _lin(q, c, c)) if linear_proj else (lambda q: _conv(q, c, c, 1))
    s = _norm(p + ".norm", c) + proj(p + ".proj_in")
    for d in range(depth):
        b = p + f".transformer_blocks.{d}"
        s += _norm(b + ".norm1", c)
        s += _lin(b + ".attn1.to_q", c, c, False) + _lin(b + ".attn1.to_k", c, c, False)
        s += _lin(b + ".attn1.to_v", c, c, False) + _lin(b + ".attn1.to_out.0", c, c)
        s += _norm(b + ".norm2", c)
        s += _lin(b + ".attn2.to_q", c, c, False) + _lin(b + ".attn2.to_k", c, ctx_dim, False)
        s += _lin(b + ".attn2.to_v", c, ctx_dim, False) + _lin(b + ".attn2.to_out.0", c, c)
        s += _norm(b + ".norm3", c)
        s += _lin(b + ".ff.net.0.proj", 8 * c, c) + _lin(b + ".ff.net.2", c, 4 * c)
    s += proj(p + ".proj_out")
    return s


def unet_structure(cfg: UNetConfig):
    """Block structure (diffusers UNet2DConditionModel.__init__ channel bookkeeping)."""
    C = cfg.block_out
    L = len(C)
    down = []
    out_ch = C[0]
    for i in range(L):
        in_ch, out_ch = out_ch, C[i]
        res = [(in_ch if j == 0 else out_ch, out_ch) for j in range(cfg.layers_per_block)]
        down.append(dict(res=res, attn=cfg.attn_levels[i], down=(i != L - 1), ch=out_ch))
    rev = list(reversed(C))
    rattn = list(reversed(cfg.attn_levels))
    up = []
    out_ch = rev[0]
    for i in range(L):
        prev, out_ch = out_ch, rev[i]
        in_ch = rev[min(i + 1, L - 1)]
        nl = cfg.layers_per_block + 1
        res = []
        for j in range(nl):
            skip = in_ch if j == nl - 1 else out_ch
            rin = prev if j == 0 else out_ch
            res.append((rin + skip, out_ch))
        up.append(dict(res=res, attn=rattn[i], up=(i != L - 1), ch=out_ch))
    return down, up


def unet_param_specs(cfg: UNetConfig):
    C = cfg.block_out
    T = cfg.temb_dim
    s = _conv("conv_in", C[0], cfg.in_ch, 3)
    s += _lin("time_embedding.linear_1", T, C[0]) + _lin("time_embedding.linear_2", T, T)
    if cfg.add_time_dim:
        s += _lin("add_embedding.linear_1", T, 6 * cfg.add_time_dim + cfg.pooled_dim) + _lin("add_embedding.linear_2", T, T)
    down, up = unet_structure(cfg)
    L = len(C)
    tf = lambda name, c, depth: _transformer(name, c, cfg.ctx_dim, depth, cfg.linear_proj)
    for i, blk in enumerate(down):
        for j, (ci, co) in enumerate(blk["res"]):
            s += _resnet(f"down_blocks.{i}.resnets.{j}", ci, co, T)
            if blk["attn"]:
                s += tf(f"down_blocks.{i}.attentions.{j}", co, cfg.depth(i))
        if blk["down"]:
            s += _conv(f"down_blocks.{i}.downsamplers.0.conv", blk["ch"], blk["ch"], 3)
    cm = C[-1]
    s += _resnet("mid_block.resnets.0", cm, cm, T)
    s += tf("mid_block.attentions.0", cm, cfg.mid_depth)
    s += _resnet("mid_block.resnets.1", cm, cm, T)
    for i, blk in enumerate(up):
        for j, (ci, co) in enumerate(blk["res"]):
            s += _resnet(f"up_blocks.{i}.resnets.{j}", ci, co, T)
            if blk["attn"]:
                s += tf(f"up_blocks.{i}.attentions.{j}", co, cfg.depth(L - 1 - i))
        if blk["up"]:
            s += _conv(f"up_blocks.{i}.upsamplers.0.conv", blk["ch"], blk["ch"], 3)
    s += _norm("conv_norm_out", C[0]) + _conv("conv_out", cfg.out_ch, C[0], 3)
    return s


def vae_structure(cfg: VAEConfig):
    rev = list(reversed(cfg.block_out))
    ups = []
    out_ch = rev[0]
    for i in range(len(rev)):
        prev, out_ch = out_ch, rev[i]
        nl = cfg.layers_per_block + 1
        res = [(prev if j == 0 else out_ch, out_ch) for j in range(nl)]
        ups.append(dict(res=res, up=(i != len(rev) - 1), ch=out_ch))
    return ups


def vae_param_specs(cfg: VAEConfig):
    cm = cfg.block_out[-1]
    s = _conv("post_quant_conv", cfg.latent_ch, cfg.latent_ch, 1)
    s += _conv("decoder.conv_in", cm, cfg.latent_ch, 3)
    s += _resnet("decoder.mid_block.resnets.0", cm, cm, 0)
    a = "decoder.mid_block.attentions.0"
    s += _norm(a + ".group_norm", cm)
    s += _lin(a + ".to_q", cm, cm) + _lin(a + ".to_k", cm, cm) + _lin(a + ".to_v", cm, cm)
    s += _lin(a + ".to_out.0", cm, cm)
    s += _resnet("decoder.mid_block.resnets.1", cm, cm, 0)
    for i, blk in enumerate(vae_structure(cfg)):
        for j, (ci, co) in enumerate(blk["res"]):
            s += _resnet(f"decoder.up_blocks.{i}.resnets.{j}", ci, co, 0)
        if blk["up"]:
            s += _conv(f"decoder.up_blocks.{i}.upsamplers.0.conv", blk["ch"], blk["ch"], 3)
    s += _norm("decoder.conv_norm_out", cfg.block_out[0])
    s += _conv("decoder.conv_out", cfg.out_ch, cfg.block_out[0], 3)
    return s


def make_params(specs, seed: int, dtype=np.float32, bf16_weights: bool = False, gains=None):
    """name -> array. bf16_weights=True rounds matrices (ndim>=2) to bf16 RNE, i.e. the values
    the GPU stores (R20: "the bf16-mode oracle uses those same rounded values upcast")."""
    gains = gains or {}
    out = {}
    for name, shape, kind, fan in specs:
        w = synth.weight(seed, name, shape, kind, fan, gains.get(name, 1.0))
        if bf16_weights and len(shape) >= 2:
            w = synth.bf16_round(w)
        out[name] = w.astype(dtype)
    return out


def unet_params(cfg: UNetConfig, seed: int, dtype=np.float32, bf16_weights=False):
    gains = {"conv_out.weight": cfg.out_gain, "conv_out.bias": cfg.out_gain}
    return make_params(unet_param_specs(cfg), seed, dtype, bf16_weights, gains)


def vae_params(cfg: VAEConfig, seed: int, dtype=np.float32, bf16_weights=False):
    return make_params(vae_param_specs(cfg), seed, dtype, bf16_weights)
