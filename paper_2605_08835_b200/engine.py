"""Python wrapper around the C-ABI engine for torch-allocated buffers (marshalling only).

torch provides device memory and streams; every computation happens in libsynerdiff.so.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import binding as B


def _stream(s):
    if s is None:
        s = torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Engine:
    def __init__(self, model="tiny", sampler="ddim", max_latent_hw=None, b_max=8, c_max=16, weight_seed=0,
                 device=0, precision="fp16"):
        """precision: "fp16" (the product default, SD_PREC_FP16: fp16 operands / activations, the bf16-valued
        weights held exactly), "bf16" (SD_PREC_BF16: the same kernels with bf16 operands / activations) or
        "fp32" (the parity mode, SD_PREC_FP32)."""
        m = {"tiny": B.SD_MODEL_TINY, "sd15": B.SD_MODEL_SD15, "sdxl": B.SD_MODEL_SDXL,
             "tinyxl": B.SD_MODEL_TINY_XL}[model]
        sm = {"ddim": B.SD_SAMPLER_DDIM, "euler": B.SD_SAMPLER_EULER}[sampler]
        tiny = model in ("tiny", "tinyxl")
        if max_latent_hw is None:
            max_latent_hw = 8 if tiny else (128 if model == "sdxl" else 64)
        prec = {"bf16": B.SD_PREC_BF16, "fp16": B.SD_PREC_FP16, "fp32": B.SD_PREC_FP32}[precision]
        cfg = B.EngineConfig(m, prec, sm, max_latent_hw, b_max, c_max, weight_seed)
        h = C.c_void_p()
        B.call("sd_engine_create", C.byref(cfg), device, C.byref(h))
        self.h = h
        self.model = model
        self.b_max = b_max
        self.precision = precision
        self.sampler = sampler
        self.device = device
        self.ctx_len, self.ctx_dim, self.pooled_dim = {"tiny": (8, 32, 0), "sd15": (77, 768, 0),
                                                       "sdxl": (77, 2048, 1280), "tinyxl": (8, 48, 40)}[model]
        self.upscale = 2 if tiny else 8      # VAE decoder: 2^(levels-1)

    def close(self):
        if self.h:
            B.lib().sd_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_weight(self, name, values):
        """sd_engine_set_weight: host fp32 values in the parameter's PyTorch layout (numpy or torch CPU)."""
        import numpy as np
        a = np.ascontiguousarray(np.asarray(values, dtype=np.float32))
        B.call("sd_engine_set_weight", self.h, name.encode(), C.c_void_p(a.ctypes.data), a.nbytes)

    def launch_count(self):
        v = C.c_int64()
        B.call("sd_engine_launch_count", self.h, C.byref(v))
        return v.value

    def warmup(self, h, w, max_req=None, n_dec=0, stream=None):
        """sd_engine_warmup: capture every step-shape graph at h×w and pool n_dec decode states."""
        B.call("sd_engine_warmup", self.h, h, w, self.b_max if max_req is None else max_req, n_dec, _stream(stream))

    def profile(self, enable: bool):
        B.call("sd_engine_profile", self.h, 1 if enable else 0)

    def profile_read(self, cls: int):
        """(ms, launches, work) for kernel class cls (0 conv, 1 gemm, 2 attention, 3 GN, 4 LN)."""
        ms, n, w = C.c_double(), C.c_int64(), C.c_double()
        B.call("sd_engine_profile_read", self.h, cls, C.byref(ms), C.byref(n), C.byref(w))
        return ms.value, n.value, w.value

    def _dev(self, t):
        return t.to(device=f"cuda:{self.device}", dtype=torch.float32).contiguous()

    def set_uncond(self, emb: torch.Tensor, pooled: torch.Tensor = None, stream=None):
        emb = self._dev(emb)
        if self.pooled_dim:
            pooled = self._dev(pooled)
            B.call("sd_ctx_set_uncond_pooled", self.h, B._p(emb), emb.shape[0], emb.shape[1], B._p(pooled),
                   pooled.numel(), _stream(stream))
        else:
            B.call("sd_ctx_set_uncond", self.h, B._p(emb), emb.shape[0], emb.shape[1], _stream(stream))
        torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()

    def register(self, emb: torch.Tensor, pooled: torch.Tensor = None, stream=None) -> int:
        emb = self._dev(emb)
        slot = C.c_int32()
        if self.pooled_dim:
            pooled = self._dev(pooled)
            B.call("sd_ctx_register_pooled", self.h, B._p(emb), emb.shape[0], emb.shape[1], B._p(pooled),
                   pooled.numel(), C.byref(slot), _stream(stream))
        else:
            B.call("sd_ctx_register", self.h, B._p(emb), emb.shape[0], emb.shape[1], C.byref(slot), _stream(stream))
        (torch.cuda.current_stream() if stream is None else stream).synchronize()
        return slot.value

    def release(self, slot: int):
        B.call("sd_ctx_release", self.h, slot)

    def init_sigma(self, n_steps: int) -> float:
        v = C.c_float()
        B.call("sd_sampler_init_sigma", self.h, n_steps, C.byref(v))
        return v.value

    @staticmethod
    def _batch(latents, steps, n_steps, has_uncond, guidance, slots):
        n = len(latents)
        h, w = latents[0].shape[-2:]
        ptrs = (C.c_void_p * n)(*[t.data_ptr() for t in latents])
        b = B.Batch(n, h, w, C.cast(ptrs, C.POINTER(C.c_void_p)),
                    (C.c_int32 * n)(*steps), (C.c_int32 * n)(*n_steps), (C.c_uint8 * n)(*[int(x) for x in has_uncond]),
                    (C.c_float * n)(*guidance), (C.c_int32 * n)(*slots) if slots is not None else None)
        return b, ptrs

    def step(self, latents, steps, n_steps, has_uncond, guidance, slots, stream=None):
        """One sd_step_batch call. latents: list of cuda fp32 [4,h,w] tensors (updated in place)."""
        b, _keep = self._batch(latents, steps, n_steps, has_uncond, guidance, slots)
        B.call("sd_step_batch", self.h, C.byref(b), _stream(stream))

    def step_eps(self, latents, steps, n_steps, has_uncond, guidance, slots, stream=None):
        """sd_debug_step_eps: the UNet ε of every row of this step (cond rows, then uncond rows, R26),
        returned as fp32 [rows, 4, h, w]; the latents are not updated."""
        b, _keep = self._batch(latents, steps, n_steps, has_uncond, guidance, slots)
        h, w = latents[0].shape[-2:]
        rows = len(latents) + sum(1 for x in has_uncond if x)
        eps = torch.empty(rows, h, w, 4, device=latents[0].device, dtype=torch.float32)
        B.call("sd_debug_step_eps", self.h, C.byref(b), B._p(eps), _stream(stream))
        return eps.permute(0, 3, 1, 2)

    def combine_update(self, latents, steps, n_steps, has_uncond, guidance, eps, stream=None):
        """sd_debug_combine_update: the K12 kernel alone with an injected ε (fp32 [rows, 4, h, w], rows
        as sd_step_batch forms them); latents are updated in place."""
        b, _keep = self._batch(latents, steps, n_steps, has_uncond, guidance, None)
        e = eps.permute(0, 2, 3, 1).contiguous()
        B.call("sd_debug_combine_update", self.h, C.byref(b), B._p(e), _stream(stream))
        (torch.cuda.current_stream() if stream is None else stream).synchronize()

    def decode(self, latent: torch.Tensor, n_chunks=1, image=None, stream=None):
        """Whole or chunked VAE decode of one fp32 [4,h,w] latent → fp32 [3,8h,8w]."""
        h, w = latent.shape[-2:]
        if image is None:
            f = self.upscale
            image = torch.empty(3, f * h, f * w, device=latent.device, dtype=torch.float32)
        st = C.c_void_p()
        for j in range(n_chunks):
            self.decode_chunk(latent, n_chunks, j, st, image, stream)
        return image

    def decode_tiled(self, latent: torch.Tensor, tile: int, halo: int, image=None, stream=None):
        """V2 independent-tile decode (an approximation; sd_vae_decode_tiled)."""
        h, w = latent.shape[-2:]
        if image is None:
            f = self.upscale
            image = torch.empty(3, f * h, f * w, device=latent.device, dtype=torch.float32)
        B.call("sd_vae_decode_tiled", self.h, B._p(latent), h, w, tile, halo, B._p(image), _stream(stream))
        return image

    def decode_chunk(self, latent, n_chunks, chunk, state: C.c_void_p, image, stream=None):
        h, w = latent.shape[-2:]
        B.call("sd_vae_decode_chunked", self.h, B._p(latent), h, w, n_chunks, chunk, C.byref(state), B._p(image),
               _stream(stream))
