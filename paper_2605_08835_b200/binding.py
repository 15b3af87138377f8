"""Thin ctypes binding of include/sd_api.h (argument marshalling only — every step of the hot path
runs in libsynerdiff.so's CUDA kernels; there is no Python or CPU fallback).

Function names mirror the C ABI. Pointers are passed as ints (e.g. torch.Tensor.data_ptr()),
streams as ints (torch.cuda.Stream.cuda_stream) or None.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

_lib = None

SD_OK, SD_E_INVAL, SD_E_NOMEM, SD_E_CUDA, SD_E_AGAIN, SD_E_STATE, SD_E_NOTSUP = 0, -1, -2, -3, -4, -5, -6
SD_MODEL_TINY, SD_MODEL_SD15, SD_MODEL_SDXL, SD_MODEL_TINY_XL = 0, 1, 2, 3
SD_PREC_BF16, SD_PREC_FP32, SD_PREC_FP16 = 0, 1, 2
SD_SAMPLER_DDIM, SD_SAMPLER_EULER = 0, 1
ACT_NONE, ACT_SILU, ACT_GEGLU = 0, 1, 2


class SDError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} -> {status_str(status)} ({status}): {msg}")
        self.status = status


class EngineConfig(C.Structure):
    _fields_ = [("model", C.c_int32), ("precision", C.c_int32), ("sampler", C.c_int32),
                ("max_latent_hw", C.c_int32), ("b_max", C.c_int32), ("c_max", C.c_int32),
                ("weight_seed", C.c_uint64)]


class Batch(C.Structure):
    _fields_ = [("n_req", C.c_int32), ("latent_h", C.c_int32), ("latent_w", C.c_int32),
                ("latents", C.POINTER(C.c_void_p)), ("step", C.POINTER(C.c_int32)),
                ("n_steps", C.POINTER(C.c_int32)), ("has_uncond", C.POINTER(C.c_uint8)),
                ("guidance", C.POINTER(C.c_float)), ("ctx_slot", C.POINTER(C.c_int32))]


class ControllerConfig(C.Structure):
    _fields_ = [("c_star", C.c_int32), ("c_max", C.c_int32), ("window", C.c_int32), ("hysteresis", C.c_int32),
                ("up_num", C.c_int32), ("up_den", C.c_int32), ("down_num", C.c_int32), ("down_den", C.c_int32)]


class ServeConfig(C.Structure):
    _fields_ = [("b_max", C.c_int32), ("a_num", C.c_int32), ("a_den", C.c_int32), ("dp_mode", C.c_int32),
                ("c_star", C.c_int32), ("ctl", ControllerConfig), ("table", C.c_void_p), ("latent_hw", C.c_int32),
                ("trace_seed", C.c_uint64), ("n_max", C.c_int32), ("policy", C.c_int32), ("ablation", C.c_int32),
                ("dyn_window_us", C.c_int64), ("n_res", C.c_int32), ("res_hw", C.POINTER(C.c_int32)),
                ("res_tables", C.POINTER(C.c_void_p)), ("vae_sms", C.c_int32)]


SD_POLICY_SYNERDIFF, SD_POLICY_NAIVE, SD_POLICY_DYNAMIC, SD_POLICY_SERIAL = 0, 1, 2, 3
SD_ABL_NO_SKIP, SD_ABL_NO_CTL = 1, 2
POLICIES = {"synerdiff": SD_POLICY_SYNERDIFF, "naive": SD_POLICY_NAIVE, "dynamic": SD_POLICY_DYNAMIC,
            "serial": SD_POLICY_SERIAL}


class Request(C.Structure):
    _fields_ = [("id", C.c_uint64), ("arrival_us", C.c_int64), ("n_steps", C.c_int32), ("guidance", C.c_float),
                ("text_emb_host", C.c_void_p), ("emb_len", C.c_int32), ("emb_dim", C.c_int32),
                ("pooled_host", C.c_void_p), ("pooled_dim", C.c_int32), ("latent_hw", C.c_int32)]


class Completion(C.Structure):
    _fields_ = [("id", C.c_uint64), ("arrival_us", C.c_int64), ("denoise_done_us", C.c_int64),
                ("decode_done_us", C.c_int64), ("n_skipped", C.c_int32), ("h", C.c_int32), ("w", C.c_int32),
                ("image_host", C.c_void_p), ("skipped_steps", C.POINTER(C.c_int32))]


class LoggedUnet(C.Structure):
    _fields_ = [("id", C.c_uint64), ("s", C.c_int32), ("n_steps", C.c_int32), ("eligible", C.c_int32),
                ("stage", C.c_int32), ("skip", C.c_int32), ("pad_", C.c_int32)]


class LoggedDecode(C.Structure):
    _fields_ = [("id", C.c_uint64), ("arrival_us", C.c_int64), ("stage", C.c_int32), ("pad_", C.c_int32)]


class Directive(C.Structure):
    _fields_ = [("level", C.c_int32), ("c", C.c_int32), ("changed", C.c_int32)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)

# name -> argtypes (restype is sd_status unless listed in _RESTYPE)
SIGNATURES = {
    "sd_engine_create": [C.POINTER(EngineConfig), I32, C.POINTER(P)],
    "sd_engine_destroy": [P],
    "sd_last_error": [],
    "sd_status_str": [I32],
    "sd_engine_launch_count": [P, PI64],
    "sd_engine_set_weight": [P, C.c_char_p, P, C.c_size_t],
    "sd_engine_profile": [P, I32],
    "sd_engine_profile_read": [P, I32, C.POINTER(C.c_double), PI64, C.POINTER(C.c_double)],
    "sd_ctx_register": [P, P, I32, I32, PI32, P],
    "sd_ctx_set_uncond": [P, P, I32, I32, P],
    "sd_ctx_register_pooled": [P, P, I32, I32, P, I32, PI32, P],
    "sd_ctx_set_uncond_pooled": [P, P, I32, I32, P, I32, P],
    "sd_ctx_release": [P, I32],
    "sd_step_batch": [P, C.POINTER(Batch), P],
    "sd_sampler_init_sigma": [P, I32, C.POINTER(C.c_float)],
    "sd_vae_decode_chunked": [P, P, I32, I32, I32, I32, C.POINTER(P), P, P],
    "sd_table_load": [C.c_char_p, C.POINTER(P)],
    "sd_table_from_arrays": [I32, PI32, PI32, PI32, PI32, PI64, PI64, C.POINTER(P)],
    "sd_table_free": [P],
    "sd_plan": [P, I32, I32, I32, I32, I32, I32, I32, PI32, I32, PI32, PI64, PI64],
    "sd_controller_create": [C.POINTER(ControllerConfig), C.POINTER(P)],
    "sd_controller_decide": [P, I64, I32, C.POINTER(Directive)],
    "sd_controller_free": [P],
    "sd_chunk_ranges": [PI64, I32, I32, PI32],
    "sd_find_b_max": [P, I32, I32, I32, PI32],
    "sd_chunk_choice": [P, I32, I32, PI32, I32, I32, I32, PI32, PI32, C.POINTER(C.c_double)],
    "sd_engine_warmup": [P, I32, I32, I32, I32, P],
    "sd_vae_decode_tiled": [P, P, I32, I32, I32, I32, P, P],
    "sd_serve_start": [P, C.POINTER(ServeConfig)],
    "sd_submit": [P, C.POINTER(Request)],
    "sd_poll": [P, C.POINTER(Completion), I32, PI32, I32],
    "sd_release": [P, C.c_uint64],
    "sd_serve_stop": [P],
    "sd_serve_window_log": [P, I32, PI64, PI64, PI32, PI32, PI32, PI32, PI32, PI32, PI32, PI32, PI32],
    "sd_set_global_load": [P, PI32, I32, C.c_uint64],
    "sd_get_load": [P, PI32],
    "sd_serve_simulate": [C.POINTER(ServeConfig), P, I32, C.POINTER(C.c_uint64), PI64, PI32, PI64, PI64, PI32, PI32],
    "sd_serve_simulate_mixed": [C.POINTER(ServeConfig), I32, C.POINTER(C.c_uint64), PI64, PI32, PI32, PI64, PI64, PI32,
                                PI32],
    "sd_vserve_create": [C.POINTER(ServeConfig), P, I32, C.POINTER(C.c_uint64), PI64, PI32, C.POINTER(P)],
    "sd_vserve_window": [P, PI32],
    "sd_vserve_get_load": [P, PI32],
    "sd_vserve_set_global_load": [P, PI32, I32, C.c_uint64],
    "sd_vserve_results": [P, PI64, PI64, PI32, PI64, PI32],
    "sd_vserve_trajectory": [P, I32, PI32, PI32, PI32, PI32],
    "sd_vserve_free": [P],
    "sd_sm_partition_create": [I32, I32, C.POINTER(P), C.POINTER(P), C.POINTER(P), PI32, PI32],
    "sd_sm_partition_destroy": [P],
    "sd_map_tasks": [PI32, I32, I32, C.POINTER(C.c_uint64), PI32, PI32, C.POINTER(C.c_uint8), I32,
                     C.POINTER(C.c_uint64), PI64, PI32, C.POINTER(C.c_uint8), PI32],
    "sd_serve_window_plan": [P, I32, PI32, I32, PI32, C.POINTER(LoggedUnet), I32, PI32, C.POINTER(LoggedDecode), I32,
                             PI32, PI32, PI32],
    "sd_vserve_window_plan": [P, I32, PI32, I32, PI32, C.POINTER(LoggedUnet), I32, PI32, C.POINTER(LoggedDecode),
                              I32, PI32, PI32, PI32],
    "sd_debug_gemm": [P, P, P, P, I32, I32, I32, I32, I32, P],
    "sd_debug_gemm_res": [P, P, P, P, I32, P, I32, I32, I32, P],
    "sd_debug_set_gemm_cg": [I32],
    "sd_debug_set_f16": [I32],
    "sd_debug_set_conv_splits": [I32],
    "sd_debug_attention": [P, P, P, P, I32, I32, I32, I32, I32, P],
    "sd_debug_attention_tc": [P, P, P, I32, I32, I32, I32, I32, P],
    "sd_debug_xattention_tc": [P, P, I32, I32, I32, P, I32, I32, I32, P, I32, P, I32, I32, I32, I32, I32, P],
    "sd_debug_groupnorm": [P, P, I32, I32, I32, I32, P, P, C.c_float, I32, P],
    "sd_debug_layernorm": [P, P, I32, I32, P, P, C.c_float, P],
    "sd_debug_conv3x3": [P, I32, P, I32, P, P, P, P, P, P, I32, I32, I32, I32, P],
    "sd_debug_conv3x3_s2": [P, I32, P, P, P, I32, I32, I32, I32, P],
    "sd_debug_conv3x3_gn": [P, I32, P, P, P, P, I32, I32, I32, I32, P, P],
    "sd_debug_gemm_gn": [P, P, P, P, P, I32, I32, I32, I32, P, P],
    "sd_debug_gemm_ln": [P, I32, P, I32, I32, P, P, P, P, C.c_float, I32, I32, P],
    "sd_debug_groupnorm_parts": [P, I32, P, P, I32, P, P, I32, I32, I32, P, P, C.c_float, I32, P],
    "sd_debug_step_eps": [P, C.POINTER(Batch), P, P],
    "sd_debug_combine_update": [P, C.POINTER(Batch), P, P],
}
_RESTYPE = {"sd_last_error": C.c_char_p, "sd_status_str": C.c_char_p}


def lib():
    """Load libsynerdiff.so. Fails loudly if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built: run `python -m paper_2605_08835_b200.build` "
                              "(or __graft_entry__.build()) — there is no CPU fallback")
        L = C.CDLL(LIB)
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RESTYPE.get(name, C.c_int32)
        _lib = L
    return _lib


def status_str(s):
    return lib().sd_status_str(s).decode()


def last_error():
    return lib().sd_last_error().decode()


def check(fn, status):
    if status != SD_OK:
        raise SDError(fn, status, last_error())
    return status


def call(name, *args):
    return check(name, getattr(lib(), name)(*args))


def window_plan(fn, handle, window):
    """sd_serve_window_plan / sd_vserve_window_plan → (level, c, stages, [unet records], [decode records]):
    unet (id, s, n_steps, eligible, stage, skip) in batch order, decode (id, arrival_us, stage) in (A, id) order."""
    st = (C.c_int32 * 96)()
    us = (LoggedUnet * 32)()
    ds = (LoggedDecode * 32)()
    ns, nu, nd, lv, c = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    call(fn, handle, window, st, 32, C.byref(ns), us, 32, C.byref(nu), ds, 32, C.byref(nd), C.byref(lv), C.byref(c))
    stages = tuple(tuple(st[3 * i:3 * i + 3]) for i in range(ns.value))
    unet = [(u.id, u.s, u.n_steps, u.eligible, u.stage, u.skip) for u in us[:nu.value]]
    dec = [(d.id, d.arrival_us, d.stage) for d in ds[:nd.value]]
    return lv.value, c.value, stages, unet, dec


def _p(x):
    """int pointer / tensor / None → c_void_p."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return C.c_void_p(int(x))


def debug_gemm(A, B, bias, D, M, N, K, out_f32=0, act=ACT_NONE, stream=None):
    call("sd_debug_gemm", _p(A), _p(B), _p(bias), _p(D), M, N, K, out_f32, act, _p(stream))


def debug_conv3x3(x, cin, x2, cin2, w, w2, bias, temb, res, y, nb, h, wd, cout, stream=None):
    call("sd_debug_conv3x3", _p(x), cin, _p(x2), cin2, _p(w), _p(w2), _p(bias), _p(temb), _p(res), _p(y),
         nb, h, wd, cout, _p(stream))
